// gnw.hpp -- header-only C++ face of the gnw C-ABI for reference (ertinv) callers.
//
// The reference's Woodbury-MINRES block (proj/src/inversion.cpp:240-271) is
//     WoodburyPreconditioner pc = build_woodbury_preconditioner(q_diag_inv, amg, J, beta, &t);
//     SaddleOperator op{&Q, &D, &J, beta};
//     Vector b = assemble_gn_rhs(m, m_ref, g, g_obs, J, D, beta);
//     auto [x, rep] = minres(op.apply, pc.apply, b, x0, tol, maxit);
// With this header it becomes:
//     gnw::GnStepSolver s(mesh_vertices, mesh_cells, amg_options);        // once per inversion
//     s.build_woodbury_preconditioner(J.values.data(), J.n_rows, beta, &t);
//     std::vector<double> b = s.assemble_gn_rhs(m, m_ref, g, g_obs);
//     gnw::MinresReport rep;  std::vector<double> x = s.minres(b, x0, tol, maxit, &rep);
// Errors are rethrown with the reference's exception types and message texts.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "gnw.h"

namespace gnw {

struct DeviceFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void throw_on(gnw_status s) {
  if (s == GNW_OK) return;
  const std::string msg = gnw_last_error();
  if (s == GNW_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (s == GNW_DEVICE) throw DeviceFailure(msg);
  throw std::runtime_error(msg);
}

struct AmgOptions {  // ertinv::AmgOptions, amg.hpp:11-23
  std::uint64_t coarse_threshold = 64;
  double strength = 0.08;
  double jacobi_damping = 2.0 / 3.0;
  double prolongation_damping = 2.0 / 3.0;
  std::uint64_t max_aggregate_size = 3;
  std::uint64_t max_levels = 25;
};

struct WoodburyBuildTimings {  // inversion.hpp:41-45
  double t_H = 0.0, t_C = 0.0, t_chol = 0.0;
};

struct MinresReport {  // minres.hpp:13-22
  std::size_t iterations = 0;
  std::vector<double> relative_residuals;
  std::vector<double> pnorm_relative_residuals;
  bool converged = false;
  double true_relative_residual = 0.0;
};

class GnStepSolver {
 public:
  // make_mixed_spaces + assemble_Q/D + amg_setup(assemble_lumped_schur(Q, D)) on `device`
  GnStepSolver(const std::vector<double>& vertices_xz, const std::vector<std::int64_t>& cells,
               const AmgOptions& o = {}, int device = 0) {
    throw_on(gnw_create(1, &device, &ctx_));
    const gnw_mesh mesh{vertices_xz.size() / 2, vertices_xz.data(), cells.size() / 3, cells.data()};
    const gnw_amg_options opts{o.coarse_threshold, o.strength, o.jacobi_damping, o.prolongation_damping,
                               o.max_aggregate_size, o.max_levels};
    try {
      throw_on(gnw_assemble(ctx_, &mesh, &opts));
      gnw_info info;
      throw_on(gnw_get_info(ctx_, &info));
      K_ = info.K;
      N_ = info.N;
    } catch (...) {
      gnw_destroy(ctx_);
      throw;
    }
  }
  ~GnStepSolver() { gnw_destroy(ctx_); }
  GnStepSolver(const GnStepSolver&) = delete;
  GnStepSolver& operator=(const GnStepSolver&) = delete;

  std::size_t n_flux_dofs() const { return K_; }
  std::size_t n_cell_dofs() const { return N_; }

  // build_woodbury_preconditioner (inversion.hpp:47-50); J row-major m x N
  void build_woodbury_preconditioner(const double* J, std::size_t m, double beta,
                                     WoodburyBuildTimings* timings = nullptr) {
    throw_on(gnw_set_preconditioner(ctx_, GNW_PC_WOODBURY));
    set_jacobian(J, m, beta, timings);
  }
  // GnAlgorithm::kLaplaceMinres (inversion.cpp:251-256): J in the operator, bare V-cycle preconditioner
  void laplace_preconditioner(const double* J, std::size_t m, double beta) {
    throw_on(gnw_set_preconditioner(ctx_, GNW_PC_LAPLACE));
    set_jacobian(J, m, beta, nullptr);
  }
  // assemble_gn_rhs (inversion.hpp:53-55)
  std::vector<double> assemble_gn_rhs(const std::vector<double>& m, const std::vector<double>& m_ref,
                                      const std::vector<double>& g, const std::vector<double>& g_obs) {
    std::vector<double> rhs(K_ + N_);
    throw_on(gnw_assemble_rhs(ctx_, m.data(), m_ref.data(), g.data(), g_obs.data(), rhs.data()));
    return rhs;
  }
  // SaddleOperator::apply / WoodburyPreconditioner::apply / amg_apply
  std::vector<double> apply_operator(const std::vector<double>& x) { return unary(gnw_apply_operator, x, K_ + N_); }
  std::vector<double> precondition(const std::vector<double>& y) { return unary(gnw_precondition, y, K_ + N_); }
  std::vector<double> amg_apply(const std::vector<double>& r) { return unary(gnw_amg_apply, r, N_); }
  // minres(op.apply, pc.apply, b, x0, tol, maxit) (minres.hpp:29-33)
  std::vector<double> minres(const std::vector<double>& b, const std::vector<double>& x0, double tol,
                             std::size_t maxit, MinresReport* report = nullptr) {
    std::vector<double> x(b.size());
    // histories: a small first buffer (not maxit + 1 -- 2 (K + N) is 42M at C3), the rest
    // fetched after the solve only when the run was longer
    std::vector<double> he(std::min<std::size_t>(maxit, 4095) + 1), hp(he.size());
    gnw_report r{};
    r.relative_residuals = he.data();
    r.pnorm_relative_residuals = hp.data();
    r.hist_cap = he.size();
    throw_on(gnw_minres_solve(ctx_, b.data(), x0.data(), x.data(), tol, maxit, &r));
    if (report) fill_report(r, he, hp, report);
    return x;
  }
  // The reference's GN-step solve as it appears in gauss_newton (inversion.cpp:259-265):
  // b = assemble_gn_rhs(...), x0 = 0, minres(op, pc, b, x0, tol, maxit) -- one call, b stays
  // on the device
  std::vector<double> solve_gn_step(const std::vector<double>& m, const std::vector<double>& m_ref,
                                    const std::vector<double>& g, const std::vector<double>& g_obs, double tol,
                                    std::size_t maxit, MinresReport* report = nullptr) {
    std::vector<double> x(K_ + N_);
    std::vector<double> he(std::min<std::size_t>(maxit, 4095) + 1), hp(he.size());
    gnw_report r{};
    r.relative_residuals = he.data();
    r.pnorm_relative_residuals = hp.data();
    r.hist_cap = he.size();
    throw_on(gnw_gn_step_solve(ctx_, m.data(), m_ref.data(), g.data(), g_obs.data(), x.data(), tol, maxit, &r));
    if (report) fill_report(r, he, hp, report);
    return x;
  }
  gnw_ctx* handle() { return ctx_; }

 private:
  void fill_report(const gnw_report& r, std::vector<double>& he, std::vector<double>& hp, MinresReport* report) {
    report->iterations = r.iterations;
    report->converged = r.converged != 0;
    report->true_relative_residual = r.true_relative_residual;
    if (r.n_hist > he.size()) {
      he.resize(r.n_hist);
      hp.resize(r.n_hist);
      throw_on(gnw_minres_history(ctx_, he.data(), hp.data(), he.size(), nullptr));
    }
    const std::size_t nh = std::min<std::size_t>(r.n_hist, he.size());
    report->relative_residuals.assign(he.begin(), he.begin() + static_cast<std::ptrdiff_t>(nh));
    report->pnorm_relative_residuals.assign(hp.begin(), hp.begin() + static_cast<std::ptrdiff_t>(nh));
  }
  void set_jacobian(const double* J, std::size_t m, double beta, WoodburyBuildTimings* timings) {
    gnw_timings t{};
    throw_on(gnw_set_jacobian(ctx_, J, m, N_, beta, &t));
    if (timings) *timings = {t.t_H, t.t_C, t.t_chol};
  }
  template <class F>
  std::vector<double> unary(F f, const std::vector<double>& in, std::size_t n_out) {
    std::vector<double> out(n_out);
    throw_on(f(ctx_, in.data(), out.data()));
    return out;
  }
  gnw_ctx* ctx_ = nullptr;
  std::size_t K_ = 0, N_ = 0;
};

}  // namespace gnw
