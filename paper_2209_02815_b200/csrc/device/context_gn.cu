// context_gn.cu -- gauss_newton (proj/src/inversion.cpp:187-292) for the iterative
// algorithms (kWoodburyMinres, kLaplaceMinres) on one context.  Every step stays on the
// device: the forward response and J (context_ert.cu) are written into context-owned
// device buffers, which the Woodbury build and the operator then reference without a
// copy (device-pointer mode, like the reference's SaddleOperator{&Q, &D, &rj.J, beta}).
#include <chrono>
#include <cmath>

#include "context.cuh"

namespace gnw {

namespace {
using Clock = std::chrono::steady_clock;

// norm2 (linalg.cpp:20-22): sqrt of the sequential dot
double norm2_seq(const std::vector<double>& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

struct PtrModeScope {  // the loop drives the context with device pointers; restore on exit
  int& mode;
  int saved;
  explicit PtrModeScope(int& m) : mode(m), saved(m) { mode = 1; }
  ~PtrModeScope() { mode = saved; }
};
}  // namespace

GnResult Context::gauss_newton(const double* m0, const double* m_ref, const host::ErtConfig* cfgs, int64_t n_cfg,
                               const double* g_obs, const GnConfig& cfg, double* m_out) {
  if (!(cfg.beta > 0.0)) throw std::invalid_argument("gauss_newton: beta must be positive");
  require_mixed();
  require_device();
  if (comm_) throw std::invalid_argument("gauss_newton: not available on a partitioned context");
  if (electrodes_.empty()) throw std::invalid_argument("gauss_newton: missing mesh or survey");
  if (n_cfg <= 0) throw std::invalid_argument("gauss_newton: observation count mismatch");
  const int64_t N = N_, K = K_, M = n_cfg;
  const uint64_t maxit = cfg.minres_maxit > 0 ? cfg.minres_maxit : 2 * static_cast<uint64_t>(K + N);
  const cudaStream_t s = stream_;

  // caller vectors are host or device per the pointer mode; the loop keeps device copies
  const bool caller_dev = ptr_mode == 1;
  std::vector<double> m(N), mref(N), gobs(M);
  auto fetch = [&](std::vector<double>& dst, const double* src, int64_t n) {
    if (caller_dev)
      GNW_CUDA_CHECK(cudaMemcpy(dst.data(), src, n * sizeof(double), cudaMemcpyDeviceToHost));
    else
      std::copy(src, src + n, dst.begin());
  };
  fetch(m, m0, N);
  fetch(mref, m_ref, N);
  fetch(gobs, g_obs, M);

  DeviceMemory gm;
  double* dm = gm.alloc<double>(N);
  double* dmref = gm.alloc<double>(N);
  double* dgobs = gm.alloc<double>(M);
  double* dJ = gm.alloc<double>(static_cast<size_t>(M) * N);
  double* dg = gm.alloc<double>(M);
  double* db = gm.alloc<double>(K + N);
  double* dx0 = gm.alloc<double>(K + N);
  double* dx = gm.alloc<double>(K + N);
  GNW_CUDA_CHECK(cudaMemcpyAsync(dmref, mref.data(), N * sizeof(double), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dgobs, gobs.data(), M * sizeof(double), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemsetAsync(dx0, 0, (K + N) * sizeof(double), s));  // x0 = 0 (inversion.cpp:262)

  PtrModeScope scope(ptr_mode);
  const int saved_pc = pc_laplace;
  pc_laplace = cfg.laplace;
  GnResult res;
  std::vector<double> g(M), delta(N);
  auto misfit_at = [&](bool want_J, GnStepReport* sr) {
    GNW_CUDA_CHECK(cudaMemcpyAsync(dm, m.data(), N * sizeof(double), cudaMemcpyHostToDevice, s));
    const auto t0 = Clock::now();
    ErtTimings et;
    response_jacobian(dm, cfgs, M, dJ, dg, cfg.forward_tol, &et);  // evaluate_response_and_jacobian
    if (sr) sr->t_forward = std::chrono::duration<double>(Clock::now() - t0).count();
    (void)want_J;
    GNW_CUDA_CHECK(cudaMemcpyAsync(g.data(), dg, M * sizeof(double), cudaMemcpyDeviceToHost, s));
    sync();
    std::vector<double> dgv(M);
    for (int64_t i = 0; i < M; ++i) dgv[i] = g[i] - gobs[i];  // inversion.cpp:225-226
    return norm2_seq(dgv);
  };
  try {
    for (uint64_t step = 0; step < cfg.max_outer_steps; ++step) {
      GnStepReport sr;
      sr.misfit = misfit_at(true, &sr);
      const auto t0 = Clock::now();
      double tm[3] = {0, 0, 0};
      // build_woodbury_preconditioner (or the Laplace preconditioner) + SaddleOperator{.., &J, beta}
      set_jacobian(dJ, M, N, cfg.beta, tm);
      sr.t_H = tm[0];
      sr.t_C = tm[1];
      sr.t_chol = tm[2];
      assemble_rhs(dm, dmref, dg, dgobs, db);                       // assemble_gn_rhs
      const MinresResult mr = minres(db, dx0, dx, cfg.minres_tol, maxit);
      sr.minres_iters = mr.iterations;
      sr.converged = mr.converged;
      sr.euclid_relative_residual = mr.true_rel;
      sr.pnorm_relative_residual = mr.hist_p.empty() ? 0.0 : mr.hist_p.back();
      GNW_CUDA_CHECK(cudaMemcpyAsync(delta.data(), dx + K, N * sizeof(double), cudaMemcpyDeviceToHost, s));
      sync();
      sr.t_norm = std::chrono::duration<double>(Clock::now() - t0).count();
      for (double v : delta)
        if (!std::isfinite(v)) throw std::runtime_error("gauss_newton: non-finite model update");
      for (int64_t i = 0; i < N; ++i) m[i] += delta[i];
      res.steps.push_back(sr);
      if (cfg.misfit_reduction_tol > 0.0 && step > 0) {  // inversion.cpp:280-283
        const double prev = res.steps[res.steps.size() - 2].misfit;
        if (sr.misfit > (1.0 - cfg.misfit_reduction_tol) * prev) break;
      }
    }
    res.final_misfit = misfit_at(false, nullptr);
  } catch (...) {
    pc_laplace = saved_pc;
    throw;
  }
  pc_laplace = saved_pc;
  if (m_out) {
    if (caller_dev)
      GNW_CUDA_CHECK(cudaMemcpy(m_out, m.data(), N * sizeof(double), cudaMemcpyHostToDevice));
    else
      std::copy(m.begin(), m.end(), m_out);
  }
  // the context must not keep pointers into this call's buffers
  destroy_graph();
  dJ_ = nullptr;
  m_ = 0;
  pa_.m = 0;
  op_.J = nullptr;
  op_.m = 0;
  return res;
}

}  // namespace gnw
