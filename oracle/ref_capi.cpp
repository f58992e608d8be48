// ref_capi.cpp -- TEST INFRASTRUCTURE: C API (orc_api.h) over the UNMODIFIED
// reference library compiled from /root/reference/proj/src by oracle/Makefile.
// Every call forwards to the reference's own functions; nothing here restates
// an algorithm.  Output: oracle/_ref/libertinv_ref.so (git-ignored).
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "ertinv/amg.hpp"
#include "ertinv/fem_mixed.hpp"
#include "ertinv/forward.hpp"
#include "ertinv/survey.hpp"
#include "ertinv/inversion.hpp"
#include "ertinv/linalg.hpp"
#include "ertinv/mesh.hpp"
#include "ertinv/minres.hpp"
#include "ertinv/sparse.hpp"
#include "orc_api.h"

using namespace ertinv;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

AmgOptions to_opts(const orc_amg_opts* o) {
  AmgOptions a;
  if (o) {
    a.coarse_threshold = o->coarse_threshold;
    a.strength = o->strength;
    a.jacobi_damping = o->jacobi_damping;
    a.prolongation_damping = o->prolongation_damping;
    a.max_aggregate_size = o->max_aggregate_size;
    a.max_levels = o->max_levels;
  }
  return a;
}
}  // namespace

struct orc_problem {
  bool mixed = false;
  Mesh mesh;
  MixedSpaces spaces;
  SparseMatrix Q, D, S;
  Vector qinv;
  AmgHierarchy amg;
  DenseMatrix J;
  double beta = 1.0;
  bool has_J = false;
  bool pc_laplace = false;
  WoodburyPreconditioner pc;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_flavor(void) { return "reference"; }

orc_problem* orc_create_mixed(const double* vertices, uint64_t n_vertices, const int64_t* cells,
                              uint64_t n_cells, const orc_amg_opts* opts) {
  auto p = std::make_unique<orc_problem>();
  int rc = guard([&] {
    std::vector<std::array<double, 2>> v(n_vertices);
    for (uint64_t i = 0; i < n_vertices; ++i) v[i] = {vertices[2 * i], vertices[2 * i + 1]};
    std::vector<std::array<std::size_t, 3>> c(n_cells);
    for (uint64_t i = 0; i < n_cells; ++i)
      c[i] = {static_cast<std::size_t>(cells[3 * i]), static_cast<std::size_t>(cells[3 * i + 1]),
              static_cast<std::size_t>(cells[3 * i + 2])};
    p->mesh = finalize_mesh(std::move(v), std::move(c), {});
    p->spaces = make_mixed_spaces(p->mesh);
    p->Q = assemble_Q(p->spaces);
    p->D = assemble_D(p->spaces);
    // inversion.cpp:210-212
    p->qinv = diagonal(p->Q);
    for (double& x : p->qinv) x = 1.0 / x;
    p->S = assemble_lumped_schur(p->Q, p->D);
    p->amg = amg_setup(p->S, to_opts(opts));
    p->mixed = true;
    p->pc.q_diag_inv = &p->qinv;
    p->pc.amg = &p->amg;
    p->pc.J = nullptr;
  });
  if (rc) return nullptr;
  return p.release();
}

orc_problem* orc_create_amg_csr(uint64_t n, const int64_t* rowptr, const int64_t* cols,
                                const double* vals, const orc_amg_opts* opts) {
  auto p = std::make_unique<orc_problem>();
  int rc = guard([&] {
    std::vector<Triplet> trip;
    for (uint64_t i = 0; i < n; ++i)
      for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
        trip.push_back({i, static_cast<std::size_t>(cols[k]), vals[k]});
    p->S = from_triplets(n, n, std::move(trip));
    p->amg = amg_setup(p->S, to_opts(opts));
  });
  if (rc) return nullptr;
  return p.release();
}

void orc_destroy(orc_problem* p) { delete p; }

int orc_sizes(const orc_problem* p, uint64_t s[8]) {
  std::memset(s, 0, 8 * sizeof(uint64_t));
  if (p->mixed) {
    s[0] = p->spaces.n_flux_dofs;
    s[1] = p->spaces.n_cell_dofs;
    s[2] = p->mesh.n_vertices();
    s[3] = p->mesh.n_cells();
    s[4] = p->mesh.n_edges();
    s[6] = p->mesh.boundary_edges.size();
  } else {
    s[1] = p->S.n_rows;
  }
  s[5] = p->amg.n_levels();
  s[7] = p->amg.levels.empty() ? 0 : p->amg.levels.back().matrix.n_rows;
  return 0;
}

int orc_mesh(const orc_problem* p, int64_t* cells, int64_t* edges, int64_t* cell_edges,
             int32_t* signs, int64_t* bedges, int32_t* btags) {
  if (!p->mixed) {
    g_err = "orc_mesh: not a mixed problem";
    return 1;
  }
  const Mesh& m = p->mesh;
  for (std::size_t c = 0; c < m.n_cells(); ++c)
    for (int k = 0; k < 3; ++k) {
      if (cells) cells[3 * c + k] = static_cast<int64_t>(m.cells[c][k]);
      if (cell_edges) cell_edges[3 * c + k] = static_cast<int64_t>(m.cell_edges[c][k]);
      if (signs) signs[3 * c + k] = m.cell_edge_signs[c][k];
    }
  for (std::size_t e = 0; e < m.n_edges(); ++e)
    for (int k = 0; k < 2; ++k)
      if (edges) edges[2 * e + k] = static_cast<int64_t>(m.edges[e][k]);
  for (std::size_t b = 0; b < m.boundary_edges.size(); ++b) {
    if (bedges) bedges[b] = static_cast<int64_t>(m.boundary_edges[b].edge);
    if (btags) btags[b] = m.boundary_edges[b].tag == BoundaryTag::kSurface ? 0 : 1;
  }
  return 0;
}

int orc_csr(const orc_problem* p, int which, uint64_t level, uint64_t* n_rows, uint64_t* n_cols,
            uint64_t* nnz, int64_t* rowptr, int64_t* cols, double* vals) {
  const SparseMatrix* A = nullptr;
  switch (which) {
    case 0: A = &p->Q; break;
    case 1: A = &p->D; break;
    case 2: A = &p->S; break;
    case 3:
    case 4:
      if (level >= p->amg.n_levels()) {
        g_err = "orc_csr: level out of range";
        return 1;
      }
      A = which == 3 ? &p->amg.levels[level].matrix : &p->amg.levels[level].prolongation;
      break;
    default: g_err = "orc_csr: bad selector"; return 1;
  }
  if (n_rows) *n_rows = A->n_rows;
  if (n_cols) *n_cols = A->n_cols;
  if (nnz) *nnz = A->nnz();
  if (rowptr)
    for (std::size_t i = 0; i < A->row_offsets.size(); ++i) rowptr[i] = static_cast<int64_t>(A->row_offsets[i]);
  if (cols)
    for (std::size_t k = 0; k < A->nnz(); ++k) cols[k] = static_cast<int64_t>(A->column_indices[k]);
  if (vals) std::memcpy(vals, A->values.data(), A->nnz() * sizeof(double));
  return 0;
}

int orc_level_inv_diag(const orc_problem* p, uint64_t level, double* out) {
  if (level >= p->amg.n_levels()) {
    g_err = "orc_level_inv_diag: level out of range";
    return 1;
  }
  const Vector& d = p->amg.levels[level].inv_diag;
  std::memcpy(out, d.data(), d.size() * sizeof(double));
  return 0;
}

int orc_coarse_cholesky(const orc_problem* p, double* out) {
  const DenseMatrix& L = p->amg.coarse_cholesky;
  std::memcpy(out, L.values.data(), L.values.size() * sizeof(double));
  return 0;
}

int orc_q_diag_inv(const orc_problem* p, double* out) {
  std::memcpy(out, p->qinv.data(), p->qinv.size() * sizeof(double));
  return 0;
}

int orc_amg_apply(const orc_problem* p, const double* r, double* z) {
  return guard([&] {
    const std::size_t n = p->amg.size();
    const Vector out = amg_apply(p->amg, std::span<const double>(r, n));
    std::memcpy(z, out.data(), n * sizeof(double));
  });
}

int orc_set_jacobian(orc_problem* p, const double* J, uint64_t m, double beta, double timings[3]) {
  return guard([&] {
    if (!p->mixed) throw std::invalid_argument("orc_set_jacobian: not a mixed problem");
    const std::size_t N = p->spaces.n_cell_dofs;
    p->beta = beta;
    if (m == 0) {
      // Laplace-only preconditioner, inversion.cpp:251-256
      p->has_J = false;
      p->J = DenseMatrix();
      p->pc = WoodburyPreconditioner();
      p->pc.q_diag_inv = &p->qinv;
      p->pc.amg = &p->amg;
      p->pc.J = nullptr;
      p->pc.beta = beta;
      if (timings) timings[0] = timings[1] = timings[2] = 0.0;
      return;
    }
    p->J = DenseMatrix(m, N);
    std::memcpy(p->J.values.data(), J, m * N * sizeof(double));
    p->has_J = true;
    if (p->pc_laplace) {  // inversion.cpp:251-256
      p->pc = WoodburyPreconditioner();
      p->pc.q_diag_inv = &p->qinv;
      p->pc.amg = &p->amg;
      p->pc.J = nullptr;
      p->pc.beta = beta;
      if (timings) timings[0] = timings[1] = timings[2] = 0.0;
      return;
    }
    WoodburyBuildTimings t;
    p->pc = build_woodbury_preconditioner(p->qinv, p->amg, p->J, beta, &t);
    if (timings) {
      timings[0] = t.t_H;
      timings[1] = t.t_C;
      timings[2] = t.t_chol;
    }
  });
}

int orc_set_pc_laplace(orc_problem* p, int laplace) {
  p->pc_laplace = laplace != 0;
  return 0;
}

int orc_get_H(const orc_problem* p, double* out) {
  std::memcpy(out, p->pc.h_hat.values.data(), p->pc.h_hat.values.size() * sizeof(double));
  return 0;
}

int orc_get_L(const orc_problem* p, double* out) {
  const auto& L = p->pc.capacitance_chol;
  std::memcpy(out, L.values.data(), L.values.size() * sizeof(double));
  return 0;
}

int orc_apply_operator(const orc_problem* p, const double* x, double* y) {
  return guard([&] {
    SaddleOperator op{&p->Q, &p->D, p->has_J ? &p->J : nullptr, p->beta};
    const std::size_t n = op.size();
    const Vector out = op.apply(std::span<const double>(x, n));
    std::memcpy(y, out.data(), n * sizeof(double));
  });
}

int orc_precondition(const orc_problem* p, const double* y, double* z) {
  return guard([&] {
    const std::size_t n = p->Q.n_rows + p->D.n_rows;
    const Vector out = p->pc.apply(std::span<const double>(y, n));
    std::memcpy(z, out.data(), n * sizeof(double));
  });
}

int orc_assemble_rhs(const orc_problem* p, const double* m, const double* m_ref, const double* g,
                     const double* g_obs, double* rhs) {
  return guard([&] {
    const std::size_t N = p->D.n_rows;
    const std::size_t M = p->J.n_rows;
    const ModelVector mv(m, m + N), mr(m_ref, m_ref + N);
    const Vector gv(g, g + M), go(g_obs, g_obs + M);
    const Vector out = assemble_gn_rhs(mv, mr, gv, go, p->J, p->D, p->beta);
    std::memcpy(rhs, out.data(), out.size() * sizeof(double));
  });
}

int orc_minres(const orc_problem* p, const double* b, const double* x0, double tol, uint64_t maxit,
               double* x, orc_minres_report* rep, double* he, double* hp, uint64_t cap) {
  return guard([&] {
    SaddleOperator op{&p->Q, &p->D, p->has_J ? &p->J : nullptr, p->beta};
    const std::size_t n = op.size();
    auto [sol, r] = minres([&op](std::span<const double> v) { return op.apply(v); },
                           [p](std::span<const double> v) { return p->pc.apply(v); },
                           std::span<const double>(b, n), std::span<const double>(x0, n), tol,
                           maxit);
    std::memcpy(x, sol.data(), n * sizeof(double));
    rep->iterations = r.iterations;
    rep->converged = r.converged ? 1 : 0;
    rep->true_relative_residual = r.true_relative_residual;
    const std::size_t h = std::min<std::size_t>(cap, r.relative_residuals.size());
    rep->n_hist = r.relative_residuals.size();
    for (std::size_t i = 0; i < h; ++i) {
      if (he) he[i] = r.relative_residuals[i];
      if (hp) hp[i] = r.pnorm_relative_residuals[i];
    }
  });
}

// Bounded CPU sample of one GN-step solve (bench.py cpu_baseline / --impl
// reference).  Times the reference's own functions on full-size operands:
//   out[0] seconds per H column (amg_apply of one J row, inversion.cpp:107-114)
//   out[1] seconds per capacitance row (matmul of k_rows J rows with an N x m
//          operand, linalg.cpp:56-70; dense J so no zero-skipping)
//   out[2] seconds of the m x m dense_cholesky (linalg.cpp:88-105), full size
//   out[3] seconds per MINRES iteration (minres.cpp:70-148) with the full
//          SaddleOperator and a WoodburyPreconditioner of the full shape (H = 0,
//          L = I: identical work per apply, guaranteed SPD)
int orc_sample_gnstep(orc_problem* p, const double* J, uint64_t m, double beta, uint64_t k_cols,
                      uint64_t k_rows, uint64_t k_iters, double out[5]) {
  return guard([&] {
    using Clock = std::chrono::steady_clock;
    const std::size_t N = p->spaces.n_cell_dofs, K = p->spaces.n_flux_dofs;
    DenseMatrix Jm(m, N);
    std::memcpy(Jm.values.data(), J, m * N * sizeof(double));
    auto t0 = Clock::now();
    Vector col(N);
    for (std::size_t i = 0; i < k_cols; ++i) {
      for (std::size_t c = 0; c < N; ++c) col[c] = Jm(i % m, c);
      const Vector h = amg_apply(p->amg, col);
      if (h.empty()) throw std::runtime_error("sample: empty V-cycle");
    }
    out[0] = std::chrono::duration<double>(Clock::now() - t0).count() / static_cast<double>(k_cols);
    DenseMatrix Jsub(k_rows, N);
    std::memcpy(Jsub.values.data(), J, k_rows * N * sizeof(double));
    DenseMatrix Hfake(N, m);
    t0 = Clock::now();
    DenseMatrix Csub = matmul(Jsub, Hfake);
    out[1] = std::chrono::duration<double>(Clock::now() - t0).count() / static_cast<double>(k_rows);
    DenseMatrix Cfull = DenseMatrix::identity(m);
    t0 = Clock::now();
    DenseMatrix L = dense_cholesky(Cfull);
    out[2] = std::chrono::duration<double>(Clock::now() - t0).count();
    WoodburyPreconditioner pc;
    pc.q_diag_inv = &p->qinv;
    pc.amg = &p->amg;
    pc.J = &Jm;
    pc.beta = beta;
    pc.h_hat = std::move(Hfake);
    pc.capacitance_chol = std::move(L);
    SaddleOperator op{&p->Q, &p->D, &Jm, beta};
    Vector b(K + N), x0(K + N, 0.0);
    for (std::size_t i = 0; i < b.size(); ++i) b[i] = std::sin(0.37 * static_cast<double>(i) + 1.0);
    // minres runs one operator and one preconditioner application before its first iteration
    // (r0 = b - A x0, z0 = P r0, minres.cpp:40-49): two runs of k and 2k iterations separate the
    // per-iteration cost from that fixed part (out[4]), which a full solve pays once.
    auto run = [&](std::size_t k) {
      const auto t = Clock::now();
      auto res = minres([&op](std::span<const double> v) { return op.apply(v); },
                        [&pc](std::span<const double> v) { return pc.apply(v); }, b, x0, 1e-300, k);
      return std::pair(std::chrono::duration<double>(Clock::now() - t).count(),
                       static_cast<double>(std::max<std::size_t>(res.second.iterations, 1)));
    };
    const auto [t1, k1] = run(k_iters);
    const auto [t2, k2] = run(2 * k_iters);
    const double per = k2 > k1 ? (t2 - t1) / (k2 - k1) : t1 / k1;
    out[3] = per;
    out[4] = std::max(0.0, t1 - k1 * per);
  });
}

int orc_response_jacobian(orc_problem* p, const int64_t* nodes, uint64_t n_nodes, const int64_t* a, const int64_t* b,
                          const int64_t* m, const int64_t* n, const double* k, uint64_t n_cfg, const double* model,
                          double* J, double* g) {
  return guard([&] {
    if (!p->mixed) throw std::invalid_argument("orc_response_jacobian: not a mixed problem");
    p->mesh.electrode_nodes.assign(nodes, nodes + n_nodes);
    Survey survey;
    for (uint64_t e = 0; e < n_nodes; ++e) survey.electrode_positions.push_back(p->mesh.vertices[nodes[e]][0]);
    for (uint64_t i = 0; i < n_cfg; ++i) {
      ElectrodeConfig c;
      c.a = static_cast<std::size_t>(a[i]);
      c.b = static_cast<std::ptrdiff_t>(b[i]);
      c.m = static_cast<std::size_t>(m[i]);
      c.n = static_cast<std::size_t>(n[i]);
      c.k = k[i];
      survey.configs.push_back(c);
    }
    const ModelVector mv(model, model + p->mesh.n_cells());
    const ResponseJacobian rj = evaluate_response_and_jacobian(p->mesh, mv, survey);
    std::memcpy(J, rj.J.values.data(), rj.J.values.size() * sizeof(double));
    std::memcpy(g, rj.g.data(), rj.g.size() * sizeof(double));
  });
}

int orc_gauss_newton(orc_problem* p, const int64_t* nodes, uint64_t n_nodes, const int64_t* a, const int64_t* b,
                     const int64_t* m, const int64_t* n, const double* k, uint64_t n_cfg, const double* g_obs,
                     const double* m_ref, const double* m0, double beta, uint64_t max_outer_steps, double minres_tol,
                     uint64_t minres_maxit, int algorithm, double misfit_reduction_tol, double* m_out,
                     double* steps, uint64_t steps_cap, uint64_t* n_steps, double* final_misfit) {
  return guard([&] {
    if (!p->mixed) throw std::invalid_argument("orc_gauss_newton: not a mixed problem");
    p->mesh.electrode_nodes.assign(nodes, nodes + n_nodes);
    Survey survey;
    for (uint64_t e = 0; e < n_nodes; ++e) survey.electrode_positions.push_back(p->mesh.vertices[nodes[e]][0]);
    for (uint64_t i = 0; i < n_cfg; ++i) {
      ElectrodeConfig c;
      c.a = static_cast<std::size_t>(a[i]);
      c.b = static_cast<std::ptrdiff_t>(b[i]);
      c.m = static_cast<std::size_t>(m[i]);
      c.n = static_cast<std::size_t>(n[i]);
      c.k = k[i];
      survey.configs.push_back(c);
    }
    const std::size_t N = p->mesh.n_cells();
    GnProblem prob;
    prob.mesh = &p->mesh;
    prob.survey = &survey;
    prob.g_obs.assign(g_obs, g_obs + n_cfg);
    prob.m_ref.assign(m_ref, m_ref + N);
    prob.m0.assign(m0, m0 + N);
    GnConfig cfg;
    cfg.beta = beta;
    cfg.max_outer_steps = max_outer_steps;
    cfg.minres_tol = minres_tol;
    cfg.minres_maxit = minres_maxit;
    cfg.algorithm = algorithm == 1 ? GnAlgorithm::kLaplaceMinres : GnAlgorithm::kWoodburyMinres;
    cfg.misfit_reduction_tol = misfit_reduction_tol;
    auto [mv, rep] = gauss_newton(prob, cfg);  // inversion.cpp:187-292, unmodified
    std::memcpy(m_out, mv.data(), N * sizeof(double));
    *n_steps = rep.steps.size();
    *final_misfit = rep.final_misfit;
    for (std::size_t i = 0; i < std::min<std::size_t>(steps_cap, rep.steps.size()); ++i) {
      const GnStepReport& q = rep.steps[i];
      double* o = steps + 5 * i;
      o[0] = q.misfit;
      o[1] = static_cast<double>(q.minres_iters);
      o[2] = q.converged ? 1.0 : 0.0;
      o[3] = q.euclid_relative_residual;
      o[4] = q.pnorm_relative_residual;
    }
  });
}

/* ---- the reference's file formats (used to pin paper_2209_02815_b200/io.py) ---- */
int orc_io_write_mesh(orc_problem* p, const int64_t* electrodes, uint64_t ne, const char* path) {
  return guard([&] {
    p->mesh.electrode_nodes.assign(electrodes, electrodes + ne);
    write_mesh_json(p->mesh, path);
  });
}

int orc_io_read_mesh(const char* path, uint64_t* nv, uint64_t* nc, uint64_t* ne, double* vertices, int64_t* cells,
                     int64_t* electrodes) {
  return guard([&] {
    const Mesh m = read_mesh_json(path);
    *nv = m.vertices.size();
    *nc = m.cells.size();
    *ne = m.electrode_nodes.size();
    if (vertices)
      for (std::size_t i = 0; i < m.vertices.size(); ++i) {
        vertices[2 * i] = m.vertices[i][0];
        vertices[2 * i + 1] = m.vertices[i][1];
      }
    if (cells)
      for (std::size_t c = 0; c < m.cells.size(); ++c)
        for (int k = 0; k < 3; ++k) cells[3 * c + k] = static_cast<int64_t>(m.cells[c][k]);
    if (electrodes)
      for (std::size_t e = 0; e < m.electrode_nodes.size(); ++e) electrodes[e] = static_cast<int64_t>(m.electrode_nodes[e]);
  });
}

int orc_io_write_survey(const int64_t* a, const int64_t* b, const int64_t* m, const int64_t* n, const double* k,
                        uint64_t count, const char* path) {
  return guard([&] {
    Survey s;
    for (uint64_t i = 0; i < count; ++i) {
      ElectrodeConfig c;
      c.a = static_cast<std::size_t>(a[i]);
      c.b = static_cast<std::ptrdiff_t>(b[i]);
      c.m = static_cast<std::size_t>(m[i]);
      c.n = static_cast<std::size_t>(n[i]);
      c.k = k[i];
      s.configs.push_back(c);
    }
    write_survey_csv(s, path);
  });
}

int orc_io_read_survey(const char* path, uint64_t* count, int64_t* a, int64_t* b, int64_t* m, int64_t* n, double* k) {
  return guard([&] {
    const Survey s = read_survey_csv(path);
    *count = s.configs.size();
    if (a)
      for (std::size_t i = 0; i < s.configs.size(); ++i) {
        a[i] = static_cast<int64_t>(s.configs[i].a);
        b[i] = static_cast<int64_t>(s.configs[i].b);
        m[i] = static_cast<int64_t>(s.configs[i].m);
        n[i] = static_cast<int64_t>(s.configs[i].n);
        k[i] = s.configs[i].k;
      }
  });
}

int orc_io_write_vector(int kind, const double* v, uint64_t count, const char* path) {
  return guard([&] {
    const Vector x(v, v + count);
    if (kind == 0)
      write_model_json(x, path);
    else
      write_observations_csv(x, path);
  });
}

int orc_io_read_vector(int kind, const char* path, uint64_t* count, double* v) {
  return guard([&] {
    const Vector x = kind == 0 ? read_model_json(path) : read_observations_csv(path);
    *count = x.size();
    if (v) std::memcpy(v, x.data(), x.size() * sizeof(double));
  });
}

int orc_io_write_result(const double* m, uint64_t N, const double* steps, uint64_t n_steps, double final_misfit,
                        uint64_t K, uint64_t M, const char* path) {
  return guard([&] {
    GnReport r;
    for (uint64_t i = 0; i < n_steps; ++i) {
      const double* q = steps + 9 * i;
      GnStepReport s;
      s.misfit = q[0];
      s.minres_iters = static_cast<std::size_t>(q[1]);
      s.converged = q[2] != 0.0;
      s.euclid_relative_residual = q[3];
      s.pnorm_relative_residual = q[4];
      s.t_H = q[5];
      s.t_C = q[6];
      s.t_chol = q[7];
      s.t_norm = q[8];
      r.steps.push_back(s);
    }
    r.final_misfit = final_misfit;
    r.n_flux_dofs = K;
    r.n_cell_dofs = N;
    r.n_measurements = M;
    write_result_json(ModelVector(m, m + N), r, path);
  });
}

int orc_geometric_factor(const double a[3], const double* b, const double m[3], const double n[3], int dim, double* k) {
  return guard([&] {
    std::optional<std::array<double, 3>> bb;
    if (b) bb = std::array<double, 3>{b[0], b[1], b[2]};
    *k = geometric_factor({a[0], a[1], a[2]}, bb, {m[0], m[1], m[2]}, {n[0], n[1], n[2]}, dim);
  });
}

int orc_dense_cholesky(uint64_t n, const double* C, double* L) {
  return guard([&] {
    DenseMatrix Cm(n, n);
    std::memcpy(Cm.values.data(), C, n * n * sizeof(double));
    const DenseMatrix Lm = dense_cholesky(Cm);
    std::memcpy(L, Lm.values.data(), n * n * sizeof(double));
  });
}

}  // extern "C"
