// gnw_capi.cu -- extern "C" boundary (include/gnw.h) over gnw::Context.
// Exceptions map to status codes exactly as SURVEY.md 8(b) specifies:
// std::invalid_argument -> GNW_INVALID_ARGUMENT, gnw::DeviceError -> GNW_DEVICE,
// any other std::exception -> GNW_NUMERICAL; the message text is the
// reference's exception text.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../../include/gnw.h"
#include "context.cuh"

using gnw::Context;

struct gnw_ctx {
  Context* c = nullptr;
  std::vector<double> hist_e, hist_p;  // residual histories of the last gnw_minres_solve
};

namespace {
thread_local std::string g_err;

// A failed collective call on an in-process partitioned rank releases the other ranks'
// barriers (they fail too) instead of leaving them waiting.
void abandon(gnw_ctx* c) {
  if (c && c->c && c->c->partitioned() && std::string(c->c->comm()->kind()) == "local")
    static_cast<gnw::LocalComm*>(const_cast<gnw::Comm*>(c->c->comm()))->hub().abandon();
}

template <class F>
gnw_status guard(F&& f, gnw_ctx* c = nullptr) {
  try {
    f();
    return GNW_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    abandon(c);
    return GNW_INVALID_ARGUMENT;
  } catch (const gnw::DeviceError& e) {
    g_err = e.what();
    abandon(c);
    return GNW_DEVICE;
  } catch (const std::exception& e) {
    g_err = e.what();
    abandon(c);
    return GNW_NUMERICAL;
  }
}

gnw::host::AmgOptions to_opts(const gnw_amg_options* o) {
  gnw::host::AmgOptions a;
  if (o) {
    a.coarse_threshold = static_cast<int64_t>(o->coarse_threshold);
    a.strength = o->strength;
    a.jacobi_damping = o->jacobi_damping;
    a.prolongation_damping = o->prolongation_damping;
    a.max_aggregate_size = static_cast<int64_t>(o->max_aggregate_size);
    a.max_levels = static_cast<int64_t>(o->max_levels);
  }
  return a;
}

Context& ctx_of(gnw_ctx* c) {
  if (!c || !c->c) throw std::invalid_argument("gnw: null context");
  return *c->c;
}
const Context& ctx_of(const gnw_ctx* c) {
  if (!c || !c->c) throw std::invalid_argument("gnw: null context");
  return *c->c;
}
}  // namespace

extern "C" {

const char* gnw_last_error(void) { return g_err.c_str(); }
const char* gnw_version(void) { return "gnw-b200 0.1 (sm_100a, FP64)"; }

gnw_status gnw_create(int n_devices, const int* devices, gnw_ctx** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("gnw_create: null output");
    *out = nullptr;
    if (n_devices > 1) throw std::invalid_argument("gnw_create: one device per context (one process per GPU)");
    const int dev = n_devices == 0 ? -1 : (devices ? devices[0] : 0);
    auto* h = new gnw_ctx;
    try {
      h->c = new Context(dev);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void gnw_destroy(gnw_ctx* ctx) {
  if (!ctx) return;
  delete ctx->c;
  delete ctx;
}

gnw_status gnw_set_pointer_mode(gnw_ctx* ctx, int mode) {
  return guard([&] {
    if (mode != GNW_HOST_POINTERS && mode != GNW_DEVICE_POINTERS) throw std::invalid_argument("gnw_set_pointer_mode: bad mode");
    ctx_of(ctx).ptr_mode = mode;
  });
}

gnw_status gnw_set_coarse_mode(gnw_ctx* ctx, int mode) {
  return guard([&] {
    if (mode != GNW_COARSE_INVERSE && mode != GNW_COARSE_CHOLESKY) throw std::invalid_argument("gnw_set_coarse_mode: bad mode");
    ctx_of(ctx).set_coarse(mode);
  });
}

gnw_status gnw_set_preconditioner(gnw_ctx* ctx, int kind) {
  return guard([&] {
    if (kind != GNW_PC_WOODBURY && kind != GNW_PC_LAPLACE) throw std::invalid_argument("gnw_set_preconditioner: bad kind");
    ctx_of(ctx).pc_laplace = kind;
  });
}

gnw_status gnw_set_loop_mode(gnw_ctx* ctx, int mode) {
  return guard([&] {
    if (mode != GNW_LOOP_REFERENCE && mode != GNW_LOOP_FUSED && mode != GNW_LOOP_AUTO &&
        mode != GNW_LOOP_LEAN && mode != GNW_LOOP_PERSISTENT)
      throw std::invalid_argument("gnw_set_loop_mode: bad mode");
    ctx_of(ctx).set_fused(mode);
  });
}

gnw_status gnw_assemble(gnw_ctx* ctx, const gnw_mesh* mesh, const gnw_amg_options* opts) {
  return guard([&] {
    if (!mesh || !mesh->vertices || !mesh->cells) throw std::invalid_argument("gnw_assemble: null mesh");
    ctx_of(ctx).assemble(mesh->vertices, static_cast<int64_t>(mesh->n_vertices), mesh->cells,
                         static_cast<int64_t>(mesh->n_cells), to_opts(opts));
  }, ctx);
}

gnw_status gnw_assemble_amg_csr(gnw_ctx* ctx, uint64_t n, const int64_t* rowptr, const int64_t* cols,
                                const double* vals, const gnw_amg_options* opts) {
  return guard([&] {
    ctx_of(ctx).assemble_amg_csr(static_cast<int64_t>(n), rowptr, cols, vals, to_opts(opts));
  });
}

gnw_status gnw_assemble_saddle_csr(gnw_ctx* ctx, const gnw_csr* Q, const gnw_csr* D, const gnw_amg_options* opts) {
  return guard([&] {
    if (!Q || !D) throw std::invalid_argument("gnw_assemble_saddle_csr: null matrix");
    if (Q->n_rows != Q->n_cols || D->n_cols != Q->n_rows) throw std::invalid_argument("gnw_assemble_saddle_csr: shape mismatch");
    const gnw::host::AmgOptions o = to_opts(opts);
    ctx_of(ctx).assemble_saddle_csr(static_cast<int64_t>(Q->n_rows), static_cast<int64_t>(D->n_rows), Q->rowptr, Q->cols,
                                    Q->vals, D->rowptr, D->cols, D->vals, opts ? &o : nullptr);
  });
}

gnw_status gnw_set_amg_hierarchy(gnw_ctx* ctx, uint64_t n_levels, const gnw_csr* A, const gnw_csr* P,
                                 const double* const* inv_diag, const double* coarse_chol, uint64_t nc,
                                 const gnw_amg_options* opts) {
  return guard([&] {
    if (n_levels == 0 || !A || !P || !inv_diag || !coarse_chol) throw std::invalid_argument("gnw_set_amg_hierarchy: null argument");
    auto csr = [](const gnw_csr& m) {
      gnw::host::Csr c;
      c.n_rows = static_cast<int64_t>(m.n_rows);
      c.n_cols = static_cast<int64_t>(m.n_cols);
      c.rowptr.assign(m.rowptr, m.rowptr + m.n_rows + 1);
      const int64_t nnz = m.n_rows ? m.rowptr[m.n_rows] : 0;
      c.cols.resize(static_cast<size_t>(nnz));
      for (int64_t k = 0; k < nnz; ++k) c.cols[static_cast<size_t>(k)] = static_cast<int32_t>(m.cols[k]);
      c.vals.assign(m.vals, m.vals + nnz);
      return c;
    };
    gnw::host::AmgHierarchy h;
    h.options = to_opts(opts);
    for (uint64_t l = 0; l < n_levels; ++l) {
      gnw::host::AmgLevel lv;
      lv.A = csr(A[l]);
      if (l + 1 < n_levels) lv.P = csr(P[l]);
      lv.inv_diag.assign(inv_diag[l], inv_diag[l] + A[l].n_rows);
      h.levels.push_back(std::move(lv));
    }
    h.nc = static_cast<int64_t>(nc);
    h.coarse_chol.assign(coarse_chol, coarse_chol + nc * nc);
    ctx_of(ctx).set_hierarchy(h);
  });
}

gnw_status gnw_set_flux_scaling(gnw_ctx* ctx, const double* q_diag_inv) {
  return guard([&] {
    if (!q_diag_inv) throw std::invalid_argument("gnw_set_flux_scaling: null argument");
    ctx_of(ctx).set_qinv(q_diag_inv);
  });
}

gnw_status gnw_get_info(const gnw_ctx* ctx, gnw_info* info) {
  return guard([&] {
    const Context& c = ctx_of(ctx);
    std::memset(info, 0, sizeof *info);
    info->K = c.K();
    info->N = c.N();
    info->n_vertices = c.mesh().nv;
    info->n_edges = c.mesh().ne;
    info->n_boundary_edges = c.mesh().boundary_edges.size();
    info->n_levels = c.amg().levels.size();
    info->coarse_n = c.amg().nc;
    info->m = c.m();
    info->beta = c.beta();
    info->device_bytes = c.device_bytes();
    info->collapse_level = c.has_device() ? c.vc_collapse_level() : -1;
  });
}

gnw_status gnw_prefetch_jacobian(gnw_ctx* ctx, const double* J, uint64_t m, uint64_t n_cells) {
  return guard([&] { ctx_of(ctx).prefetch_jacobian(J, static_cast<int64_t>(m), static_cast<int64_t>(n_cells)); });
}

gnw_status gnw_set_jacobian(gnw_ctx* ctx, const double* J, uint64_t m, uint64_t n_cells, double beta,
                            gnw_timings* timings) {
  return guard([&] {
    double t[3] = {0, 0, 0};
    ctx_of(ctx).set_jacobian(J, static_cast<int64_t>(m), static_cast<int64_t>(n_cells), beta, t);
    if (timings) {
      timings->t_H = t[0];
      timings->t_C = t[1];
      timings->t_chol = t[2];
    }
  }, ctx);
}

gnw_status gnw_apply_operator(gnw_ctx* ctx, const double* x, double* y) {
  return guard([&] { ctx_of(ctx).apply_operator(x, y); }, ctx);
}
gnw_status gnw_precondition(gnw_ctx* ctx, const double* y, double* z) {
  return guard([&] { ctx_of(ctx).precondition(y, z); }, ctx);
}
gnw_status gnw_amg_apply(gnw_ctx* ctx, const double* r, double* z) {
  return guard([&] { ctx_of(ctx).amg_apply(r, z); });
}
gnw_status gnw_get_woodbury(gnw_ctx* ctx, double* H, double* L) {
  return guard([&] { ctx_of(ctx).get_woodbury(H, L); });
}
gnw_status gnw_assemble_rhs(gnw_ctx* ctx, const double* m, const double* m_ref, const double* g, const double* g_obs,
                            double* rhs) {
  return guard([&] { ctx_of(ctx).assemble_rhs(m, m_ref, g, g_obs, rhs); }, ctx);
}

gnw_status gnw_minres_solve(gnw_ctx* ctx, const double* b, const double* x0, double* x, double tol, uint64_t maxit,
                            gnw_report* report) {
  return guard([&] {
    gnw::MinresResult r = ctx_of(ctx).minres(b, x0, x, tol, maxit);
    ctx->hist_e = r.hist_e;
    ctx->hist_p = r.hist_p;
    if (report) {
      report->iterations = r.iterations;
      report->converged = r.converged ? 1 : 0;
      report->true_relative_residual = r.true_rel;
      report->n_hist = r.hist_e.size();
      const uint64_t h = std::min<uint64_t>(report->hist_cap, r.hist_e.size());
      for (uint64_t k = 0; k < h; ++k) {
        if (report->relative_residuals) report->relative_residuals[k] = r.hist_e[k];
        if (report->pnorm_relative_residuals) report->pnorm_relative_residuals[k] = r.hist_p[k];
      }
    }
  }, ctx);
}

gnw_status gnw_gn_step_solve(gnw_ctx* ctx, const double* m, const double* m_ref, const double* g, const double* g_obs,
                             double* x, double tol, uint64_t maxit, gnw_report* report) {
  return guard([&] {
    gnw::MinresResult r = ctx_of(ctx).gn_step_solve(m, m_ref, g, g_obs, x, tol, maxit);
    ctx->hist_e = r.hist_e;
    ctx->hist_p = r.hist_p;
    if (report) {
      report->iterations = r.iterations;
      report->converged = r.converged ? 1 : 0;
      report->true_relative_residual = r.true_rel;
      report->n_hist = r.hist_e.size();
      const uint64_t h = std::min<uint64_t>(report->hist_cap, r.hist_e.size());
      for (uint64_t k = 0; k < h; ++k) {
        if (report->relative_residuals) report->relative_residuals[k] = r.hist_e[k];
        if (report->pnorm_relative_residuals) report->pnorm_relative_residuals[k] = r.hist_p[k];
      }
    }
  }, ctx);
}

gnw_status gnw_minres_history(const gnw_ctx* ctx, double* relative_residuals, double* pnorm_relative_residuals,
                              uint64_t cap, uint64_t* n_hist) {
  return guard([&] {
    ctx_of(ctx);
    const uint64_t n = ctx->hist_e.size();
    if (n_hist) *n_hist = n;
    const uint64_t h = std::min<uint64_t>(cap, n);
    if (relative_residuals && h) std::memcpy(relative_residuals, ctx->hist_e.data(), h * sizeof(double));
    if (pnorm_relative_residuals && h) std::memcpy(pnorm_relative_residuals, ctx->hist_p.data(), h * sizeof(double));
  });
}

// ------------------------------------------------------- partitioned contexts
gnw_status gnw_nccl_unique_id(unsigned char id[128]) {
  return guard([&] {
    if (!id) throw std::invalid_argument("gnw_nccl_unique_id: null output");
    gnw::nccl_unique_id(id);
  });
}

gnw_status gnw_create_partitioned(int device, int rank, int world, const unsigned char id[128], gnw_ctx** out) {
  return guard([&] {
    if (!out || !id) throw std::invalid_argument("gnw_create_partitioned: null argument");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("gnw_create_partitioned: bad rank/world");
    auto* h = new gnw_ctx;
    try {
      h->c = new Context(device);
      h->c->set_comm(std::make_shared<gnw::NcclComm>(id, rank, world, device));
    } catch (...) {
      delete h->c;
      delete h;
      throw;
    }
    *out = h;
  });
}

gnw_status gnw_create_local_group(int device, int world, gnw_ctx** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("gnw_create_local_group: null output");
    if (world < 1) throw std::invalid_argument("gnw_create_local_group: world size must be >= 1");
    auto hub = std::make_shared<gnw::LocalHub>(world);
    std::vector<gnw_ctx*> made;
    try {
      for (int r = 0; r < world; ++r) {
        auto* h = new gnw_ctx;
        made.push_back(h);
        h->c = new Context(device);
        h->c->set_comm(std::make_shared<gnw::LocalComm>(hub, r));
      }
    } catch (...) {
      for (gnw_ctx* h : made) {
        delete h->c;
        delete h;
      }
      throw;
    }
    for (int r = 0; r < world; ++r) out[r] = made[r];
  });
}

gnw_status gnw_partition_cells(uint64_t n_cells, int world, int64_t* lo) {
  return guard([&] {
    if (!lo) throw std::invalid_argument("gnw_partition_cells: null output");
    const std::vector<long long> p = gnw::partition_cells(static_cast<long long>(n_cells), world);
    for (size_t r = 0; r < p.size(); ++r) lo[r] = p[r];
  });
}

gnw_status gnw_partition_saddle(const gnw_ctx* ctx, int world, int rank, uint64_t sizes[4], int64_t* local_to_global,
                                int64_t* recv_off, int64_t* send_off, int32_t* send_idx) {
  return guard([&] {
    const Context& c = ctx_of(ctx);
    if (!c.mixed() || !c.assembled()) throw std::invalid_argument("gnw_partition_saddle: not assembled");
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("gnw_partition_saddle: bad rank/world");
    const std::vector<long long> lo = gnw::partition_cells(c.N(), world);
    const gnw::host::SaddlePartition sp = gnw::host::partition_saddle(c.mesh(), c.Q(), c.D(), lo, rank);
    const gnw::host::Halo& h = sp.halo;
    if (sizes) {
      sizes[0] = sp.K_l;
      sizes[1] = sp.N_l;
      sizes[2] = h.ghost_global.size();
      sizes[3] = h.send_idx.size();
    }
    if (local_to_global) {
      std::copy(h.own_global.begin(), h.own_global.end(), local_to_global);
      std::copy(h.ghost_global.begin(), h.ghost_global.end(), local_to_global + h.n_own);
    }
    if (recv_off) std::copy(h.recv_off.begin(), h.recv_off.end(), recv_off);
    if (send_off) std::copy(h.send_off.begin(), h.send_off.end(), send_off);
    if (send_idx) std::copy(h.send_idx.begin(), h.send_idx.end(), send_idx);
  });
}

gnw_status gnw_partition_csr(const gnw_ctx* ctx, int world, int rank, int which, uint64_t* n_rows, uint64_t* nnz,
                             int64_t* rowptr, int32_t* cols, double* vals) {
  return guard([&] {
    const Context& c = ctx_of(ctx);
    if (!c.mixed() || !c.assembled()) throw std::invalid_argument("gnw_partition_csr: not assembled");
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("gnw_partition_csr: bad rank/world");
    const std::vector<long long> lo = gnw::partition_cells(c.N(), world);
    const gnw::host::SaddlePartition sp = gnw::host::partition_saddle(c.mesh(), c.Q(), c.D(), lo, rank);
    const gnw::host::Csr* A = which == 0 ? &sp.Q : which == 1 ? &sp.D : which == 2 ? &sp.Dt : nullptr;
    if (!A) throw std::invalid_argument("gnw_partition_csr: which must be 0 (Q), 1 (D) or 2 (D^T)");
    if (n_rows) *n_rows = A->n_rows;
    if (nnz) *nnz = A->nnz();
    if (rowptr) std::copy(A->rowptr.begin(), A->rowptr.end(), rowptr);
    if (cols) std::copy(A->cols.begin(), A->cols.end(), cols);
    if (vals) std::copy(A->vals.begin(), A->vals.end(), vals);
  });
}

gnw_status gnw_get_partition(const gnw_ctx* ctx, int* rank, int* world, int64_t* c_lo, int64_t* c_hi) {
  return guard([&] {
    const Context& c = ctx_of(ctx);
    if (rank) *rank = c.partitioned() ? c.comm()->rank : 0;
    if (world) *world = c.partitioned() ? c.comm()->world : 1;
    if (c_lo) *c_lo = c.partitioned() ? c.c_lo() : 0;
    if (c_hi) *c_hi = c.partitioned() ? c.c_hi() : c.N();
  });
}

gnw_status gnw_export_csr(const gnw_ctx* ctx, int which, uint64_t level, uint64_t* n_rows, uint64_t* n_cols,
                          uint64_t* nnz, int64_t* rowptr, int64_t* cols, double* vals) {
  return guard([&] {
    const Context& c = ctx_of(ctx);
    if (!c.assembled()) throw std::invalid_argument("gnw_export_csr: context not assembled");
    const gnw::host::Csr* A = nullptr;
    static const gnw::host::Csr empty{};
    switch (which) {
      case 0: A = &c.Q(); break;
      case 1: A = &c.D(); break;
      case 2: A = &c.S(); break;
      case 3:
      case 4:
        if (level >= c.amg().levels.size()) throw std::invalid_argument("gnw_export_csr: level out of range");
        A = which == 3 ? &c.amg().levels[level].A : &c.amg().levels[level].P;
        break;
      default: throw std::invalid_argument("gnw_export_csr: bad selector");
    }
    if (n_rows) *n_rows = A->n_rows;
    if (n_cols) *n_cols = A->n_cols;
    if (nnz) *nnz = A->nnz();
    if (rowptr) {
      if (A->rowptr.empty())
        rowptr[0] = 0;
      else
        std::memcpy(rowptr, A->rowptr.data(), A->rowptr.size() * sizeof(int64_t));
    }
    if (cols)
      for (int64_t k = 0; k < A->nnz(); ++k) cols[k] = A->cols[k];
    if (vals && A->nnz()) std::memcpy(vals, A->vals.data(), A->vals.size() * sizeof(double));
  });
}

gnw_status gnw_export_mesh(const gnw_ctx* ctx, int64_t* cells, int64_t* edges, int64_t* cell_edges,
                           int32_t* cell_edge_signs, int64_t* boundary_edges, int32_t* boundary_tags) {
  return guard([&] {
    const Context& c = ctx_of(ctx);
    if (!c.mixed()) throw std::invalid_argument("gnw_export_mesh: not a mixed problem");
    const auto& m = c.mesh();
    if (cells) std::memcpy(cells, m.cells.data(), m.cells.size() * sizeof(int64_t));
    if (edges) std::memcpy(edges, m.edges.data(), m.edges.size() * sizeof(int64_t));
    if (cell_edges) std::memcpy(cell_edges, m.cell_edges.data(), m.cell_edges.size() * sizeof(int64_t));
    if (cell_edge_signs) std::memcpy(cell_edge_signs, m.cell_signs.data(), m.cell_signs.size() * sizeof(int32_t));
    if (boundary_edges)
      std::memcpy(boundary_edges, m.boundary_edges.data(), m.boundary_edges.size() * sizeof(int64_t));
    if (boundary_tags) std::memcpy(boundary_tags, m.boundary_tags.data(), m.boundary_tags.size() * sizeof(int32_t));
  });
}

gnw_status gnw_dense_cholesky(gnw_ctx* ctx, uint64_t n, const double* C, double* L) {
  return guard([&] { ctx_of(ctx).dense_cholesky(static_cast<int64_t>(n), C, L); });
}

gnw_status gnw_set_electrodes(gnw_ctx* ctx, const int64_t* nodes, uint64_t n) {
  return guard([&] { ctx_of(ctx).set_electrodes(nodes, static_cast<int64_t>(n)); });
}

gnw_status gnw_response_jacobian(gnw_ctx* ctx, const double* m, const gnw_ert_config* cfgs, uint64_t n_cfg, double* J,
                                 double* g, double tol, gnw_ert_stats* stats) {
  return guard([&] {
    std::vector<gnw::host::ErtConfig> c(n_cfg);
    for (uint64_t i = 0; i < n_cfg; ++i) c[i] = {cfgs[i].a, cfgs[i].b, cfgs[i].m, cfgs[i].n, cfgs[i].k};
    gnw::ErtTimings t;
    ctx_of(ctx).response_jacobian(m, c.data(), static_cast<int64_t>(n_cfg), J, g, tol, &t);
    if (stats) *stats = {t.t_assemble, t.t_amg, t.t_solve, t.t_jacobian, t.pcg_iterations, t.gmg_levels};
  });
}

gnw_status gnw_gauss_newton(gnw_ctx* ctx, const double* m0, const double* m_ref, const gnw_ert_config* cfgs,
                            uint64_t n_cfg, const double* g_obs, const gnw_gn_config* config, double* m_out,
                            gnw_gn_step* steps, uint64_t steps_cap, uint64_t* n_steps, double* final_misfit) {
  return guard([&] {
    if (!config || !m0 || !m_ref || !cfgs || !g_obs) throw std::invalid_argument("gauss_newton: null argument");
    if (config->algorithm != GNW_PC_WOODBURY && config->algorithm != GNW_PC_LAPLACE)
      throw std::invalid_argument("gauss_newton: only the iterative algorithms (Woodbury / Laplace MINRES)");
    gnw::GnConfig c;
    c.beta = config->beta;
    c.max_outer_steps = config->max_outer_steps;
    c.minres_tol = config->minres_tol;
    c.minres_maxit = config->minres_maxit;
    c.laplace = config->algorithm == GNW_PC_LAPLACE;
    c.misfit_reduction_tol = config->misfit_reduction_tol;
    if (config->forward_tol > 0.0) c.forward_tol = config->forward_tol;
    std::vector<gnw::host::ErtConfig> e(n_cfg);
    for (uint64_t i = 0; i < n_cfg; ++i) e[i] = {cfgs[i].a, cfgs[i].b, cfgs[i].m, cfgs[i].n, cfgs[i].k};
    const gnw::GnResult r =
        ctx_of(ctx).gauss_newton(m0, m_ref, e.data(), static_cast<int64_t>(n_cfg), g_obs, c, m_out);
    if (n_steps) *n_steps = r.steps.size();
    if (final_misfit) *final_misfit = r.final_misfit;
    for (uint64_t k = 0; steps && k < std::min<uint64_t>(steps_cap, r.steps.size()); ++k) {
      const gnw::GnStepReport& q = r.steps[k];
      steps[k] = {q.misfit, q.minres_iters, q.converged ? 1 : 0, q.euclid_relative_residual,
                  q.pnorm_relative_residual, q.t_H, q.t_C, q.t_chol, q.t_norm, q.t_forward};
    }
  });
}

gnw_status gnw_geometric_factor(const double a[3], const double* b, const double m[3], const double n[3], int dim,
                                double* k) {
  return guard([&] { *k = gnw::host::geometric_factor(a, b, m, n, dim); });
}

gnw_status gnw_event_record(gnw_ctx* ctx, int slot) {
  return guard([&] { ctx_of(ctx).event_record(slot); });
}

gnw_status gnw_event_elapsed(gnw_ctx* ctx, int a, int b, double* seconds) {
  return guard([&] { *seconds = ctx_of(ctx).event_elapsed(a, b); });
}

gnw_status gnw_profile_kernel(gnw_ctx* ctx, int kernel, int reps, double* seconds, double* algorithmic) {
  return guard([&] { ctx_of(ctx).profile_kernel(kernel, reps, seconds, algorithmic); });
}

gnw_status gnw_get_stats(const gnw_ctx* ctx, gnw_stats* stats) {
  return guard([&] {
    const Context& c = ctx_of(ctx);
    stats->t_minres = c.t_minres;
    stats->t_rhs = c.t_rhs;
    stats->kernel_launches = c.launches;
    stats->setup_kernel_launches = c.setup_launches;
    stats->loop_restarts = c.loop_restarts;
    stats->fused_iterations = c.last_fused_iters_;
    stats->lean_iterations = c.last_sched_iters_[2];
    stats->persistent_iterations = c.last_persist_iters_;
    stats->comm_calls = c.comm_calls();
    stats->comm_bytes = c.comm_bytes();
  });
}

}  // extern "C"
