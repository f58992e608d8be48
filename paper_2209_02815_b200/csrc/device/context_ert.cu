// context_ert.cu -- ERT response and Jacobian on the device (BASELINE C4/C5):
// evaluate_response_and_jacobian (proj/src/forward.cpp:100-172).
//
// The reference factorises the P1 stiffness with a sparse LU (Eigen) and solves one
// unit pole per used electrode.  Here the stiffness is assembled on the host (values
// depend on m, pattern cached per mesh), an SA-AMG hierarchy of it is built with the
// reference's amg_setup, and ALL pole solves run as one batched PCG on the device
// (columns interleaved, one batched V-cycle per iteration).  The cellwise gradients and
// the J rows / response g are then formed by two device kernels.
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>

#include "context.cuh"
#include "ert_kernels.cuh"

namespace gnw {

namespace {
using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }
}  // namespace

void Context::set_electrodes(const int64_t* nodes, int64_t n) {
  require_mixed();
  electrodes_.assign(nodes, nodes + n);
  double scale = 0.0;
  for (double v : mesh_.vertices) scale = std::max(scale, std::abs(v));
  for (int64_t e : electrodes_) {
    if (e < 0 || e >= mesh_.nv) throw std::invalid_argument("finalize_mesh: electrode index out of range");
    if (std::abs(mesh_.vertices[2 * e + 1]) > 1e-9 * scale)  // forward.cpp:102-112
      throw std::invalid_argument("evaluate_response_and_jacobian: survey electrode is not a mesh node");
  }
  if (fwd_.free_to_node.empty()) fwd_ = host::forward_structure(mesh_);
}

void Context::response_jacobian(const double* mdl, const host::ErtConfig* cfgs, int64_t n_cfg, double* J_out,
                                double* g_out, double tol, ErtTimings* tm) {
  require_mixed();
  require_device();
  if (comm_) throw std::invalid_argument("evaluate_response_and_jacobian: not available on a partitioned context");
  if (electrodes_.empty()) throw std::invalid_argument("evaluate_response_and_jacobian: electrode count mismatch");
  const int64_t ne = static_cast<int64_t>(electrodes_.size());
  const int64_t N = mesh_.nc;
  const cudaStream_t s = stream_;
  ErtTimings t;
  // used electrodes -> batched columns (forward.cpp:115-121)
  std::vector<int> col(ne, -1);
  std::vector<int64_t> used;
  for (int64_t i = 0; i < n_cfg; ++i) {
    const host::ErtConfig& c = cfgs[i];
    const int64_t ids[4] = {c.a, c.m, c.n, c.b};
    for (int k = 0; k < 4; ++k) {
      if (k == 3 && c.b == host::kPoleAtInfinity) continue;
      if (ids[k] < 0 || ids[k] >= ne) throw std::invalid_argument("attach_electrode_positions: electrode index out of range");
      if (col[ids[k]] < 0) col[ids[k]] = 0;
    }
  }
  for (int64_t e = 0; e < ne; ++e)
    if (col[e] >= 0) {
      col[e] = static_cast<int>(used.size());
      used.push_back(e);
    }
  const int b = static_cast<int>(used.size());
  for (int64_t e : used)
    if (fwd_.node_to_free[electrodes_[e]] < 0)  // forward.cpp:86-88
      throw std::invalid_argument("solve_unit_pole: electrode sits on the grounded boundary");
  // model on the host (the stiffness values are host work, bit-exact with assemble_forward)
  std::vector<double> m_host(N);
  if (ptr_mode == 1)
    GNW_CUDA_CHECK(cudaMemcpy(m_host.data(), mdl, N * sizeof(double), cudaMemcpyDeviceToHost));
  else
    std::memcpy(m_host.data(), mdl, N * sizeof(double));

  auto t0 = Clock::now();
  const host::Csr Kst = host::forward_stiffness(fwd_, m_host.data());  // assemble_forward, forward.cpp:58-80
  t.t_assemble = since(t0);

  const int64_t nf = fwd_.n_free;
  const size_t nb = static_cast<size_t>(nf) * b;
  // Mesh-only device structure, uploaded once per mesh: the stiffness pattern (values are
  // re-uploaded per model), cells, free numbering, cell geometry.
  if (!emem_) {
    emem_ = std::make_unique<DeviceMemory>();
    DeviceMemory& em = *emem_;
    ek_ = upload_csr(em, Kst, s);
    ecells_ = em.alloc<int64_t>(3 * N);
    en2f_ = em.alloc<int64_t>(mesh_.nv);
    egrad_ = em.alloc<double>(6 * N);
    earea_ = em.alloc<double>(N);
    GNW_CUDA_CHECK(cudaMemcpyAsync(ecells_, mesh_.cells.data(), 3 * N * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    GNW_CUDA_CHECK(cudaMemcpyAsync(en2f_, fwd_.node_to_free.data(), mesh_.nv * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    GNW_CUDA_CHECK(cudaMemcpyAsync(egrad_, fwd_.grad.data(), 6 * N * sizeof(double), cudaMemcpyHostToDevice, s));
    GNW_CUDA_CHECK(cudaMemcpyAsync(earea_, fwd_.area.data(), N * sizeof(double), cudaMemcpyHostToDevice, s));
  } else {
    GNW_CUDA_CHECK(cudaMemcpyAsync(ek_.vals, Kst.vals.data(), Kst.vals.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  const DCsr dK = ek_;
  // Work buffers, kept while (columns, configurations, pointer mode) stay the same.
  const bool own_out = ptr_mode != 1;
  if (!ews_ || ews_b_ != b || ews_ncfg_ != n_cfg || ews_own_ != own_out) {
    ews_.reset();
    ews_ = std::make_unique<DeviceMemory>();
    DeviceMemory& w = *ews_;
    ew_.X = w.alloc<double>(nb);
    ew_.R = w.alloc<double>(nb);
    ew_.Z = w.alloc<double>(nb);
    ew_.P = w.alloc<double>(nb);
    ew_.AP = w.alloc<double>(nb);
    ew_.sc = w.alloc<double>(8 * static_cast<size_t>(b));
    ew_.active = w.alloc<int>(b);
    ew_.part = w.alloc<double>(2 * static_cast<size_t>(col_dots_chunks(nf)) * b + 16);
    ew_.unit = w.alloc<int64_t>(b);
    ew_.m = w.alloc<double>(N);
    ew_.gx = w.alloc<double>(static_cast<size_t>(b) * N);
    ew_.gz = w.alloc<double>(static_cast<size_t>(b) * N);
    ew_.cfg = w.alloc<ErtCfgDev>(n_cfg);
    ew_.col = w.alloc<int>(ne);
    ew_.gpart = w.alloc<double>(static_cast<size_t>(jacobian_chunks(N)) * n_cfg);
    ew_.J = own_out ? w.alloc<double>(static_cast<size_t>(n_cfg) * N) : nullptr;
    ew_.g = w.alloc<double>(n_cfg);
    ews_b_ = b;
    ews_ncfg_ = n_cfg;
    ews_own_ = own_out;
  }
  double *X = ew_.X, *R = ew_.R, *Z = ew_.Z, *P = ew_.P, *AP = ew_.AP, *part = ew_.part;
  int* active = ew_.active;
  double *rz = ew_.sc, *rz_new = ew_.sc + 2 * b, *pap = ew_.sc + 4 * b, *rr = ew_.sc + 6 * b;
  const double* dm = mdl;  // the model on the device
  if (ptr_mode != 1) {
    GNW_CUDA_CHECK(cudaMemcpyAsync(ew_.m, mdl, N * sizeof(double), cudaMemcpyHostToDevice, s));
    dm = ew_.m;
  }

  t0 = Clock::now();
  // PCG preconditioner only (the reference solves exactly).  Structured unit-square meshes:
  // geometric multigrid built on the device from sigma (ert_gmg.cu).  Otherwise (or with env
  // GNW_ERT_PC=amg) the reference's amg_setup of K on the host with default options; the
  // lumped filtering can leave a non-positive diagonal (the survey's AMG caveat), in which
  // case the unfiltered hierarchy (strength 0, always well defined) is used.
  if (fwd_gmg_n_ < 0) fwd_gmg_n_ = ErtGmg::structured_n(mesh_, fwd_);
  bool use_gmg = fwd_gmg_n_ > 0;
  if (const char* e = std::getenv("GNW_ERT_PC"))
    if (std::string(e) == "amg") use_gmg = false;
  if (use_gmg) {
    fwd_gmg_.build(fwd_gmg_n_, dm, b, dflag_, s);
    int fail = 0;
    GNW_CUDA_CHECK(cudaMemcpyAsync(&fail, dflag_, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync();
    if (fail) throw std::runtime_error("evaluate_response_and_jacobian: coarse grid operator not positive definite");
  } else {
    host::AmgHierarchy hK;
    try {
      hK = host::amg_setup(Kst, host::AmgOptions{});
    } catch (const std::invalid_argument&) {
      host::AmgOptions o;
      o.strength = 0.0;
      hK = host::amg_setup(Kst, o);
    }
    fwd_amg_.upload(hK, s);
  }
  t.t_amg = since(t0);
  t.gmg_levels = use_gmg ? static_cast<uint64_t>(fwd_gmg_.levels()) : 0;
  auto precondition = [&](const double* r, double* z) {
    if (use_gmg)
      fwd_gmg_.vcycle(r, z, s);
    else
      fwd_amg_.vcycle_batch(r, b, z, 0, st_plain_, s);
  };
  {  // right-hand sides: column q is the unit vector of electrode used[q] (solve_unit_pole)
    std::vector<int64_t> unit(b);
    for (int q = 0; q < b; ++q) unit[q] = fwd_.node_to_free[electrodes_[used[q]]];
    GNW_CUDA_CHECK(cudaMemcpyAsync(ew_.unit, unit.data(), b * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    unit_columns(R, ew_.unit, nf, b, s);
    std::vector<int> act(b, 1);
    GNW_CUDA_CHECK(cudaMemcpyAsync(active, act.data(), b * sizeof(int), cudaMemcpyHostToDevice, s));
    GNW_CUDA_CHECK(cudaMemsetAsync(X, 0, nb * sizeof(double), s));
  }
  // batched PCG on K u = e (one column per used electrode; ||e|| = 1)
  cudaEvent_t* ev = jev_;
  for (int k = 0; k < 4; ++k)
    if (!ev[k]) GNW_CUDA_CHECK(cudaEventCreate(&ev[k]));
  GNW_CUDA_CHECK(cudaEventRecord(ev[0], s));
  precondition(R, Z);
  GNW_CUDA_CHECK(cudaMemcpyAsync(P, Z, nb * sizeof(double), cudaMemcpyDeviceToDevice, s));
  col_dots(R, Z, nf, b, part, counters_ + 8, rz, 0, s);
  std::vector<double> rrh(b);
  std::vector<int> act(b, 1);
  const int maxit = 2000;
  int it = 0;
  for (; it < maxit; ++it) {
    spmm(dK, P, AP, b, s);
    col_dots(P, AP, nf, b, part, counters_ + 8, pap, 0, s);
    pcg_xr(X, R, P, AP, rz, pap, active, nf, b, s);
    col_dots(R, R, nf, b, part, counters_ + 8, rr, 0, s);
    GNW_CUDA_CHECK(cudaMemcpyAsync(rrh.data(), rr, b * sizeof(double), cudaMemcpyDeviceToHost, s));
    sync();
    bool any = false;
    for (int q = 0; q < b; ++q) {
      if (!std::isfinite(rrh[q])) throw std::runtime_error("evaluate_response_and_jacobian: non-finite response");
      if (act[q] && std::sqrt(rrh[q]) <= tol) act[q] = 0;
      any |= act[q] != 0;
    }
    if (!any) {
      ++it;
      break;
    }
    GNW_CUDA_CHECK(cudaMemcpyAsync(active, act.data(), b * sizeof(int), cudaMemcpyHostToDevice, s));
    precondition(R, Z);
    col_dots(R, Z, nf, b, part, counters_ + 8, rz_new, 0, s);
    pcg_p(P, Z, rz_new, rz, active, nf, b, s);
    std::swap(rz, rz_new);
  }
  t.pcg_iterations = it;
  GNW_CUDA_CHECK(cudaEventRecord(ev[1], s));
  // cellwise gradients and J / g
  std::vector<ErtCfgDev> hc(n_cfg);
  for (int64_t i = 0; i < n_cfg; ++i)
    hc[i] = {static_cast<int>(cfgs[i].a), static_cast<int>(cfgs[i].b), static_cast<int>(cfgs[i].m),
             static_cast<int>(cfgs[i].n), cfgs[i].k};
  GNW_CUDA_CHECK(cudaMemcpyAsync(ew_.cfg, hc.data(), n_cfg * sizeof(ErtCfgDev), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(ew_.col, col.data(), ne * sizeof(int), cudaMemcpyHostToDevice, s));
  double* dJ = ptr_mode == 1 ? J_out : ew_.J;
  double* dg = ptr_mode == 1 ? g_out : ew_.g;
  GNW_CUDA_CHECK(cudaEventRecord(ev[2], s));
  cell_grad(ecells_, en2f_, egrad_, X, b, N, ew_.gx, ew_.gz, s);
  jacobian(ew_.cfg, static_cast<int>(n_cfg), ew_.col, ew_.gx, ew_.gz, dm, earea_, N, dJ, N, ew_.gpart, dg, s);
  GNW_CUDA_CHECK(cudaEventRecord(ev[3], s));
  if (ptr_mode != 1) {
    GNW_CUDA_CHECK(cudaMemcpyAsync(J_out, dJ, static_cast<size_t>(n_cfg) * N * sizeof(double), cudaMemcpyDeviceToHost, s));
    GNW_CUDA_CHECK(cudaMemcpyAsync(g_out, dg, n_cfg * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  std::vector<double> gh(n_cfg);
  GNW_CUDA_CHECK(cudaMemcpyAsync(gh.data(), dg, n_cfg * sizeof(double), cudaMemcpyDeviceToHost, s));
  sync();
  for (double v : gh)
    if (!std::isfinite(v)) throw std::runtime_error("evaluate_response_and_jacobian: non-finite response");
  float ms = 0.f;
  GNW_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
  t.t_solve = ms * 1e-3;
  GNW_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[2], ev[3]));
  t.t_jacobian = ms * 1e-3;
  if (tm) *tm = t;
}

}  // namespace gnw
