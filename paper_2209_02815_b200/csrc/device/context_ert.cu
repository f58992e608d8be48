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
  // model on the host (stiffness values and AMG setup are host work)
  std::vector<double> m_host(N);
  if (ptr_mode == 1)
    GNW_CUDA_CHECK(cudaMemcpy(m_host.data(), mdl, N * sizeof(double), cudaMemcpyDeviceToHost));
  else
    std::memcpy(m_host.data(), mdl, N * sizeof(double));

  auto t0 = Clock::now();
  const host::Csr Kst = host::forward_stiffness(fwd_, m_host.data());  // assemble_forward, forward.cpp:58-80
  t.t_assemble = since(t0);
  t0 = Clock::now();
  // PCG preconditioner only (the reference solves exactly): default SA-AMG options; the
  // lumped filtering can leave a non-positive diagonal (the survey's AMG caveat), in
  // which case the unfiltered hierarchy (strength 0, always well defined) is used.
  host::AmgHierarchy hK;
  try {
    hK = host::amg_setup(Kst, host::AmgOptions{});
  } catch (const std::invalid_argument&) {
    host::AmgOptions o;
    o.strength = 0.0;
    hK = host::amg_setup(Kst, o);
  }
  fwd_amg_.upload(hK, s);
  t.t_amg = since(t0);

  emem_ = std::make_unique<DeviceMemory>();
  DeviceMemory& em = *emem_;
  const int64_t nf = fwd_.n_free;
  const size_t nb = static_cast<size_t>(nf) * b;
  const DCsr dK = upload_csr(em, Kst, s);
  double* X = em.alloc<double>(nb);
  double* R = em.alloc<double>(nb);
  double* Z = em.alloc<double>(nb);
  double* P = em.alloc<double>(nb);
  double* AP = em.alloc<double>(nb);
  double* sc = em.alloc<double>(8 * static_cast<size_t>(b));  // rz, rz_new, pap, rr (+ xx slots)
  int* active = em.alloc<int>(b);
  double* part = em.alloc<double>(2 * static_cast<size_t>(col_dots_chunks(nf)) * b + 16);
  double *rz = sc, *rz_new = sc + 2 * b, *pap = sc + 4 * b, *rr = sc + 6 * b;
  {
    std::vector<double> Rh(nb, 0.0);
    for (int q = 0; q < b; ++q) Rh[static_cast<size_t>(fwd_.node_to_free[electrodes_[used[q]]]) * b + q] = 1.0;
    GNW_CUDA_CHECK(cudaMemcpyAsync(R, Rh.data(), nb * sizeof(double), cudaMemcpyHostToDevice, s));
    std::vector<int> act(b, 1);
    GNW_CUDA_CHECK(cudaMemcpyAsync(active, act.data(), b * sizeof(int), cudaMemcpyHostToDevice, s));
    GNW_CUDA_CHECK(cudaMemsetAsync(X, 0, nb * sizeof(double), s));
    sync();
  }
  // batched PCG on K u = e (one column per used electrode; ||e|| = 1)
  cudaEvent_t* ev = jev_;
  for (int k = 0; k < 4; ++k)
    if (!ev[k]) GNW_CUDA_CHECK(cudaEventCreate(&ev[k]));
  GNW_CUDA_CHECK(cudaEventRecord(ev[0], s));
  fwd_amg_.vcycle_batch(R, b, Z, 0, st_plain_, s);
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
    fwd_amg_.vcycle_batch(R, b, Z, 0, st_plain_, s);
    col_dots(R, Z, nf, b, part, counters_ + 8, rz_new, 0, s);
    pcg_p(P, Z, rz_new, rz, active, nf, b, s);
    std::swap(rz, rz_new);
  }
  t.pcg_iterations = it;
  GNW_CUDA_CHECK(cudaEventRecord(ev[1], s));
  // cellwise gradients and J / g
  int64_t* dcells = em.alloc<int64_t>(3 * N);
  int64_t* dn2f = em.alloc<int64_t>(mesh_.nv);
  double* dgrad = em.alloc<double>(6 * N);
  double* darea = em.alloc<double>(N);
  double* gx = em.alloc<double>(static_cast<size_t>(b) * N);
  double* gz = em.alloc<double>(static_cast<size_t>(b) * N);
  GNW_CUDA_CHECK(cudaMemcpyAsync(dcells, mesh_.cells.data(), 3 * N * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dn2f, fwd_.node_to_free.data(), mesh_.nv * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dgrad, fwd_.grad.data(), 6 * N * sizeof(double), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(darea, fwd_.area.data(), N * sizeof(double), cudaMemcpyHostToDevice, s));
  std::vector<ErtCfgDev> hc(n_cfg);
  for (int64_t i = 0; i < n_cfg; ++i)
    hc[i] = {static_cast<int>(cfgs[i].a), static_cast<int>(cfgs[i].b), static_cast<int>(cfgs[i].m),
             static_cast<int>(cfgs[i].n), cfgs[i].k};
  ErtCfgDev* dcfg = em.alloc<ErtCfgDev>(n_cfg);
  int* dcol = em.alloc<int>(ne);
  GNW_CUDA_CHECK(cudaMemcpyAsync(dcfg, hc.data(), n_cfg * sizeof(ErtCfgDev), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dcol, col.data(), ne * sizeof(int), cudaMemcpyHostToDevice, s));
  const double* dm = mdl;
  if (ptr_mode != 1) {
    double* tmpm = em.alloc<double>(N);
    GNW_CUDA_CHECK(cudaMemcpyAsync(tmpm, mdl, N * sizeof(double), cudaMemcpyHostToDevice, s));
    dm = tmpm;
  }
  double* dJ = ptr_mode == 1 ? J_out : em.alloc<double>(static_cast<size_t>(n_cfg) * N);
  double* dg = ptr_mode == 1 ? g_out : em.alloc<double>(n_cfg);
  double* gpart = em.alloc<double>(static_cast<size_t>(jacobian_chunks(N)) * n_cfg);
  GNW_CUDA_CHECK(cudaEventRecord(ev[2], s));
  cell_grad(dcells, dn2f, dgrad, X, b, N, gx, gz, s);
  jacobian(dcfg, static_cast<int>(n_cfg), dcol, gx, gz, dm, darea, N, dJ, N, gpart, dg, s);
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
