// context.cu -- device-resident Woodbury-MINRES GN-step solver (host driver).
//
// One context = one GPU, one stream.  The MINRES loop runs as ONE CUDA graph
// with a conditional WHILE node whose body is one iteration (7 + 4 x levels
// kernels); the loop predicate is set on the device by the update kernel, so
// the host does not synchronise per iteration.  It only wakes up when the
// recurred residual crosses tol (the reference's true-residual verification,
// minres.cpp:108-120), on exhaustion, on maxit or on a numerical error.
#include "context.cuh"
#include "sparse_device.cuh"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <limits>
#include <cstdlib>
#include <cstring>

namespace gnw {

uint64_t launch_count();

namespace {

template <class T>
void h2d(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) GNW_CUDA_CHECK(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

VSel ring3(double* const* p, int off) { return vring(p, 3, off); }
VSel ring2(double* const* p, int off) { return vring(p, 2, off); }

}  // namespace

Context::Context(int device) : device_(device) {
  if (device_ < 0) return;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw DeviceError("gnw: no CUDA device available (the product has no CPU fallback)");
  if (device_ >= n) throw std::invalid_argument("gnw_create: device index out of range");
  GNW_CUDA_CHECK(cudaSetDevice(device_));
  cudaDeviceProp prop;
  GNW_CUDA_CHECK(cudaGetDeviceProperties(&prop, device_));
  if (prop.major < 10) throw DeviceError("gnw: this build targets sm_100a (B200); found sm_" + std::to_string(prop.major) + std::to_string(prop.minor));
  sm_count_ = prop.multiProcessorCount;
  if (const char* e = std::getenv("GNW_PAD")) pad_ = std::max(0LL, std::atoll(e) / 2 * 2);
  if (const char* e = std::getenv("GNW_NO_GRAPH")) no_graph_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("GNW_LOOP_MODE")) fused_ = std::min(3, std::max(0, std::atoi(e)));  // gnw.h GNW_LOOP_*
  if (const char* e = std::getenv("GNW_CINV_REFINE")) cinv_refine_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("GNW_AUTO_SCHED")) auto_sched_ = std::min(2, std::max(0, std::atoi(e)));
  if (const char* e = std::getenv("GNW_FORK_VCYCLE")) fork_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("GNW_RG_RESERVE")) rg_reserve_ = std::max(0, std::atoi(e));
  // A blocking stream: ordered with the legacy default stream, so device-pointer
  // callers (e.g. torch on its default stream) need no extra synchronisation.
  GNW_CUDA_CHECK(cudaStreamCreateWithFlags(&stream_, cudaStreamDefault));
  {
    int lo = 0, hi = 0;  // the latency-bound V-cycle branch gets the higher priority
    GNW_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GNW_CUDA_CHECK(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, hi));
    for (auto& e : fork_ev_) GNW_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  for (auto& e : mev_) GNW_CUDA_CHECK(cudaEventCreate(&e));
  for (auto& e : rhs_ev_) GNW_CUDA_CHECK(cudaEventCreate(&e));
  for (auto& e : tri_ev_) GNW_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // host->device staging of the next Jacobian (prefetch_jacobian) runs on its own stream
  GNW_CUDA_CHECK(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
  for (auto& e : stage_ev_) GNW_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  st_ = mem_.alloc<MinresState>(1);
  st_plain_ = mem_.alloc<MinresState>(1);
  counters_ = mem_.alloc<unsigned>(16);
  dflag_ = mem_.alloc<int>(4);
  GNW_CUDA_CHECK(cudaMemsetAsync(counters_, 0, 16 * sizeof(unsigned), stream_));
  GNW_CUDA_CHECK(cudaMemsetAsync(st_plain_, 0, sizeof(MinresState), stream_));
  GNW_CUDA_CHECK(cudaMallocHost(&h_st_, 2 * sizeof(MinresState)));
  sync();
}

Context::~Context() {
  if (device_ < 0) return;
  cudaSetDevice(device_);
  destroy_graph();
  if (stream_) cudaStreamSynchronize(stream_);
  for (auto& e : events_)
    if (e) cudaEventDestroy(e);
  for (auto& e : jev_)
    if (e) cudaEventDestroy(e);
  for (auto& e : rhs_ev_)
    if (e) cudaEventDestroy(e);
  for (auto& e : tri_ev_)
    if (e) cudaEventDestroy(e);
  for (auto& e : mev_)
    if (e) cudaEventDestroy(e);
  for (auto& e : fork_ev_)
    if (e) cudaEventDestroy(e);
  if (side_) cudaStreamSynchronize(side_);
  if (copy_) cudaStreamSynchronize(copy_);
  for (auto& e : stage_ev_)
    if (e) cudaEventDestroy(e);
  fused_pre_.clear();  // stream-ordered blocks: freed before their stream is destroyed
  stage_mem_.reset();
  jmem_.reset();
  damg_.reset();
  fwd_amg_.reset();
  ews_.reset();
  emem_.reset();
  mem_.release_all();
  if (h_st_) cudaFreeHost(h_st_);
  if (side_) cudaStreamDestroy(side_);
  if (copy_) cudaStreamDestroy(copy_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Context::sync() { GNW_CUDA_CHECK(cudaStreamSynchronize(stream_)); }

void Context::require_device() const {
  if (device_ < 0) throw DeviceError("gnw: context has no device (created with n_devices = 0)");
}
void Context::require_mixed() const {
  if (!assembled_ || !mixed_) throw std::invalid_argument("gnw: context is not assembled with a mixed problem");
}

void Context::destroy_graph() {
  for (int k = 0; k < 3; ++k) {
    if (graph_exec_[k]) cudaGraphExecDestroy(graph_exec_[k]);
    if (graph_[k]) cudaGraphDestroy(graph_[k]);
    graph_exec_[k] = nullptr;
    graph_[k] = nullptr;
    graph_nodes_[k] = 0;
  }
}

// ---------------------------------------------------------------- assembly
void Context::assemble(const double* vertices, int64_t nv, const int64_t* cells, int64_t nc,
                       const host::AmgOptions& o) {
  destroy_graph();
  // Env GNW_DEVICE_SPGEMM=1: the setup's sparse products run on this context's device
  // (spgemm.cu, bit-identical to the host / reference sparse_matmul).  Off by default: the
  // products themselves take 3-40 ms on the B200 against 60-600 ms on 16 host cores, but
  // the host hierarchy around them makes every product a pageable upload + download
  // (n = 2048: 9.2 s setup against 7.5 s on the host).  A device-resident setup is next.
  struct HookGuard {
    explicit HookGuard(Context* c) {
      const char* e = std::getenv("GNW_DEVICE_SPGEMM");
      const char* mn = std::getenv("GNW_SPGEMM_MIN");  // products below which the host is used
      const int64_t min_products = mn ? std::atoll(mn) : (int64_t{1} << 20);
      if (c->has_device() && e && std::atoi(e) != 0)
        host::set_spgemm_hook(
            [](const host::Csr& A, const host::Csr& B, void* u) {
              Context* cx = static_cast<Context*>(u);
              GNW_CUDA_CHECK(cudaSetDevice(cx->device_));
              return device_spgemm(A, B, cx->stream_);
            },
            c, min_products);
    }
    ~HookGuard() { host::set_spgemm_hook(nullptr, nullptr, 0); }
  } hook_guard(this);
  const auto t0 = std::chrono::steady_clock::now();
  mesh_ = host::finalize_mesh(vertices, nv, cells, nc);  // mesh.cpp:85-154
  const auto t1 = std::chrono::steady_clock::now();
  Q_ = host::assemble_Q(mesh_);                          // fem_mixed.cpp:29-68
  const auto t1q = std::chrono::steady_clock::now();
  D_ = host::assemble_D(mesh_);                          // fem_mixed.cpp:70-82
  const auto t1d = std::chrono::steady_clock::now();
  // Device contexts run the Schur complement's product and the whole level pipeline of
  // amg_setup on the device (sparse_device.cuh, bit-identical; only the greedy aggregation
  // stays on the host).  Env GNW_DEVICE_SETUP=0: the host code.
  const bool dev_setup = device_setup_enabled(nc);
  fused_pre_.clear();
  if (dev_setup) GNW_CUDA_CHECK(cudaSetDevice(device_));
  S_ = dev_setup ? device_lumped_schur(Q_, D_, stream_) : host::lumped_schur(Q_, D_);  // fem_mixed.cpp:84-94
  const auto t2 = std::chrono::steady_clock::now();
  try {
    amg_ = dev_setup ? device_amg_setup(S_, o, stream_, comm_ ? nullptr : &fused_pre_, DeviceAmg::collapse_max())
                     : host::amg_setup(S_, o);           // amg.cpp:115-187
  } catch (...) {
    fused_pre_.clear();  // a setup error on a deeper level leaves the finished levels' operators behind
    throw;
  }
  if (const char* e = std::getenv("GNW_SETUP_TIMING"))
    if (std::atoi(e) != 0)
      std::fprintf(stderr, "[gnw setup] finalize_mesh %.1f ms, assemble Q %.1f ms, D %.1f ms, S_hat %.1f ms\n",
                   std::chrono::duration<double, std::milli>(t1 - t0).count(),
                   std::chrono::duration<double, std::milli>(t1q - t1).count(),
                   std::chrono::duration<double, std::milli>(t1d - t1q).count(),
                   std::chrono::duration<double, std::milli>(t2 - t1d).count());
  K_ = mesh_.ne;
  N_ = mesh_.nc;
  mixed_ = true;
  finish_assembly();
}

// The device side of an assembly: fresh work state, the saddle structure and the hierarchy
// (or, partitioned, the rank's local operators, halos and the partitioned V-cycle).
void Context::finish_assembly() {
  assembled_ = true;
  m_ = 0;
  hist_cap_ = 0;
  hist_e_ = hist_p_ = nullptr;
  if (device_ >= 0) {
    GNW_CUDA_CHECK(cudaSetDevice(device_));
    jmem_.reset();
    damg_.reset();
    fwd_amg_.reset();
    emem_.reset();
    ews_.reset();
    ews_b_ = -1;
    fwd_gmg_n_ = -1;
    jm_m_ = -1;
    dJ_ = nullptr;
    dq_ = nullptr;
    pa_.m = 0;
    mem_.release_all();
    ppart_ = ptpart_ = nullptr;
    pbar_ = nullptr;
    ppart_m_ = 0;
    st_ = mem_.alloc<MinresState>(1);
    st_plain_ = mem_.alloc<MinresState>(1);
    counters_ = mem_.alloc<unsigned>(16);
    dflag_ = mem_.alloc<int>(4);
    GNW_CUDA_CHECK(cudaMemsetAsync(counters_, 0, 16 * sizeof(unsigned), stream_));
    GNW_CUDA_CHECK(cudaMemsetAsync(st_plain_, 0, sizeof(MinresState), stream_));
    if (comm_) {  // row partition (context_rowpart.cu): local operators, halos, partitioned V-cycle
      setup_rowpart();
    } else {
      const bool timing = [] {
        const char* e = std::getenv("GNW_SETUP_TIMING");
        return e != nullptr && std::atoi(e) != 0;
      }();
      const auto t0 = std::chrono::steady_clock::now();
      upload_structure();
      sync();
      const auto t1 = std::chrono::steady_clock::now();
      upload_hierarchy();
      if (timing)
        std::fprintf(stderr, "[gnw setup] upload saddle structure %.1f ms, hierarchy (device V-cycle operators) %.1f ms\n",
                     std::chrono::duration<double, std::milli>(t1 - t0).count(),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
    }
    sync();
  }
}

// The mixed problem from its assembled Q (K x K) and D (N x K) instead of a mesh -- the
// reference's own objects (SaddleOperator{&Q, &D, ...}, inversion.hpp:18-26) -- and, with
// options, the hierarchy amg_setup(assemble_lumped_schur(Q, D), o) (inversion.cpp:196-213).
// Without options no hierarchy is built (set_hierarchy supplies one).
void Context::assemble_saddle_csr(int64_t K, int64_t N, const int64_t* qrp, const int64_t* qci, const double* qv,
                                  const int64_t* drp, const int64_t* dci, const double* dv, const host::AmgOptions* o) {
  destroy_graph();
  if (comm_) throw std::invalid_argument("gnw_assemble_saddle_csr: partitioned contexts assemble from a mesh");
  if (K <= 0 || N <= 0 || !qrp || !drp) throw std::invalid_argument("gnw_assemble_saddle_csr: empty or null matrix");
  auto csr = [](int64_t nr, int64_t nc, const int64_t* rp, const int64_t* ci, const double* v) {
    host::Csr A;
    A.n_rows = nr;
    A.n_cols = nc;
    A.rowptr.assign(rp, rp + nr + 1);
    if (rp[0] != 0) throw std::invalid_argument("gnw_assemble_saddle_csr: rowptr[0] != 0");
    const int64_t nnz = rp[nr];
    A.cols.resize(static_cast<size_t>(nnz));
    for (int64_t k = 0; k < nnz; ++k) {
      if (ci[k] < 0 || ci[k] >= nc) throw std::invalid_argument("gnw_assemble_saddle_csr: column index out of range");
      A.cols[static_cast<size_t>(k)] = static_cast<int32_t>(ci[k]);
    }
    A.vals.assign(v, v + nnz);
    return A;
  };
  Q_ = csr(K, K, qrp, qci, qv);
  D_ = csr(N, K, drp, dci, dv);
  mesh_ = host::Mesh{};
  S_ = host::lumped_schur(Q_, D_);                        // fem_mixed.cpp:84-94
  fused_pre_.clear();
  if (o && device_setup_enabled(N)) {
    GNW_CUDA_CHECK(cudaSetDevice(device_));
    try {
      amg_ = device_amg_setup(S_, *o, stream_, &fused_pre_, DeviceAmg::collapse_max());
    } catch (...) {
      fused_pre_.clear();
      throw;
    }
  } else {
    amg_ = o ? host::amg_setup(S_, *o) : host::AmgHierarchy{};  // amg.cpp:115-187
  }
  K_ = K;
  N_ = N;
  mixed_ = true;
  finish_assembly();
}

// Replaces the AMG hierarchy (a caller's own AmgHierarchy, e.g. WoodburyPreconditioner::amg);
// the Woodbury factors depend on it, so the Jacobian must be set again.
void Context::set_hierarchy(const host::AmgHierarchy& h) {
  require_mixed();
  if (comm_) throw std::invalid_argument("gnw_set_amg_hierarchy: not on a partitioned context");
  if (h.levels.empty() || h.levels[0].A.n_rows != N_) throw std::invalid_argument("gnw_set_amg_hierarchy: size mismatch");
  destroy_graph();
  amg_ = h;
  m_ = 0;
  op_.m = 0;
  pa_.m = 0;
  jm_m_ = -1;
  jmem_.reset();
  dJ_ = nullptr;
  if (device_ >= 0) {
    damg_.upload(amg_, stream_);
    sync();
  }
}

// The flux block of the preconditioner, diag(Q)^-1 (WoodburyPreconditioner::q_diag_inv,
// inversion.hpp:31), given instead of computed from Q.
void Context::set_qinv(const double* q) {
  require_mixed();
  require_device();
  if (comm_) throw std::invalid_argument("gnw_set_flux_scaling: not on a partitioned context");
  GNW_CUDA_CHECK(cudaMemcpy(const_cast<double*>(pa_.qinv), q, K_ * sizeof(double), cudaMemcpyHostToDevice));
}

void Context::assemble_amg_csr(int64_t n, const int64_t* rowptr, const int64_t* cols, const double* vals,
                               const host::AmgOptions& o) {
  destroy_graph();
  std::vector<int64_t> r, c;
  std::vector<double> v;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      r.push_back(i);
      c.push_back(cols[k]);
      v.push_back(vals[k]);
    }
  S_ = host::from_triplets(n, n, std::move(r), std::move(c), std::move(v));
  amg_ = host::amg_setup(S_, o);
  mesh_ = host::Mesh{};
  Q_ = D_ = host::Csr{};
  K_ = 0;
  N_ = n;
  mixed_ = false;
  assembled_ = true;
  m_ = 0;
  hist_cap_ = 0;
  hist_e_ = hist_p_ = nullptr;
  if (device_ >= 0) {
    GNW_CUDA_CHECK(cudaSetDevice(device_));
    jmem_.reset();
    damg_.reset();
    fwd_amg_.reset();
    emem_.reset();
    ews_.reset();
    ews_b_ = -1;
    fwd_gmg_n_ = -1;
    jm_m_ = -1;
    dJ_ = nullptr;
    dq_ = nullptr;
    pa_.m = 0;
    mem_.release_all();
    ppart_ = ptpart_ = nullptr;
    pbar_ = nullptr;
    ppart_m_ = 0;
    st_ = mem_.alloc<MinresState>(1);
    st_plain_ = mem_.alloc<MinresState>(1);
    counters_ = mem_.alloc<unsigned>(16);
    dflag_ = mem_.alloc<int>(4);
    GNW_CUDA_CHECK(cudaMemsetAsync(counters_, 0, 16 * sizeof(unsigned), stream_));
    GNW_CUDA_CHECK(cudaMemsetAsync(st_plain_, 0, sizeof(MinresState), stream_));
    upload_hierarchy();
    io_a_ = mem_.alloc<double>(n);
    io_b_ = mem_.alloc<double>(n);
    sync();
  }
}

void Context::upload_structure() {
  const cudaStream_t s = stream_;
  op_ = OperatorArgs{};
  op_.Q = upload_csr(mem_, Q_, s);
  op_.D = upload_csr(mem_, D_, s);
  {
    const host::Csr Dt = host::transpose(D_);
    op_.Dt = upload_csr(mem_, Dt, s);
    if (!std::getenv("GNW_SADDLE_CSR")) {  // experiment switch: the CSR loops of round 1
      const char* ee = std::getenv("GNW_SADDLE_ENCODE");  // 0: plain double values (A/B experiments)
      const int enc = (ee && std::atoi(ee) == 0) ? 0 : 1;
      op_.Qs = upload_sell(mem_, Q_, s, 2 * enc);
      op_.Ds = upload_sell(mem_, D_, s, enc);
      op_.Dts = upload_sell(mem_, Dt, s, enc);
    }
  }
  op_.K = K_;
  op_.N = N_;
  dnib_ = mem_.alloc<double>(1);
  op_.neg_inv_beta = dnib_;
  std::vector<double> qinv = host::diagonal(Q_);  // inversion.cpp:210-211
  for (double& v : qinv) v = 1.0 / v;
  pa_ = PrecArgs{};
  double* dq = mem_.alloc<double>(K_);
  h2d(dq, qinv.data(), qinv.size(), s);
  pa_.qinv = dq;
  pa_.K = K_;
  pa_.N = N_;
  pa_.neg_inv_beta = dnib_;
  alloc_vectors(K_ + N_, K_, N_);
}

// MINRES work vectors of n_alloc entries (K edge rows + N cell rows, plus ghosts when
// partitioned) and the per-block partial buffers of the fused reductions
void Context::alloc_vectors(long long n_alloc, long long K, long long N) {
  const int64_t n = n_alloc;
  b_ = mem_.alloc<double>(n);
  x_ = mem_.alloc<double>(n);
  r_ = mem_.alloc<double>(n);
  az_ = mem_.alloc<double>(n);
  tmp_ = mem_.alloc<double>(n);
  tmp2_ = mem_.alloc<double>(n);
  for (int k = 0; k < 3; ++k) {
    V_[k] = mem_.alloc<double>(n);
    W_[k] = mem_.alloc<double>(n);
    U_[k] = mem_.alloc<double>(n);
    Vk_[k] = V_[k] + K;
  }
  for (int k = 0; k < 2; ++k) Z_[k] = mem_.alloc<double>(n);
  io_a_ = mem_.alloc<double>(n);
  io_b_ = mem_.alloc<double>(n);
  io_c_ = mem_.alloc<double>(n);
  io_d_ = mem_.alloc<double>(n);
  const int64_t nb = (K + N + 255) / 256 + 16;
  opart_ = mem_.alloc<double>(nb * 3);
  fpart_ = mem_.alloc<double>(nb * 3);
  upart_ = mem_.alloc<double>(nb * 3);
  rpart_ = mem_.alloc<double>(nb * 3);
  plan_ = plan_h_ = row_gemv_plan(N, 1);  // re-planned for the row count by set_jacobian
  n_comb_blocks_ = combine_blocks(K, N);
  cpart_ = mem_.alloc<double>(3 * (static_cast<size_t>(n_comb_blocks_) + 16));  // one triple per combine block
  ctot_ = mem_.alloc<double>(4);  // their sum (k_sum_triples)
}

// Env GNW_DEVICE_SETUP: 1 always, 0 never; unset: from 200 000 cells up.  Measured gnw_assemble of
// a device context, device against host setup (tools/setup_compare.py): n = 256 (131 072 cells)
// 0.34 against 0.22 s, n = 512 0.44 against 0.71 s, n = 1024 1.5 against 3.0 s, n = 2048 7.9 against 15.3 s.
bool Context::device_setup_enabled(int64_t n_cells) const {
  if (!has_device()) return false;
  if (const char* e = std::getenv("GNW_DEVICE_SETUP")) return std::atoi(e) != 0;
  return n_cells >= 200000;
}

void Context::upload_hierarchy() {
  if (!amg_.levels.empty()) damg_.upload(amg_, stream_, 1, fused_pre_.empty() ? nullptr : &fused_pre_);  // adopts them
  const bool had_dev = !fused_pre_.empty();
  fused_pre_.clear();
  fused_pre_.shrink_to_fit();
  if (had_dev || device_setup_enabled(N_)) device_setup_trim();  // the setup's pool blocks go back to the driver
  svc_ = mem_.alloc<double>(std::max<int64_t>(N_, 1));
  sync();
}

// ----------------------------------------------------------------- V-cycle
// amg.cpp:90-111, one symmetric V-cycle; level 0 input may be a ring slot.
void Context::vcycle(VSel r0, double* out0, const MinresState* st, cudaStream_t s) {
  if (!comm_ && damg_.empty()) throw std::invalid_argument("amg_apply: empty hierarchy");
  if (comm_) {  // the partitioned V-cycle (part_amg.cuh), one-pass levels + replicated tail
    if (coarse_mode == 1) throw std::invalid_argument("partitioned solve: the exact coarse mode is single-GPU only");
    return pamg_->vcycle(r0, out0, st, stream_);
  }
  damg_.vcycle(r0, out0, st, coarse_mode == 1, s ? s : stream_);
}

// ------------------------------------------------------------ stage helpers
double* Context::stage_in(const double* p, size_t n, double* dev) {
  if (ptr_mode == 1) return const_cast<double*>(p);
  h2d(dev, p, n, stream_);
  return dev;
}
void Context::stage_out(double* host, const double* dev, size_t n) {
  if (ptr_mode == 1) {
    if (host != dev) GNW_CUDA_CHECK(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
    sync();
    return;
  }
  GNW_CUDA_CHECK(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
}

// ------------------------------------------------------------- Jacobian
void Context::set_jacobian(const double* J, int64_t m, int64_t n_cells, double beta, double timings[3]) {
  require_mixed();
  if (timings) timings[0] = timings[1] = timings[2] = 0.0;
  if (m > 0 && !(beta > 0.0)) throw std::invalid_argument("build_woodbury_preconditioner: beta <= 0");
  if (m > 0 && n_cells != local_n()) throw std::invalid_argument("build_woodbury_preconditioner: J shape mismatch");
  require_device();
  m_ = m;
  beta_ = beta;
  {
    const double nib = -1.0 / beta;  // axpy(-1.0 / beta, ...), inversion.cpp:66, :85
    GNW_CUDA_CHECK(cudaMemcpyAsync(dnib_, &nib, sizeof(double), cudaMemcpyHostToDevice, stream_));
  }
  if (m == 0) {  // no low-rank term at all (J == nullptr in SaddleOperator and preconditioner)
    destroy_graph();
    op_.J = nullptr;
    op_.m = 0;
    pa_.m = 0;
    pa_.Ht = pa_.Cinv = pa_.Lc = nullptr;
    return;
  }
  if (m > kMaxStageM) throw std::invalid_argument("gnw_set_jacobian: m > 8192 not supported");

  const cudaStream_t s = stream_;
  const long long Nl = local_n();  // columns of J / Ht held here (all N on one GPU)
  // Jacobian-shaped buffers persist across calls with the same (m, N, pointer
  // mode): no cudaMalloc/cudaFree (and no implied device sync) per GN step.
  const bool want_owned = ptr_mode != 1;
  if (!jmem_ || jm_m_ != m || jm_owned_ != want_owned) {
    destroy_graph();
    jmem_.reset();
    jmem_ = std::make_unique<DeviceMemory>();
    DeviceMemory& jm = *jmem_;
    u_ = jm.alloc<double>(m);
    plan_ = row_gemv_plan(Nl, static_cast<int>(m));
    plan_h_ = row_gemv_plan(Nl, static_cast<int>(m), fork_ ? rg_reserve_ : 0);  // nchunks <= plan_'s
    gpart_ = jm.alloc<double>(static_cast<size_t>(plan_.nchunks) * m);
    ldh_ = Nl + pad_;
    jown_ = want_owned ? jm.alloc<double>(static_cast<size_t>(m) * ldh_) : nullptr;
    dHt_ = jm.alloc<double>(static_cast<size_t>(m) * ldh_);
    dC_ = jm.alloc<double>(m * m);
    dL_ = jm.alloc<double>(m * m);
    dCinv_ = jm.alloc<double>(m * m);
    dY_ = jm.alloc<double>(m * m);
    t_ = jm.alloc<double>(m);
    t2_ = jm.alloc<double>(m);
    tpart_ = jm.alloc<double>(static_cast<size_t>(plan_.nchunks) * m);
    dq_ = jm.alloc<double>(std::max<long long>(nd(), 1));
    bq_ = jm.alloc<double>(std::max<long long>(nd(), 1));
    cres_ = jm.alloc<double>(m);
    if (comm_) {
      const int P = comm_->world;
      u_part_ = jm.alloc<double>(m);
      t_part_ = jm.alloc<double>(m);
      gath_ = jm.alloc<double>(static_cast<size_t>(P) * std::max<int64_t>(m, 1));
      Cpart_ = jm.alloc<double>(static_cast<size_t>(m) * m);
      Cgath_ = jm.alloc<double>(static_cast<size_t>(P) * m * m);
    }
    const DgemmPlan lo = dgemm_plan(static_cast<int>(m), Nl, 0, sm_count_);
    const DgemmPlan fu = dgemm_plan(static_cast<int>(m), Nl, 1, sm_count_);
    const size_t pl = static_cast<size_t>(lo.splits) * lo.npairs * lo.tile * lo.tile;
    const size_t pf = static_cast<size_t>(fu.splits) * fu.npairs * fu.tile * fu.tile;
    dpart_ = jm.alloc<double>(std::max(pl, pf) + 2 * 4096);
    jm_m_ = m;
    jm_owned_ = want_owned;
    for (auto& e : jev_)
      if (!e) GNW_CUDA_CHECK(cudaEventCreate(&e));
  }
  if (ptr_mode == 1) {
    // Device pointers: J is referenced, not copied -- the reference's
    // SaddleOperator/WoodburyPreconditioner also hold a non-owning pointer to J
    // (inversion.hpp:21, :35); the caller keeps it alive while the context uses it.
    if (dJ_ != J) destroy_graph();  // the loop graph bakes the J pointer
    dJ_ = const_cast<double*>(J);
    ldj_ = Nl;
    j_borrowed_ = true;
  } else {
    if (dJ_ != jown_) destroy_graph();
    dJ_ = jown_;
    ldj_ = ldh_;  // owned copy: padded rows like Ht
    j_borrowed_ = false;
    if (staged_src_ == J && staged_m_ == m && staged_n_ == Nl && staged_ld_ == ldj_) {
      issue_stage();  // no-op unless no solve ran since the prefetch
      // prefetch_jacobian already moved these bytes over PCIe beside the previous solve:
      // one device copy (2 x 8 m N bytes of HBM traffic) instead of the host transfer
      GNW_CUDA_CHECK(cudaStreamWaitEvent(s, stage_ev_[0], 0));
      GNW_CUDA_CHECK(cudaMemcpyAsync(dJ_, jstage_, static_cast<size_t>(staged_rows_) * ldj_ * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
      GNW_CUDA_CHECK(cudaEventRecord(stage_ev_[1], s));  // the staging buffer is free again
      if (staged_rows_ < m)  // partial stage (C3/C5): the remaining rows cross PCIe now
        GNW_CUDA_CHECK(cudaMemcpy2DAsync(dJ_ + static_cast<size_t>(staged_rows_) * ldj_, ldj_ * sizeof(double),
                                         J + static_cast<size_t>(staged_rows_) * Nl, Nl * sizeof(double),
                                         Nl * sizeof(double), m - staged_rows_, cudaMemcpyHostToDevice, s));
    } else {
      GNW_CUDA_CHECK(cudaMemcpy2DAsync(dJ_, ldj_ * sizeof(double), J, Nl * sizeof(double), Nl * sizeof(double), m,
                                       cudaMemcpyHostToDevice, s));
    }
    staged_src_ = nullptr;
    stage_deferred_ = false;
  }
  op_.J = dJ_;
  op_.ldj = ldj_;
  pa_.ldj = ldj_;
  pa_.ldh = ldh_;
  op_.m = static_cast<int>(m);
  if (pc_laplace) {  // Alg. 4: J stays in the operator, plain Laplace preconditioner
    if (pa_.m != 0) destroy_graph();
    pa_.m = 0;
    sync();
    return;
  }
  if (pa_.m != static_cast<int>(m)) destroy_graph();
  if (!comm_ && damg_.empty()) throw std::invalid_argument("build_woodbury_preconditioner: empty hierarchy");

  cudaEvent_t* ev = jev_;
  const uint64_t l0 = launch_count();
  GNW_CUDA_CHECK(cudaEventRecord(ev[0], s));
  // H = S_hat^-1 J^T by batched V-cycles (inversion.cpp:107-114); stored as Ht (m x N)
  {
    int b = damg_.batch_capacity();
    if (!comm_ && b < ((m + 31) / 32) * 32 && b < 512) {
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      const double per_col = 8.0 * static_cast<double>(N_) * 8.0;  // level-0 arrays x ~2 for coarser levels
      int64_t bmax = static_cast<int64_t>(0.5 * static_cast<double>(free_b) / per_col);
      bmax = std::max<int64_t>(32, std::min<int64_t>(bmax, 512) / 32 * 32);
      b = static_cast<int>(std::min<int64_t>(((m + 31) / 32) * 32, bmax));
      damg_.ensure_batch(b);
    }
    if (comm_) {
      build_h_rowpart();
    } else {
      for (int64_t i0 = 0; i0 < m; i0 += b) {
        const int bb = static_cast<int>(std::min<int64_t>(b, m - i0));
        transpose_rows_to_batch(dJ_, N_, ldj_, static_cast<int>(i0), bb, damg_.batch_in(), s);
        if (!damg_.vcycle_batch(damg_.batch_in(), bb, damg_.batch_out(), coarse_mode == 1, st_plain_, s,
                                dHt_ + i0 * ldh_, ldh_))
          transpose_batch_to_rows(damg_.batch_out(), N_, ldh_, static_cast<int>(i0), bb, dHt_, s);
      }
    }
    GNW_CUDA_CHECK(cudaEventRecord(ev[1], s));
  }
  // C = I + (J H)/beta (inversion.cpp:37-43), lower triangle
  DgemmPlan plan = dgemm_plan(static_cast<int>(m), Nl, 0, sm_count_);
  // partitioned: C = I + (sum_r J_r H_r^T)/beta from the ranks' raw partials, fixed order
  auto capacitance = [&](const DgemmPlan& pl) {
    if (!comm_) return capacitance_dgemm(dJ_, ldj_, dHt_, ldh_, static_cast<int>(m), N_, beta, pl, dpart_, dC_, s);
    fill_zero(Cpart_, m * m, s);
    capacitance_dgemm(dJ_, ldj_, dHt_, ldh_, static_cast<int>(m), Nl, 0.0, pl, dpart_, Cpart_, s);
    comm_->allgather(Cpart_, Cgath_, m * m, s);
    capacitance_reduce(Cgath_, comm_->world, static_cast<int>(m), beta, dC_, s);
  };
  {
    capacitance(plan);
    GNW_CUDA_CHECK(cudaEventRecord(ev[2], s));
    // L = chol(C), retry once after symmetrisation (inversion.cpp:21-35)
    cholesky_blocked(dC_, dY_, dL_, static_cast<int>(m), dflag_, s);
    int fail = 0;
    GNW_CUDA_CHECK(cudaMemcpyAsync(&fail, dflag_, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync();
    if (fail) {
      DgemmPlan full = dgemm_plan(static_cast<int>(m), Nl, 1, sm_count_);
      capacitance(full);
      symmetrize(dC_, static_cast<int>(m), s);
      cholesky_blocked(dC_, dY_, dL_, static_cast<int>(m), dflag_, s);
      GNW_CUDA_CHECK(cudaMemcpyAsync(&fail, dflag_, sizeof(int), cudaMemcpyDeviceToHost, s));
      sync();
      if (fail) throw std::runtime_error("dense_cholesky: matrix not positive definite");
    }
    cholesky_inverse(dL_, dY_, dCinv_, static_cast<int>(m), s);
    if (!fail) mirror_lower(dC_, static_cast<int>(m), s);  // full C for the fused loops' refinement
    GNW_CUDA_CHECK(cudaEventRecord(ev[3], s));
    // kappa(C) >= (max L_ii / min L_ii)^2: beyond ~1e10 the explicit inverse is not accurate
    // enough for the preconditioner (its error grows like eps kappa), so C^-1 t runs as the
    // reference does, by the triangular solves with L (cholesky_solve_in_place, linalg.cpp:107-123)
    std::vector<double> ld(static_cast<size_t>(m));
    GNW_CUDA_CHECK(cudaMemcpy2DAsync(ld.data(), sizeof(double), dL_, (m + 1) * sizeof(double), sizeof(double), m,
                                     cudaMemcpyDeviceToHost, s));
    sync();
    double dmax = 0.0, dmin = std::numeric_limits<double>::infinity();
    for (double v : ld) {
      dmax = std::max(dmax, std::fabs(v));
      dmin = std::min(dmin, std::fabs(v));
    }
    const bool tri = !(dmin > 0.0) || (dmax / dmin) * (dmax / dmin) > 1e10;
    if (tri != (pa_.cap_tri != 0)) destroy_graph();
    pa_.cap_tri = tri ? 1 : 0;
  }
  float ms[3];
  for (int k = 0; k < 3; ++k) GNW_CUDA_CHECK(cudaEventElapsedTime(&ms[k], ev[k], ev[k + 1]));
  if (timings) {
    timings[0] = ms[0] * 1e-3;
    timings[1] = ms[1] * 1e-3;
    timings[2] = ms[2] * 1e-3;
  }
  setup_launches = launch_count() - l0;
  pa_.m = static_cast<int>(m);
  pa_.Ht = dHt_;
  pa_.Cinv = dCinv_;
  pa_.Lc = dL_;
}

// Starts the host->device transfer of the NEXT step's Jacobian on the copy stream, into a
// staging buffer, so it overlaps whatever the context runs meanwhile (the current step's
// MINRES).  The next set_jacobian with the same host pointer and shape waits for it on the
// device and takes the staged bytes; any other set_jacobian drops the stage.  The caller
// keeps the host array unchanged until then (pinned memory gives the overlap; pageable
// memory makes the copy synchronous, still correct).  Host-pointer mode only.  When a second
// J-sized buffer does not fit beside the solve's working set, nothing is staged.
void Context::prefetch_jacobian(const double* J, int64_t m, int64_t n_cells) {
  require_mixed();
  require_device();
  if (ptr_mode == 1) throw std::invalid_argument("gnw_prefetch_jacobian: host-pointer mode only");
  if (J == nullptr || m <= 0 || m > kMaxStageM) throw std::invalid_argument("gnw_prefetch_jacobian: bad J");
  if (n_cells != local_n()) throw std::invalid_argument("gnw_prefetch_jacobian: J shape mismatch");
  const long long Nl = local_n();
  const long long ld = Nl + pad_;  // the owned copy's padded row stride (set_jacobian)
  // Stage as many leading rows of J as fit beside the solve: all of them at C1/C2/C4; at
  // C3/C5 (J + H already take 127-137 GB of the 179) the rows that fit in what is left, and
  // set_jacobian copies only the remainder over PCIe.
  int64_t rows = m;
  // (re)size only when the shape changes: a partial stage (C3/C5) keeps its buffer across
  // steps instead of re-entering this branch (device sync + a tens-of-GB free/malloc) each call
  if (stage_key_m_ != m || stage_key_ld_ != ld) {
    GNW_CUDA_CHECK(cudaStreamSynchronize(copy_));
    sync();  // a pending consume of the old buffer
    stage_mem_.reset();
    stage_cap_ = 0;
    stage_key_m_ = stage_key_ld_ = -1;
    size_t free_b = 0, total_b = 0;
    GNW_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
    const size_t margin = size_t{4} << 30;
    const size_t row_b = static_cast<size_t>(ld) * sizeof(double);
    rows = free_b > margin ? std::min<int64_t>(m, static_cast<int64_t>((free_b - margin) / row_b)) : 0;
    if (const char* e = std::getenv("GNW_STAGE_ROWS_MAX")) rows = std::min<int64_t>(rows, std::atoll(e));  // tests
    stage_key_m_ = m;
    stage_key_ld_ = ld;
    if (rows < std::max<int64_t>(1, m / 16)) {  // too little to matter: set_jacobian copies as usual
      staged_src_ = nullptr;
      stage_deferred_ = false;
      return;
    }
    stage_mem_ = std::make_unique<DeviceMemory>();
    jstage_ = stage_mem_->alloc<double>(static_cast<size_t>(rows) * ld);
    stage_cap_ = static_cast<size_t>(rows) * ld;
    GNW_CUDA_CHECK(cudaEventRecord(stage_ev_[1], stream_));
  }
  if (stage_cap_ == 0) {  // this shape stages nothing (decided above on an earlier call)
    staged_src_ = nullptr;
    stage_deferred_ = false;
    return;
  }
  rows = std::min<int64_t>(m, static_cast<int64_t>(stage_cap_ / static_cast<size_t>(ld)));
  staged_src_ = J;
  staged_m_ = m;
  staged_rows_ = rows;
  staged_n_ = Nl;
  staged_ld_ = ld;
  stage_deferred_ = true;
}

// The staged copy is issued once the next MINRES has its own inputs on the device (or by
// set_jacobian if no solve comes first): host->device copies share the copy engine, so a
// 1 GB transfer queued ahead of minres's b / x0 uploads would hold the solve back.
void Context::issue_stage() {
  if (!stage_deferred_) return;
  stage_deferred_ = false;
  // the previous stage must have been consumed (device-side order, no host wait)
  GNW_CUDA_CHECK(cudaStreamWaitEvent(copy_, stage_ev_[1], 0));
  GNW_CUDA_CHECK(cudaMemcpy2DAsync(jstage_, staged_ld_ * sizeof(double), staged_src_, staged_n_ * sizeof(double),
                                   staged_n_ * sizeof(double), staged_rows_, cudaMemcpyHostToDevice, copy_));
  GNW_CUDA_CHECK(cudaEventRecord(stage_ev_[0], copy_));
}

// --------------------------------------------------------------- operator
// fused: the MINRES loop's A zhat takes J^T u from q = J^T t' (fused_active()).
void Context::operator_into(VSel x, int scaled, VSel y, MinresState* st, int loop, bool fused) {
  OperatorArgs op = op_;
  if (comm_) {  // partitioned: ghosts of x, u = sum_r J_r x_r (fixed-order), own rows, delta reduced
    exchange_saddle(resolve(x));
    if (fused) {
      op.q = dq_;
    } else if (m_ > 0) {
      row_gemv(dJ_, static_cast<int>(m_), Nl_, ldj_, x, Kl_, scaled, st, gpart_, counters_ + 0, u_part_, plan_,
               stream_);
      reduce_m(u_part_, u_, m_, stream_);
    }
    saddle_operator(op, x, scaled, u_, y, st, 0, opart_, counters_ + 1, stream_);
    reduce_scratch(st, 0, 1);
    if (loop) delta_coef(st, stream_);
    return;
  }
  if (fused) {
    op.q = dq_;
  } else if (m_ > 0 && !(exp_skip_ & 1)) {
    VSel xs = x;  // J acts on the cell part
    row_gemv(dJ_, static_cast<int>(m_), N_, ldj_, xs, K_, scaled, st, gpart_, counters_ + 0, u_, plan_, stream_);
  }
  if (!(exp_skip_ & 2)) saddle_operator(op, x, scaled, u_, y, st, loop, opart_, counters_ + 1, stream_);
}

int Context::loop_sched() const {
  if (!fused_ || fused_off_ || m_ == 0 || pa_.m == 0 || dq_ == nullptr) return 0;
  if (fused_ != 2) return fused_ == 1 ? 1 : 2;
  if (auto_sched_) return auto_sched_;
  // auto: lean trades one dense sweep (8 m N bytes) for a second, serialised V-cycle, which
  // runs well below the HBM roofline on small levels (latency-bound): lean when the sweep
  // outweighs two V-cycles' bytes (C2-C5; C1 stays fused)
  return 8.0 * static_cast<double>(m_) * static_cast<double>(N_) > 2.0 * vcycle_bytes() ? 2 : 1;
}

// The persistent cooperative kernel (minres_persistent.cu) runs the lean schedule's arithmetic
// for problems whose working set stays in L2: requested (GNW_LOOP_PERSISTENT) or picked by
// GNW_LOOP_AUTO (env GNW_PERSISTENT=0: never).
bool Context::persistent_eligible() const {
  static const bool env_on = [] {
    const char* e = std::getenv("GNW_PERSISTENT");
    return !(e && std::atoi(e) == 0);
  }();
  if (persist_mode_ == 0 || (persist_mode_ == 1 && !env_on)) return false;
  if (comm_ || no_graph_ || coarse_mode != 0 || pc_laplace || loop_sched() == 0) return false;
  if (m_ < 1 || m_ > persistent_max_m() || pa_.cap_tri || !cinv_refine_ || dC_ == nullptr || dq_ == nullptr || bq_ == nullptr)
    return false;
  if (op_.Qs.width <= 0 || op_.Dts.width <= 0 || op_.Ds.width <= 0) return false;
  PersistArgs probe;
  if (!damg_.fill_persist(probe)) return false;
  // the vectors, J, H and the dense tail together must stay L2-resident (B200: 126 MB)
  const double bytes = 16.0 * static_cast<double>(m_) * static_cast<double>(N_) + 8.0 * 20.0 * static_cast<double>(K_ + N_) +
                       8.0 * static_cast<double>(probe.nM) * probe.nM;
  return bytes <= 96e6;
}

void Context::apply_operator(const double* x, double* y) {
  require_mixed();
  require_device();
  if (comm_) {  // global x in (own entries and ghosts read from it), global y out
    global_to_local(global_in(x, K_ + N_, gio_a_), io_a_, true);
    operator_into(vfixed(io_a_), 0, vfixed(io_b_), st_plain_, 0);
    local_to_global(io_b_, gio_b_);
    return global_out(y, gio_b_, K_ + N_);
  }
  const size_t n = K_ + N_;
  double* dx = stage_in(x, n, io_a_);
  double* dy = ptr_mode == 1 ? y : io_b_;
  operator_into(vfixed(dx), 0, vfixed(dy), st_plain_, 0);
  stage_out(y, dy, n);
}

// z = P^-1 y.  In the loop, y = v_next is formed on the fly from Az, v_cur, v_prev.
void Context::precondition_into(VSel y, VSel yv2, VSel z, MinresState* st, int loop, VSel vcur, VSel vprev,
                                int sched) {
  pa_.exact = coarse_mode;
  PrecArgs pa = pa_;
  if (sched == 1) {  // fused: the finish sweep also forms q = J^T t' for the next operator
    pa.J = dJ_;
    pa.q = dq_;
  }
  if (sched != 0 && cinv_refine_) {
    pa.Cfull = dC_;
    pa.cres = cres_;
  }
  const VSel az = loop ? vfixed(az_) : y;
  if (!(exp_skip_ & 4)) combine_elem(pa, az, vcur, vprev, y, z, loop, st, cpart_, stream_);
  // partitioned: the m-partials of the row GEMVs and the finish kernel's dots are summed over the
  // ranks (fixed order) before anything reads them
  double* tdst = comm_ ? t_part_ : t_;
  auto reduce_t = [&]() {
    if (comm_) reduce_m(t_part_, t_, pa.m, stream_);
  };
  // single GPU: the combine kernel's dot partials are pre-summed on a side branch beside the
  // dense sweeps (k_sum_triples), so the finish kernel adds one triple
  static const bool tri_branch = [] {  // env GNW_TRI_BRANCH=0: the finish kernel sums the partials
    const char* e = std::getenv("GNW_TRI_BRANCH");
    return !(e && std::atoi(e) == 0);
  }();
  const bool pre = tri_branch && fork_ && !comm_ && !(exp_skip_ & (4 | 64));  // the finish kernel joins the branch
  if (pre) {
    GNW_CUDA_CHECK(cudaEventRecord(tri_ev_[0], stream_));
    GNW_CUDA_CHECK(cudaStreamWaitEvent(side_, tri_ev_[0], 0));
    sum_triples(cpart_, n_comb_blocks_, ctot_, side_);
    GNW_CUDA_CHECK(cudaEventRecord(tri_ev_[1], side_));
  }
  auto finish = [&](const PrecArgs& pf) {
    if (pre) GNW_CUDA_CHECK(cudaStreamWaitEvent(stream_, tri_ev_[1], 0));
    finish_precondition(pf, svc_, t2_, y, z, comm_ ? 0 : loop, st, pre ? ctot_ : cpart_, pre ? 1 : n_comb_blocks_,
                        fpart_, counters_ + 3, stream_);
    if (comm_) {
      reduce_scratch(st, 0, 3);
      if (loop) givens_from_scratch(st, stream_);
    }
  };
  if (sched == 2) {
    // lean: H = B J^T and B is linear, so z2 = B v2 - H t' / beta = B (v2 - J^T t' / beta).
    // Two dense sweeps (t = H^T v2; q = J^T t', which is also the next operator's J^T u up
    // to 1 / gamma) and ONE V-cycle, on the sweep's output y' = v2 - q / beta.
    if (!(exp_skip_ & 8)) {
      row_gemv(pa.Ht, pa.m, pa.N, pa.ldh, y, pa.K, 0, st, tpart_, counters_ + 2, tdst, plan_, stream_);
      reduce_t();
    }
    if (!(exp_skip_ & 32)) capacitance_solve(pa, t_, t2_, stream_);
    if (!(exp_skip_ & 256)) col_sweep(dJ_, ldj_, t2_, pa.m, pa.N, dq_, stream_, y, pa.K, st, pa.neg_inv_beta, bq_);
    if (!(exp_skip_ & 16)) vcycle(vfixed(bq_), svc_, st);
    PrecArgs pf = pa;
    pf.m = 0;  // z2 = B y' is the V-cycle's output: the finish step is elementwise
    if (!(exp_skip_ & 64)) finish(pf);
    return;
  }
  // s = B y2 and t = H^T y2 both read only y2: the V-cycle (latency-bound, few
  // CTAs on its coarse levels) runs on side_ beside the bandwidth-bound GEMV.
  const bool fork = fork_ && pa.m > 0;
  if (fork) {
    GNW_CUDA_CHECK(cudaEventRecord(fork_ev_[0], stream_));
    GNW_CUDA_CHECK(cudaStreamWaitEvent(side_, fork_ev_[0], 0));
    if (!(exp_skip_ & 16)) vcycle(yv2, svc_, st, side_);
    GNW_CUDA_CHECK(cudaEventRecord(fork_ev_[1], side_));
  }
  if (pa.m > 0 && !(exp_skip_ & 8)) {  // t = H^T v2 (matvec_transpose(h_hat, y2), inversion.cpp:82)
    row_gemv(pa.Ht, pa.m, pa.N, pa.ldh, y, pa.K, 0, st, tpart_, counters_ + 2, tdst, plan_h_, stream_);
    reduce_t();
  }
  if (!fork && !(exp_skip_ & 16)) vcycle(yv2, svc_, st);
  if (!(exp_skip_ & 32)) capacitance_solve(pa, t_, t2_, stream_);
  if (fork) GNW_CUDA_CHECK(cudaStreamWaitEvent(stream_, fork_ev_[1], 0));
  if (!(exp_skip_ & 64)) finish(pa);
}

void Context::precondition(const double* y, double* z) {
  require_mixed();
  require_device();
  if (comm_) {
    global_to_local(global_in(y, K_ + N_, gio_a_), io_a_, false);
    precondition_into(vfixed(io_a_), vfixed(io_a_ + Kl_), vfixed(io_b_), st_plain_, 0, vfixed(io_a_), vfixed(io_a_),
                      loop_sched());
    local_to_global(io_b_, gio_b_);
    return global_out(z, gio_b_, K_ + N_);
  }
  const size_t n = K_ + N_;
  double* dy = stage_in(y, n, io_a_);
  double* dz = ptr_mode == 1 ? z : io_b_;
  precondition_into(vfixed(dy), vfixed(dy + K_), vfixed(dz), st_plain_, 0, vfixed(dy), vfixed(dy));
  stage_out(z, dz, n);
}

void Context::amg_apply(const double* r, double* z) {
  if (!assembled_) throw std::invalid_argument("amg_apply: empty hierarchy");
  require_device();
  if (comm_) {  // the partitioned V-cycle on the own cells of a global r; global z
    const double* g = global_in(r, N_, gio_c_);
    GNW_CUDA_CHECK(cudaMemcpyAsync(io_a_, g + c_lo_, Nl_ * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
    vcycle(vfixed(io_a_), io_b_, st_plain_);
    GNW_CUDA_CHECK(cudaMemcpyAsync(gio_d_ + c_lo_, io_b_, Nl_ * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
    const int P = comm_->world;
    std::vector<long long> off(P), cnt(P);
    for (int q = 0; q < P; ++q) {
      off[q] = part_lo_[q];
      cnt[q] = part_lo_[q + 1] - part_lo_[q];
    }
    comm_->allgatherv(gio_d_, off, cnt, stream_);
    return global_out(z, gio_d_, N_);
  }
  const size_t n = N_;
  double* dr = stage_in(r, n, io_a_);
  double* dz = ptr_mode == 1 ? z : io_b_;
  vcycle(vfixed(dr), dz, st_plain_);
  stage_out(z, dz, n);
}

void Context::assemble_rhs(const double* mdl, const double* mref, const double* g, const double* gobs, double* rhs) {
  require_mixed();
  require_device();
  if (m_ == 0) throw std::invalid_argument("assemble_gn_rhs: shape mismatch");
  // g - g_obs is formed inside the rhs kernel (same subtraction as inversion.cpp:137-138):
  // no device -> host round trip and no host sync before the launch
  const double* dgv = g;
  const double* dgo = gobs;
  if (ptr_mode != 1) {
    h2d(t_, g, m_, stream_);
    h2d(t2_, gobs, m_, stream_);
    dgv = t_;
    dgo = t2_;
  }
  if (comm_) {  // own edges read m - m_ref on their ghost cells too (cell layout of the local D^T)
    const double* gm = global_in(mdl, N_, gio_c_);
    gather_rows(cell_l2g_, n_cell_l2g_, gm, io_a_, 1, stream_);
    const double* gr = global_in(mref, N_, gio_d_);
    gather_rows(cell_l2g_, n_cell_l2g_, gr, io_b_, 1, stream_);
    GNW_CUDA_CHECK(cudaEventRecord(rhs_ev_[0], stream_));
    gnw::assemble_rhs(op_, beta_, io_a_, io_b_, dgv, dgo, io_c_, stream_);
    GNW_CUDA_CHECK(cudaEventRecord(rhs_ev_[1], stream_));
    local_to_global(io_c_, gio_b_);
    global_out(rhs, gio_b_, K_ + N_);
  } else {
    double* dm = stage_in(mdl, N_, io_a_);
    double* dmr = stage_in(mref, N_, io_b_);
    double* dr = ptr_mode == 1 ? rhs : io_c_;
    GNW_CUDA_CHECK(cudaEventRecord(rhs_ev_[0], stream_));
    gnw::assemble_rhs(op_, beta_, dm, dmr, dgv, dgo, dr, stream_);
    GNW_CUDA_CHECK(cudaEventRecord(rhs_ev_[1], stream_));
    stage_out(rhs, dr, K_ + N_);
  }
  float ms = 0.f;
  GNW_CUDA_CHECK(cudaEventElapsedTime(&ms, rhs_ev_[0], rhs_ev_[1]));
  t_rhs = ms * 1e-3;
}

// The reference's GN-step solve (inversion.cpp:259-265): b = assemble_gn_rhs(...), x0 = 0,
// minres(op, pc, b, x0, tol, maxit) as ONE call.  The right-hand side is assembled straight into
// the solver's b on the device and never visits the host; the zero start needs no transfer.
MinresResult Context::gn_step_solve(const double* mdl, const double* mref, const double* g, const double* gobs,
                                    double* x, double tol, uint64_t maxit) {
  if (!(tol > 0.0)) throw std::invalid_argument("minres: tol must be positive");
  require_mixed();
  require_device();
  if (comm_) throw std::invalid_argument("gn_step_solve: single-GPU contexts (partitioned: assemble_rhs + minres_solve)");
  if (m_ == 0) throw std::invalid_argument("assemble_gn_rhs: shape mismatch");
  const double* dgv = g;
  const double* dgo = gobs;
  if (ptr_mode != 1) {
    h2d(t_, g, m_, stream_);
    h2d(t2_, gobs, m_, stream_);
    dgv = t_;
    dgo = t2_;
  }
  double* dm = stage_in(mdl, N_, io_a_);
  double* dmr = stage_in(mref, N_, io_b_);
  GNW_CUDA_CHECK(cudaEventRecord(rhs_ev_[0], stream_));
  gnw::assemble_rhs(op_, beta_, dm, dmr, dgv, dgo, b_, stream_);
  GNW_CUDA_CHECK(cudaEventRecord(rhs_ev_[1], stream_));
  MinresResult r = minres(nullptr, nullptr, x, tol, maxit);
  float ms = 0.f;
  GNW_CUDA_CHECK(cudaEventElapsedTime(&ms, rhs_ev_[0], rhs_ev_[1]));
  t_rhs = ms * 1e-3;
  return r;
}

// ------------------------------------------------------------------ MINRES
// One MINRES iteration (minres.cpp:70-148) as device work, ring slots chosen on the
// device from st_->j.  Captured once into the conditional-WHILE graph body, or
// launched per iteration by the host in GNW_NO_GRAPH (profiling) mode.
void Context::launch_iteration(unsigned long long cond_handle, int use_cond) {
  const int sc = loop_sched();
  operator_into(ring2(Z_, 0), 1, vfixed(az_), st_, 1, sc != 0);             // Az = A zhat, delta
  precondition_into(ring3(V_, 2), ring3(Vk_, 2), ring2(Z_, 1), st_, 1,       // v_next, z_next = P^-1 v_next,
                    ring3(V_, 1), ring3(V_, 0), sc);                         // gamma_next, Givens
  if (!(exp_skip_ & 128)) {
    minres_update(kd() + nd(), ring2(Z_, 0), vfixed(az_), ring3(W_, 0), ring3(W_, 1), ring3(W_, 2), ring3(U_, 0),
                  ring3(U_, 1), ring3(U_, 2), x_, r_, st_, hist_e_, hist_p_, hist_cap_, upart_, counters_ + 4,
                  cond_handle, comm_ ? 3 : use_cond, stream_);
    if (comm_) {  // ||r||^2 over the ranks, then the loop-control epilogue on every rank
      reduce_scratch(st_, 6, 1);
      update_tail_from_scratch(st_, hist_e_, hist_p_, hist_cap_, stream_);
    }
  }
}

void Context::build_graph() {
  const int slot = loop_sched();
  if (graph_exec_[slot]) cudaGraphExecDestroy(graph_exec_[slot]);
  if (graph_[slot]) cudaGraphDestroy(graph_[slot]);
  graph_exec_[slot] = nullptr;
  graph_[slot] = nullptr;
  cudaGraph_t g;
  GNW_CUDA_CHECK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  GNW_CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  alignas(cudaGraphNodeParams) unsigned char pbuf[sizeof(cudaGraphNodeParams)] = {};
  cudaGraphNodeParams& p = *reinterpret_cast<cudaGraphNodeParams*>(pbuf);
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  GNW_CUDA_CHECK(cudaGraphAddNode(&node, g, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  const uint64_t l0 = launch_count();
  GNW_CUDA_CHECK(cudaStreamBeginCaptureToGraph(stream_, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  // iteration j: v_prev = V[j%3], v_cur = V[(j+1)%3], v_next = V[(j+2)%3] (same for w, u);
  //              z_cur = Z[j%2], z_next = Z[(j+1)%2]
  try {
    launch_iteration(static_cast<unsigned long long>(h), 1);
  } catch (...) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(stream_, &dummy);
    cudaGraphDestroy(g);
    throw;
  }
  GNW_CUDA_CHECK(cudaStreamEndCapture(stream_, &body));
  graph_nodes_[slot] = launch_count() - l0;
  GNW_CUDA_CHECK(cudaGraphInstantiate(&graph_exec_[slot], g, 0));
  graph_[slot] = g;
}

MinresResult Context::minres(const double* b, const double* x0, double* x, double tol, uint64_t maxit) {
  if (!(tol > 0.0)) throw std::invalid_argument("minres: tol must be positive");
  require_mixed();
  require_device();
  const int64_t n = kd() + nd();  // own rows (partitioned: b and x0 are global, taken apart below)
  const cudaStream_t s = stream_;
  MinresResult res;
  const CommTally tally0 = comm_tally();
  const uint64_t l0 = launch_count();
  uint64_t graph_launched = 0;  // kernels run inside loop-graph launches
  uint64_t sched_iters[3] = {0, 0, 0};  // iterations run per loop schedule
  uint64_t built_now = 0;

  const long long cap = static_cast<long long>(std::min<uint64_t>(maxit, 4u << 20)) + 1;
  if (cap > hist_cap_) {
    destroy_graph();
    hist_e_ = mem_.alloc<double>(cap);
    hist_p_ = mem_.alloc<double>(cap);
    hist_cap_ = cap;
  }
  cudaEvent_t e0, e1;
  GNW_CUDA_CHECK(cudaEventCreate(&e0));
  GNW_CUDA_CHECK(cudaEventCreate(&e1));
  // b == nullptr: b_ already holds the right-hand side (gn_step_solve assembled it there);
  // x0 == nullptr: the zero start of the reference's GN step (inversion.cpp:261)
  if (comm_ && (b == nullptr || x0 == nullptr))
    throw std::invalid_argument("minres: partitioned solves take b and x0 explicitly");
  if (comm_) {
    global_to_local(global_in(b, K_ + N_, gio_a_), b_, false);
    global_to_local(global_in(x0, K_ + N_, gio_b_), x_, false);
  } else {
    if (b != nullptr) {
      if (ptr_mode == 1)
        GNW_CUDA_CHECK(cudaMemcpyAsync(b_, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      else
        h2d(b_, b, n, s);
    }
    if (x0 == nullptr)
      GNW_CUDA_CHECK(cudaMemsetAsync(x_, 0, n * sizeof(double), s));
    else if (ptr_mode == 1)
      GNW_CUDA_CHECK(cudaMemcpyAsync(x_, x0, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    else
      h2d(x_, x0, n, s);
  }
  GNW_CUDA_CHECK(cudaEventRecord(e0, s));
  auto read_plain = [&]() {
    GNW_CUDA_CHECK(cudaMemcpyAsync(h_st_ + 1, st_plain_, sizeof(MinresState), cudaMemcpyDeviceToHost, s));
    sync();
    return h_st_[1];
  };
  // r = b - A x  (and ||b||).  With the zero start A x0 is exactly zero (every product is a
  // signed zero and every row sum +0.0, so b - A x0 = b bit for bit): no operator pass
  if (x0 == nullptr)
    GNW_CUDA_CHECK(cudaMemsetAsync(az_, 0, n * sizeof(double), s));
  else
    operator_into(vfixed(x_), 0, vfixed(az_), st_plain_, 0);
  residual(n, b_, az_, r_, st_plain_, 1, rpart_, counters_ + 5, s);
  if (comm_) reduce_scratch(st_plain_, 4, 2);
  MinresState ps = read_plain();
  issue_stage();  // b and x0 are on the device now: a prefetched J may take the copy engine
  const double bnorm = std::sqrt(ps.scratch[5]);
  auto finish = [&]() {
    GNW_CUDA_CHECK(cudaEventRecord(e1, s));
    sync();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    t_minres = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    launches = launch_count() - l0 - built_now + graph_launched;
    comm_calls_ = comm_tally().calls - tally0.calls;
    comm_bytes_ = comm_tally().bytes - tally0.bytes;
    if (comm_) {
      local_to_global(x_, gio_a_);
      global_out(x, gio_a_, K_ + N_);
    } else {
      stage_out(x, x_, n);
    }
  };
  if (bnorm == 0.0) {  // minres.cpp:32-39
    res.converged = (ps.scratch[4] == 0.0);
    res.hist_e.push_back(0.0);
    res.hist_p.push_back(0.0);
    finish();
    return res;
  }
  fused_off_ = (fused_ == 2 && tol < kAutoFusedTol);  // auto: tight tolerances keep the reference schedule
  // One MINRES cycle from r_ (minres.cpp:44-63) with iteration index j0: z = P^-1 r,
  // gamma_1, and the initial ring vectors v_prev = 0, v_cur = r, w = u = 0 in the slots
  // iteration j0 reads.  Returns gamma_1 (the cycle's), or throws like the reference.
  auto start_cycle = [&](long long j0, double* gamma_out, double* rel_out) {
    double* zc = Z_[j0 % 2];
    precondition_into(vfixed(r_), vfixed(r_ + kd()), vfixed(zc), st_plain_, 0, vfixed(r_), vfixed(r_),
                      loop_sched());
    const MinresState q = read_plain();
    if (q.scratch[0] < 0.0) throw std::runtime_error("minres: preconditioner is not positive definite");
    *gamma_out = std::sqrt(q.scratch[0]);
    *rel_out = std::sqrt(q.scratch[4]) / bnorm;  // residual kernel's ||r||^2 (scratch[4] untouched since)
    fill_zero(V_[j0 % 3], n, s);
    GNW_CUDA_CHECK(cudaMemcpyAsync(V_[(j0 + 1) % 3], r_, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    for (long long k = j0; k < j0 + 2; ++k) {
      fill_zero(W_[k % 3], n, s);
      fill_zero(U_[k % 3], n, s);
    }
  };
  double gamma1 = 0.0, rel0 = 0.0;
  start_cycle(1, &gamma1, &rel0);
  res.hist_e.push_back(rel0);
  res.hist_p.push_back(1.0);
  if (rel0 <= tol) {
    res.converged = true;
    res.true_rel = rel0;
    finish();
    return res;
  }
  if (gamma1 == 0.0) throw std::runtime_error("minres: breakdown (zero preconditioned residual, nonzero residual)");
  MinresState st;
  std::memset(&st, 0, sizeof st);
  st.gamma_prev = 1.0;
  st.gamma_cur = gamma1;
  st.c_prev = st.c_cur = 1.0;
  st.s_prev = st.s_cur = 0.0;
  st.eta = gamma1;
  st.gamma1 = gamma1;
  st.bnorm = bnorm;
  st.tol = tol;
  st.exhausted_tol = 1e-13 * gamma1;
  st.inv_gamma = 1.0 / gamma1;
  st.j = 1;
  st.maxit = static_cast<long long>(maxit);
  st.status = maxit >= 1 ? kRunning : kMaxit;
  *h_st_ = st;
  GNW_CUDA_CHECK(cudaMemcpyAsync(st_, h_st_, sizeof(MinresState), cudaMemcpyHostToDevice, s));
  const bool host_loop = no_graph_ || comm_ != nullptr;  // partitioned: exchanges between the phases
  auto ensure_graph = [&]() -> cudaGraphExec_t {
    const int slot = loop_sched();
    if (!graph_exec_[slot]) {
      build_graph();
      built_now += graph_nodes_[slot];
    }
    return graph_exec_[slot];
  };
  // the persistent kernel replaces the graph loop while the fast schedules are active
  uint64_t persist_iters = 0;
  auto run_persistent = [&]() -> bool {
    if (!persistent_eligible()) return false;
    PersistArgs a;
    if (!damg_.fill_persist(a)) return false;
    const int nb = sm_count_;
    if (ppart_ == nullptr || ppart_m_ < static_cast<int>(m_)) {
      ppart_ = mem_.alloc<double>(static_cast<size_t>(nb) * 8);
      ptpart_ = mem_.alloc<double>(static_cast<size_t>(nb) * static_cast<size_t>(persistent_max_m()));
      pbar_ = mem_.alloc<unsigned>(64);  // arrival counter and released epoch
      ppart_m_ = persistent_max_m();
    }
    a.op = op_;
    a.K = K_;
    a.N = N_;
    a.m = static_cast<int>(m_);
    a.qinv = pa_.qinv;
    a.Ht = pa_.Ht;
    a.ldh = pa_.ldh;
    a.J = dJ_;
    a.ldj = ldj_;
    a.Cinv = pa_.Cinv;
    a.Cfull = dC_;
    a.neg_inv_beta = pa_.neg_inv_beta;
    for (int k = 0; k < 3; ++k) {
      a.V[k] = V_[k];
      a.W[k] = W_[k];
      a.U[k] = U_[k];
    }
    a.Z[0] = Z_[0];
    a.Z[1] = Z_[1];
    a.az = az_;
    a.x = x_;
    a.r = r_;
    a.bq = bq_;
    a.dq = dq_;
    a.st = st_;
    a.hist_e = hist_e_;
    a.hist_p = hist_p_;
    a.hist_cap = hist_cap_;
    a.part = ppart_;
    a.tpart = ptpart_;
    a.bar = pbar_;
    a.max_iters = 1 << 20;
    static const bool prof = [] {  // env GNW_PERSIST_PROFILE=1: phase times of CTA 0 on stderr
      const char* e = std::getenv("GNW_PERSIST_PROFILE");
      return e && std::atoi(e) != 0;
    }();
    if (!prof) return launch_minres_persistent(a, sm_count_, s);
    unsigned long long* dprof = nullptr;
    GNW_CUDA_CHECK(cudaMalloc(&dprof, 8 * sizeof(unsigned long long)));
    GNW_CUDA_CHECK(cudaMemsetAsync(dprof, 0, 8 * sizeof(unsigned long long), s));
    a.prof = dprof;
    const bool ok = launch_minres_persistent(a, sm_count_, s);
    unsigned long long hp[8];
    GNW_CUDA_CHECK(cudaMemcpyAsync(hp, dprof, sizeof hp, cudaMemcpyDeviceToHost, s));
    sync();
    cudaFree(dprof);
    std::fprintf(stderr, "[gnw persistent] ns per phase (whole launch): B %llu, C %llu, restrict %llu, dense %llu, up+dots %llu, "
                         "F+A %llu, tail %llu\n", hp[0], hp[1], hp[2], hp[3], hp[4], hp[5], hp[6]);
    return ok;
  };
  if (!host_loop && !persistent_eligible()) ensure_graph();
  std::vector<std::pair<uint64_t, double>> overrides;  // verified residuals replace recurred ones
  auto true_residual_rel = [&](double* rout) {
    operator_into(vfixed(x_), 0, vfixed(tmp2_), st_plain_, 0);
    residual(n, b_, tmp2_, rout, st_plain_, 0, rpart_, counters_ + 5, s);
    if (comm_) reduce_scratch(st_plain_, 4, 1);
    const MinresState q = read_plain();
    return std::sqrt(q.scratch[4]) / bnorm;
  };
  bool done = false;
  while (!done) {
    MinresState cur;
    if (h_st_->status == kRunning && host_loop) {  // host-driven loop (profiling, partitioned): one sync per iteration
      host_j_ = h_st_->j;
      ++sched_iters[loop_sched()];
      launch_iteration(0, 0);
      GNW_CUDA_CHECK(cudaMemcpyAsync(h_st_, st_, sizeof(MinresState), cudaMemcpyDeviceToHost, s));
      sync();
      if (h_st_->status == kRunning) continue;
    } else if (h_st_->status == kRunning && run_persistent()) {
      const long long it0 = h_st_->iterations;
      GNW_CUDA_CHECK(cudaMemcpyAsync(h_st_, st_, sizeof(MinresState), cudaMemcpyDeviceToHost, s));
      sync();
      const uint64_t done_now = static_cast<uint64_t>(h_st_->iterations - it0);
      persist_iters += done_now;
      sched_iters[2] += done_now;  // the lean schedule's arithmetic
    } else if (h_st_->status == kRunning) {
      const long long it0 = h_st_->iterations;
      const cudaGraphExec_t ge = ensure_graph();
      const uint64_t nodes = graph_nodes_[loop_sched()];
      GNW_CUDA_CHECK(cudaGraphLaunch(ge, s));
      GNW_CUDA_CHECK(cudaMemcpyAsync(h_st_, st_, sizeof(MinresState), cudaMemcpyDeviceToHost, s));
      sync();
      graph_launched += static_cast<uint64_t>(h_st_->iterations - it0) * nodes;  // direct launches count as issued
      sched_iters[loop_sched()] += static_cast<uint64_t>(h_st_->iterations - it0);
    }
    cur = *h_st_;
    switch (cur.status) {
      case kErrNotPD: throw std::runtime_error("minres: preconditioner is not positive definite");
      case kErrStagnated: throw std::runtime_error("minres: breakdown (stagnated rotation)");
      case kVerify: {  // minres.cpp:108-120: r <- b - A x
        const double rel_true = true_residual_rel(r_);
        overrides.emplace_back(cur.iterations, rel_true);
        if (rel_true <= 10.0 * tol) {
          res.converged = true;
          res.true_rel = rel_true;
          done = true;
          break;
        }
        if (fused_active()) {
          // The fused schedule's A zhat comes from the Woodbury identity, whose rounding
          // grows like 1/beta; when that drift keeps the true residual above 10 tol, the
          // solve restarts from x on the reference schedule (r = b - A x is in r_).
          fused_off_ = true;
          ++loop_restarts;
          const long long j0 = cur.j + 1;
          double g1 = 0.0, rr = 0.0;
          start_cycle(j0, &g1, &rr);
          if (g1 == 0.0) throw std::runtime_error("minres: breakdown (zero preconditioned residual, nonzero residual)");
          MinresState st2 = cur;  // keeps gamma1, bnorm, tol, exhausted_tol, maxit, iterations
          st2.gamma_prev = 1.0;
          st2.gamma_cur = g1;
          st2.c_prev = st2.c_cur = 1.0;
          st2.s_prev = st2.s_cur = 0.0;
          st2.eta = g1;
          st2.inv_gamma = 1.0 / g1;
          st2.j = j0;
          st2.status = j0 > st2.maxit ? kMaxit : kRunning;
          *h_st_ = st2;
          GNW_CUDA_CHECK(cudaMemcpyAsync(st_, h_st_, sizeof(MinresState), cudaMemcpyHostToDevice, s));
          break;
        }
        if (cur.gamma_next <= cur.exhausted_tol) {
          h_st_->status = kExhausted;
          continue;
        }
        minres_rotate(st_, s);
        GNW_CUDA_CHECK(cudaMemcpyAsync(h_st_, st_, sizeof(MinresState), cudaMemcpyDeviceToHost, s));
        sync();
        break;
      }
      case kExhausted: {  // minres.cpp:122-133
        const double rel_true = true_residual_rel(tmp_);
        res.true_rel = rel_true;
        if (rel_true <= 10.0 * tol) {
          res.converged = true;
          done = true;
          break;
        }
        throw std::runtime_error("minres: breakdown (Krylov space exhausted before convergence)");
      }
      case kMaxit: {  // minres.cpp:150-154
        res.true_rel = true_residual_rel(tmp_);
        res.converged = false;
        done = true;
        break;
      }
      default: throw DeviceError("minres: unexpected device status");
    }
  }
  res.iterations = static_cast<uint64_t>(h_st_->iterations);
  last_iterations = res.iterations;
  for (int k = 0; k < 3; ++k) last_sched_iters_[k] = std::min<uint64_t>(sched_iters[k], res.iterations);
  last_fused_iters_ = last_sched_iters_[1] + last_sched_iters_[2];
  last_persist_iters_ = std::min<uint64_t>(persist_iters, res.iterations);
  const uint64_t nh = std::min<uint64_t>(res.iterations + 1, static_cast<uint64_t>(hist_cap_));
  std::vector<double> he(nh), hp(nh);
  GNW_CUDA_CHECK(cudaMemcpyAsync(he.data(), hist_e_, nh * sizeof(double), cudaMemcpyDeviceToHost, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(hp.data(), hist_p_, nh * sizeof(double), cudaMemcpyDeviceToHost, s));
  sync();
  for (uint64_t k = 1; k < nh; ++k) {
    res.hist_e.push_back(he[k]);
    res.hist_p.push_back(hp[k]);
  }
  for (auto& ov : overrides)
    if (ov.first < res.hist_e.size()) res.hist_e[ov.first] = ov.second;
  finish();
  return res;
}

void Context::get_woodbury(double* H, double* L) {
  require_device();
  if (comm_) throw std::invalid_argument("get_woodbury: H is partitioned across ranks");
  if (m_ == 0 || pa_.m == 0) return;
  if (H) {
    std::vector<double> ht(static_cast<size_t>(m_) * N_);
    GNW_CUDA_CHECK(cudaMemcpy2D(ht.data(), N_ * sizeof(double), dHt_, ldh_ * sizeof(double), N_ * sizeof(double), m_,
                                cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < m_; ++i)
      for (int64_t c = 0; c < N_; ++c) H[c * m_ + i] = ht[i * N_ + c];
  }
  if (L) GNW_CUDA_CHECK(cudaMemcpy(L, dL_, m_ * m_ * sizeof(double), cudaMemcpyDeviceToHost));
}

void Context::event_record(int slot) {
  require_device();
  if (slot < 0 || slot >= 16) throw std::invalid_argument("gnw_event_record: slot out of range");
  if (!events_[slot]) GNW_CUDA_CHECK(cudaEventCreate(&events_[slot]));
  GNW_CUDA_CHECK(cudaEventRecord(events_[slot], stream_));
}

double Context::event_elapsed(int a, int b) {
  require_device();
  if (a < 0 || a >= 16 || b < 0 || b >= 16 || !events_[a] || !events_[b])
    throw std::invalid_argument("gnw_event_elapsed: slot not recorded");
  GNW_CUDA_CHECK(cudaEventSynchronize(events_[b]));
  float ms = 0.f;
  GNW_CUDA_CHECK(cudaEventElapsedTime(&ms, events_[a], events_[b]));
  return ms * 1e-3;
}

// B_V, the algorithmic bytes of one single-RHS V-cycle
double Context::vcycle_bytes() const {
  double bv = 0.0;
  const size_t L = amg_.levels.size();
  for (size_t l = 0; l + 1 < L; ++l) {
    const double n = static_cast<double>(amg_.levels[l].A.n_rows);
    const double nA = static_cast<double>(amg_.levels[l].A.nnz()), nP = static_cast<double>(amg_.levels[l].P.nnz());
    bv += 2 * (12 * nA + 4 * (n + 1)) + 2 * (12 * nP + 4 * (n + 1)) + 16 * n + 48 * n;
  }
  const double nl = static_cast<double>(amg_.nc);
  return bv + 8 * nl * nl + 32 * nl;
}

// Algorithmic traffic per launch (SURVEY.md 8(d) conventions) and isolated timing.
void Context::profile_kernel(int kernel, int reps, double* seconds, double* algorithmic) {
  require_mixed();
  require_device();
  if (comm_) throw std::invalid_argument("gnw_profile_kernel: single GPU only");
  if (reps < 1) reps = 1;
  const cudaStream_t s = stream_;
  const double K = static_cast<double>(K_), N = static_cast<double>(N_), m = static_cast<double>(m_);
  const double nnzQ = static_cast<double>(Q_.nnz()), nnzD = static_cast<double>(D_.nnz());
  const double bv = vcycle_bytes();  // B_V
  const double hm = (pa_.m > 0) ? m : 0.0;  // H present (Woodbury)
  double alg = 0.0;
  switch (kernel) {
    case 0: alg = 8 * m * N + 8 * N + 8 * m; break;
    case 1: alg = (12 * nnzQ + 4 * (K + 1)) + (12 * nnzD + 4 * (K + 1)) + (12 * nnzD + 4 * (N + 1)) + 8 * m * N +
                  16 * (K + N) + 8 * m;
      break;
    case 2: alg = 48 * K + 32 * N + 8 * hm * N; break;
    case 3: alg = 8 * hm * N + 24 * N + 8 * hm; break;
    case 4: alg = bv; break;
    case 5: alg = 96 * (K + N); break;
    case 6: alg = 2.0 * m * m * N; break;
    case 9: alg = (12 * nnzQ + 4 * (K + 1)) + (12 * nnzD + 4 * (K + 1)) + (12 * nnzD + 4 * (N + 1)) + 8 * N +
                  16 * (K + N);
      break;
    case 10: alg = 16 * hm * N + 32 * N + 8 * hm; break;
    case 11: alg = 8 * m * N + 24 * N + 8 * m; break;
    case 12: alg = 24 * N; break;
    case 7:
    case 8:
      alg = 16 * m * N + 16 * hm * N + (12 * nnzQ + 4 * (K + 1)) + 2 * (12 * nnzD + 4 * (N + 1)) + bv +
            8 * (20 * (K + N) + K);
      break;
    default: throw std::invalid_argument("gnw_profile_kernel: unknown kernel");
  }
  if (kernel == 7 && last_iterations) {  // schedules: fused skips the J zhat2 sweep; lean also the
    const double it = static_cast<double>(last_iterations);  // H t sweep, for a second V-cycle
    alg -= 8 * m * N * static_cast<double>(last_sched_iters_[1]) / it;
    alg -= 16 * m * N * static_cast<double>(last_sched_iters_[2]) / it;  // lean: one V-cycle too
  }
  *algorithmic = alg;
  if (kernel >= 9 && kernel <= 12 && !(m_ > 0 && pa_.m > 0 && dq_))
    throw std::invalid_argument("gnw_profile_kernel: the fused kernels need a Woodbury Jacobian");
  if (kernel == 7) {
    *seconds = last_iterations ? t_minres / static_cast<double>(last_iterations) : 0.0;
    return;
  }
  if ((kernel == 0 || kernel == 6) && m_ == 0) throw std::invalid_argument("gnw_profile_kernel: no Jacobian set");
  if (kernel == 8) {  // one loop-body graph (no loop control) replayed; env GNW_EXP_SKIP drops parts of it
    if (comm_ || hist_cap_ == 0) throw std::invalid_argument("gnw_profile_kernel: run minres first (single GPU)");
    const char* e = std::getenv("GNW_EXP_SKIP");
    exp_skip_ = e ? std::atoi(e) : 0;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    try {
      GNW_CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      launch_iteration(0, 2);
      GNW_CUDA_CHECK(cudaStreamEndCapture(s, &g));
      GNW_CUDA_CHECK(cudaGraphInstantiate(&ge, g, 0));
    } catch (...) {
      exp_skip_ = 0;
      // leave neither stream capturing and no sticky error behind for the next launch
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        cudaGraph_t dead = nullptr;
        cudaStreamEndCapture(s, &dead);
        if (dead) cudaGraphDestroy(dead);
      }
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      throw;
    }
    exp_skip_ = 0;
    GNW_CUDA_CHECK(cudaGraphLaunch(ge, s));
    sync();
    cudaEvent_t a0, a1;
    GNW_CUDA_CHECK(cudaEventCreate(&a0));
    GNW_CUDA_CHECK(cudaEventCreate(&a1));
    GNW_CUDA_CHECK(cudaEventRecord(a0, s));
    for (int r = 0; r < reps; ++r) GNW_CUDA_CHECK(cudaGraphLaunch(ge, s));
    GNW_CUDA_CHECK(cudaEventRecord(a1, s));
    sync();
    float ms = 0.f;
    GNW_CUDA_CHECK(cudaEventElapsedTime(&ms, a0, a1));
    cudaEventDestroy(a0);
    cudaEventDestroy(a1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    *seconds = ms * 1e-3 / reps;
    return;
  }
  const int64_t n = K_ + N_;
  fill_zero(io_a_, n, s);
  fill_zero(io_b_, n, s);
  fill_zero(io_c_, n, s);
  fill_zero(io_d_, n, s);
  DeviceMemory pm;
  double* part = nullptr;
  DgemmPlan plan{};
  if (kernel == 6) {
    plan = dgemm_plan(static_cast<int>(m_), N_, 0, sm_count_);
    part = pm.alloc<double>(static_cast<size_t>(plan.splits) * plan.npairs * plan.tile * plan.tile + 2 * 4096);
  }
  auto launch = [&]() {
    switch (kernel) {
      case 0: row_gemv(dJ_, static_cast<int>(m_), N_, ldj_, vfixed(io_a_), K_, 0, st_plain_, gpart_, counters_ + 0, u_, plan_, s); break;
      case 1: saddle_operator(op_, vfixed(io_a_), 0, u_ ? u_ : io_d_, vfixed(io_b_), st_plain_, 0, opart_, counters_ + 1, s); break;
      case 2:
        combine_precondition(pa_, vfixed(io_a_), vfixed(io_a_), vfixed(io_a_), vfixed(io_a_), vfixed(io_b_), 0,
                             st_plain_, nullptr, cpart_, tpart_, counters_ + 2, t_, plan_, s);
        break;
      case 3:
        finish_precondition(pa_, svc_, t2_ ? t2_ : io_d_, vfixed(io_a_), vfixed(io_b_), 0, st_plain_, cpart_,
                            n_comb_blocks_, fpart_, counters_ + 3, s);
        break;
      case 4: vcycle(vfixed(io_a_ + K_), io_b_, st_plain_); break;
      case 5:
        minres_update(n, vfixed(io_a_), vfixed(io_a_), vfixed(io_a_), vfixed(io_a_), vfixed(io_b_), vfixed(io_a_),
                      vfixed(io_a_), vfixed(io_c_), io_d_, tmp_, st_plain_, nullptr, nullptr, 0, upart_, counters_ + 4,
                      0, 2, s);
        break;
      case 9: {
        OperatorArgs op = op_;
        op.q = dq_;
        saddle_operator(op, vfixed(io_a_), 0, u_, vfixed(io_b_), st_plain_, 0, opart_, counters_ + 1, s);
        break;
      }
      case 10: {
        PrecArgs pa = pa_;
        pa.J = dJ_;
        pa.q = dq_;
        finish_precondition(pa, svc_, t2_, vfixed(io_a_), vfixed(io_b_), 0, st_plain_, cpart_, n_comb_blocks_, fpart_,
                            counters_ + 3, s);
        break;
      }
      case 11: col_sweep(dJ_, ldj_, t2_, static_cast<int>(m_), N_, dq_, s); break;
      case 12: {
        PrecArgs pa = pa_;
        pa.m = 0;
        finish_precondition(pa, svc_, t2_, vfixed(io_a_), vfixed(io_b_), 0, st_plain_, cpart_, n_comb_blocks_, fpart_,
                            counters_ + 3, s);
        break;
      }
      case 6: capacitance_dgemm(dJ_, ldj_, dHt_ ? dHt_ : dJ_, dHt_ ? ldh_ : ldj_, static_cast<int>(m_), N_, beta_, plan, part, dC_ ? dC_ : io_d_, s); break;
    }
  };
  launch();  // warm-up
  sync();
  cudaEvent_t e0, e1;
  GNW_CUDA_CHECK(cudaEventCreate(&e0));
  GNW_CUDA_CHECK(cudaEventCreate(&e1));
  GNW_CUDA_CHECK(cudaEventRecord(e0, s));
  for (int r = 0; r < reps; ++r) launch();
  GNW_CUDA_CHECK(cudaEventRecord(e1, s));
  sync();
  float ms = 0.f;
  GNW_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *seconds = ms * 1e-3 / reps;
}

void Context::dense_cholesky(int64_t n, const double* C, double* L) {
  require_device();
  DeviceMemory tm;
  double* dC = tm.alloc<double>(n * n);
  double* dL = tm.alloc<double>(n * n);
  double* dW = tm.alloc<double>(n * n);
  h2d(dC, C, n * n, stream_);
  if (coarse_mode == 2)  // single-CTA left-looking variant, kept for cross-checking
    gnw::cholesky(dC, dL, static_cast<int>(n), dflag_, stream_);
  else
    gnw::cholesky_blocked(dC, dW, dL, static_cast<int>(n), dflag_, stream_);
  int fail = 0;
  GNW_CUDA_CHECK(cudaMemcpyAsync(&fail, dflag_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
  GNW_CUDA_CHECK(cudaMemcpyAsync(L, dL, n * n * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  if (fail) throw std::runtime_error("dense_cholesky: matrix not positive definite");
}

}  // namespace gnw
