// part_amg.cu -- see part_amg.cuh.
#include "part_amg.cuh"

#include <algorithm>
#include <cstdlib>
#include <stdexcept>

namespace gnw {

void note_launch(const char* what);

namespace {

__global__ void k_gather_rows(const int* __restrict__ idx, long long n, const double* __restrict__ in,
                              double* __restrict__ out, int b) {
  griddep_wait();
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * b) return;
  const long long k = t / b;
  const int q = static_cast<int>(t % b);
  const int i = idx[k];
  out[t] = i >= 0 ? in[static_cast<long long>(i) * b + q] : 0.0;
}

__global__ void k_scatter_rows(const int* __restrict__ idx, long long n, const double* __restrict__ in,
                               double* __restrict__ out, int b) {
  griddep_wait();
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * b) return;
  const long long k = t / b;
  const int i = idx[k];
  if (i >= 0) out[static_cast<long long>(i) * b + t % b] = in[t];
}

__global__ void k_copy_vsel(VSel xs, const MinresState* st, long long n, double* __restrict__ out) {
  griddep_wait();
  const double* __restrict__ x = vsel(xs, st);
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = x[i];
}

unsigned blocks(long long n) { return static_cast<unsigned>(std::max<long long>(1, (n + 255) / 256)); }

}  // namespace

void gather_rows(const int* idx, long long n, const double* in, double* out, int b, cudaStream_t s) {
  if (n <= 0) return;
  GNW_LAUNCH(launch_k(k_gather_rows, blocks(n * b), 256, 0, s, idx, n, in, out, b));
  note_launch("gather_rows");
}
void scatter_rows(const int* idx, long long n, const double* in, double* out, int b, cudaStream_t s) {
  if (n <= 0) return;
  GNW_LAUNCH(launch_k(k_scatter_rows, blocks(n * b), 256, 0, s, idx, n, in, out, b));
  note_launch("scatter_rows");
}

DHalo upload_halo(DeviceMemory& mem, const host::Halo& h, cudaStream_t s) {
  DHalo d;
  d.n_own = h.n_own;
  d.n_local = h.n_local();
  d.n_send = static_cast<long long>(h.send_idx.size());
  d.send_off.assign(h.send_off.begin(), h.send_off.end());
  d.recv_off.assign(h.recv_off.begin(), h.recv_off.end());
  d.send_idx = mem.alloc<int>(std::max<long long>(d.n_send, 1));
  if (d.n_send)
    GNW_CUDA_CHECK(cudaMemcpyAsync(d.send_idx, h.send_idx.data(), d.n_send * sizeof(int), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  return d;
}

CommTally& comm_tally() {
  thread_local CommTally t;  // per rank thread (in-process ranks run one per thread)
  return t;
}

void halo_exchange(Comm& comm, DHalo& h, double* v, int b, DeviceMemory& mem, cudaStream_t s) {
  const int P = comm.world;
  if (P == 1) return;
  comm_tally().calls += 1;
  comm_tally().bytes += 8.0 * static_cast<double>(h.n_send) * b;
  if (b > h.bmax) {  // the pack buffer grows with the widest exchange (the setup's b columns)
    h.sendbuf = mem.alloc<double>(static_cast<size_t>(std::max<long long>(h.n_send, 1)) * b);
    h.bmax = b;
  }
  gather_rows(h.send_idx, h.n_send, v, h.sendbuf, b, s);
  std::vector<const double*> send(P);
  std::vector<double*> recv(P);
  std::vector<long long> sc(P), rc(P);
  for (int q = 0; q < P; ++q) {
    send[q] = h.sendbuf + h.send_off[q] * b;
    sc[q] = (h.send_off[q + 1] - h.send_off[q]) * b;
    recv[q] = v + (h.n_own + h.recv_off[q]) * b;
    rc[q] = (h.recv_off[q + 1] - h.recv_off[q]) * b;
  }
  comm.alltoallv(send, sc, recv, rc, s);
}

void PartAmg::build(const host::AmgHierarchy& h, const std::vector<int32_t>& cell_owner, Comm* comm,
                    long long rows_rep, cudaStream_t s) {
  comm_ = comm;
  const int P = comm->world, me = comm->rank;
  const int L = static_cast<int>(h.levels.size());
  lt_ = L - 1;
  for (int l = 1; l < L; ++l)
    if (h.levels[l].A.n_rows <= rows_rep) {
      lt_ = l;
      break;
    }
  if (L == 1) lt_ = 0;
  // owners of every level down to lt
  std::vector<std::vector<int32_t>> own(lt_ + 1);
  own[0] = cell_owner;
  for (int l = 0; l < lt_; ++l) own[l + 1] = host::coarse_owners(h.levels[l].P, own[l]);
  // the fused operators of the partitioned levels (global, identical on every rank)
  const double omega = h.options.jacobi_damping;
  std::vector<host::FusedCycleOps> ops(lt_);
  for (int l = 0; l < lt_; ++l) {
    std::vector<double> wd(h.levels[l].inv_diag.size());
    for (size_t i = 0; i < wd.size(); ++i) wd[i] = omega * h.levels[l].inv_diag[i];
    ops[l] = host::fused_cycle_ops(h.levels[l].A, h.levels[l].P, wd);
  }
  // halos: level-l space is read by S_l (own l), Tt_l (own l+1) and T_{l-1} (own l-1)
  std::vector<std::vector<host::Halo>> halos(lt_ + 1);
  for (int l = 0; l <= lt_; ++l) {
    std::vector<std::vector<int64_t>> refs(P);
    for (int r = 0; r < P; ++r) {
      if (l < lt_) {
        host::append_refs(ops[l].S, host::owned(own[l], r), refs[r]);
        host::append_refs(ops[l].Tt, host::owned(own[l + 1], r), refs[r]);
      }
      if (l > 0) host::append_refs(ops[l - 1].T, host::owned(own[l - 1], r), refs[r]);
    }
    halos[l] = host::build_halos(own[l], P, refs, me);
  }
  lv_.clear();
  for (int l = 0; l < lt_; ++l) {
    Level v;
    const std::vector<int64_t> mine = host::owned(own[l], me), mine1 = host::owned(own[l + 1], me);
    const host::Halo& H = halos[l][me];
    v.halo = upload_halo(mem_, H, s);
    v.d.n = static_cast<int>(H.n_own);
    const host::Csr lS = host::localize(ops[l].S, mine, H), lT = host::localize(ops[l].T, mine, halos[l + 1][me]),
                    lTt = host::localize(ops[l].Tt, mine1, H);
    v.d.S = upload_csr(mem_, lS, s);
    v.d.T = upload_csr(mem_, lT, s);
    v.d.Tt = upload_csr(mem_, lTt, s);
    v.d.gS = vc_group_lanes(v.d.S.nnz + v.d.T.nnz, std::max(v.d.n, 1));
    v.d.gTt = vc_group_lanes(v.d.Tt.nnz, std::max(v.d.Tt.n_rows, 1));
    // lane-ELL copies with coded entries for the single-RHS level kernels, like the single-GPU
    // hierarchy (same sums in the same order: the partitioned cycle stays bitwise the single-GPU one)
    const char* le = std::getenv("GNW_VC_LELL");
    if (!(le && std::atoi(le) == 0) && lS.n_rows > 0 && lTt.n_rows > 0) {
      v.d.Sl = upload_lell(mem_, lS, v.d.gS, s);
      v.d.Tl = upload_lell(mem_, lT, v.d.gS, s);
      v.d.Ttl = upload_lell(mem_, lTt, v.d.gTt, s);
    }
    v.d.fused = 1;
    v.d.R = v.d.Tt;  // the batched restriction reads R (mvcf_restrict)
    v.r = mem_.alloc<double>(H.n_local());
    v.e = mem_.alloc<double>(H.n_local());
    lv_.push_back(v);
  }
  // replicated tail from level lt: the sub-hierarchy on every rank
  host::AmgHierarchy sub;
  sub.levels.assign(h.levels.begin() + lt_, h.levels.end());
  sub.coarse_chol = h.coarse_chol;
  sub.nc = h.nc;
  sub.options = h.options;
  // the tail collapses where the whole hierarchy's cycle would (DeviceAmg::build_collapse's rule)
  int gc = -1;
  const char* ce = std::getenv("GNW_VC_COLLAPSE");
  if (!(ce && std::atoi(ce) == 0))
    for (int l = 1; l + 1 < L; ++l)
      if (h.levels[l].A.n_rows <= DeviceAmg::collapse_max()) {
        gc = l;
        break;
      }
  tail_.upload(sub, s, gc == lt_ ? 0 : 1);
  const host::Halo& Ht = halos[lt_][me];
  tail_n_ = h.levels[lt_].A.n_rows;
  tail_n_own_ = Ht.n_own;
  tail_nlocal_ = Ht.n_local();
  tail_maxown_ = 0;
  for (int r = 0; r < P; ++r) tail_maxown_ = std::max<long long>(tail_maxown_, halos[lt_][r].n_own);
  std::vector<int> gidx(static_cast<size_t>(P) * tail_maxown_, -1);
  for (int r = 0; r < P; ++r)
    for (long long k = 0; k < halos[lt_][r].n_own; ++k)
      gidx[static_cast<size_t>(r) * tail_maxown_ + k] = static_cast<int>(halos[lt_][r].own_global[k]);
  tail_gidx_n_ = static_cast<long long>(gidx.size());
  tail_gidx_ = mem_.alloc<int>(std::max<long long>(tail_gidx_n_, 1));
  GNW_CUDA_CHECK(cudaMemcpyAsync(tail_gidx_, gidx.data(), gidx.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  std::vector<int> l2g(static_cast<size_t>(tail_nlocal_));
  for (long long k = 0; k < Ht.n_own; ++k) l2g[k] = static_cast<int>(Ht.own_global[k]);
  for (size_t k = 0; k < Ht.ghost_global.size(); ++k) l2g[Ht.n_own + k] = static_cast<int>(Ht.ghost_global[k]);
  tail_l2g_ = mem_.alloc<int>(std::max<long long>(tail_nlocal_, 1));
  if (tail_nlocal_)
    GNW_CUDA_CHECK(cudaMemcpyAsync(tail_l2g_, l2g.data(), l2g.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  tail_r_ = mem_.alloc<double>(std::max<long long>(tail_nlocal_, 1));
  tail_e_ = mem_.alloc<double>(std::max<long long>(tail_nlocal_, 1));
  tail_pad_ = mem_.alloc<double>(std::max<long long>(tail_maxown_, 1));
  tail_gath_ = mem_.alloc<double>(std::max<long long>(P * tail_maxown_, 1));
  tail_rf_ = mem_.alloc<double>(std::max<long long>(tail_n_, 1));
  tail_ef_ = mem_.alloc<double>(std::max<long long>(tail_n_, 1));
  if (!lv_.empty()) r0_ = lv_[0].r;
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
}

void PartAmg::tail_gather(const double* own, int b, double* full, cudaStream_t s) {
  double* pad = b == 1 ? tail_pad_ : btail_pad_;
  double* gath = b == 1 ? tail_gath_ : btail_gath_;
  if (tail_n_own_)
    GNW_CUDA_CHECK(cudaMemcpyAsync(pad, own, tail_n_own_ * b * sizeof(double), cudaMemcpyDeviceToDevice, s));
  comm_->allgather(pad, gath, tail_maxown_ * b, s);
  comm_tally().calls += 1;
  comm_tally().bytes += 8.0 * static_cast<double>(tail_maxown_) * b * comm_->world;
  scatter_rows(tail_gidx_, tail_gidx_n_, gath, full, b, s);  // padding (index -1) is skipped
}

void PartAmg::vcycle(VSel r0, double* out0, const MinresState* st, cudaStream_t s) {
  const int nl = static_cast<int>(lv_.size());
  if (nl == 0) {  // the whole cycle replicated
    GNW_LAUNCH(launch_k(k_copy_vsel, blocks(tail_n_own_), 256, 0, s, r0, st, tail_n_own_, tail_r_));
    tail_gather(tail_r_, 1, tail_rf_, s);
    tail_.vcycle(vfixed(tail_rf_), tail_ef_, st, 0, s);
    gather_rows(tail_l2g_, tail_n_own_, tail_ef_, out0, 1, s);
    return;
  }
  GNW_LAUNCH(launch_k(k_copy_vsel, blocks(lv_[0].halo.n_own), 256, 0, s, r0, st, lv_[0].halo.n_own, r0_));
  for (int l = 0; l < nl; ++l) {
    halo_exchange(*comm_, lv_[l].halo, lv_[l].r, 1, mem_, s);
    vcf_restrict(lv_[l].d, vfixed(lv_[l].r), l + 1 < nl ? lv_[l + 1].r : tail_r_, st, s);
  }
  tail_gather(tail_r_, 1, tail_rf_, s);
  tail_.vcycle(vfixed(tail_rf_), tail_ef_, st, 0, s);
  gather_rows(tail_l2g_, tail_nlocal_, tail_ef_, tail_e_, 1, s);
  for (int l = nl - 1; l >= 0; --l) {
    const double* ec = l + 1 < nl ? lv_[l + 1].e : tail_e_;
    vcf_up(lv_[l].d, vfixed(lv_[l].r), ec, l == 0 ? out0 : lv_[l].e, st, s);
    if (l > 0) halo_exchange(*comm_, lv_[l].halo, lv_[l].e, 1, mem_, s);
  }
}

void PartAmg::ensure_batch(int b) {
  if (bmem_ && bcap_ >= b) return;
  bmem_ = std::make_unique<DeviceMemory>();
  for (Level& v : lv_) {
    v.mr = bmem_->alloc<double>(static_cast<size_t>(v.halo.n_local) * b);
    v.me = bmem_->alloc<double>(static_cast<size_t>(v.halo.n_local) * b);
  }
  const long long P = comm_->world;
  btail_r_ = bmem_->alloc<double>(static_cast<size_t>(std::max<long long>(tail_nlocal_, 1)) * b);
  btail_e_ = bmem_->alloc<double>(static_cast<size_t>(std::max<long long>(tail_nlocal_, 1)) * b);
  btail_pad_ = bmem_->alloc<double>(static_cast<size_t>(std::max<long long>(tail_maxown_, 1)) * b);
  btail_gath_ = bmem_->alloc<double>(static_cast<size_t>(std::max<long long>(P * tail_maxown_, 1)) * b);
  btail_rf_ = bmem_->alloc<double>(static_cast<size_t>(std::max<long long>(tail_n_, 1)) * b);
  btail_ef_ = bmem_->alloc<double>(static_cast<size_t>(std::max<long long>(tail_n_, 1)) * b);
  bcap_ = b;
}

void PartAmg::vcycle_batch(const double* X, int b, double* Y, const MinresState* st_plain, cudaStream_t s) {
  ensure_batch(b);
  const int nl = static_cast<int>(lv_.size());
  if (nl == 0) {
    tail_gather(X, b, btail_rf_, s);
    tail_.vcycle_batch(btail_rf_, b, btail_ef_, 0, st_plain, s);
    gather_rows(tail_l2g_, tail_n_own_, btail_ef_, Y, b, s);
    return;
  }
  GNW_CUDA_CHECK(cudaMemcpyAsync(lv_[0].mr, X, static_cast<size_t>(lv_[0].halo.n_own) * b * sizeof(double),
                                 cudaMemcpyDeviceToDevice, s));
  for (int l = 0; l < nl; ++l) {
    halo_exchange(*comm_, lv_[l].halo, lv_[l].mr, b, mem_, s);
    mvcf_restrict(lv_[l].d, lv_[l].mr, l + 1 < nl ? lv_[l + 1].mr : btail_r_, b, s);
  }
  tail_gather(btail_r_, b, btail_rf_, s);
  tail_.vcycle_batch(btail_rf_, b, btail_ef_, 0, st_plain, s);
  gather_rows(tail_l2g_, tail_nlocal_, btail_ef_, btail_e_, b, s);
  for (int l = nl - 1; l >= 0; --l) {
    const double* ec = l + 1 < nl ? lv_[l + 1].me : btail_e_;
    mvcf_up(lv_[l].d, lv_[l].mr, ec, l == 0 ? Y : lv_[l].me, b, nullptr, 0, s);
    if (l > 0) halo_exchange(*comm_, lv_[l].halo, lv_[l].me, b, mem_, s);
  }
}

}  // namespace gnw
