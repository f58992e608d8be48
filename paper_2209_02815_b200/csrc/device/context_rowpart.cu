// context_rowpart.cu -- the row-partitioned multi-GPU mode of the context (
// BASELINE north_star: "MINRES vectors by mesh rows with NVLink halo exchange and NCCL allreduce
// for the dot products").
//
// Rank r owns a contiguous range of cells (whole mesh rows on a unit square, partition_cells)
// and the edges whose first cell it owns (also contiguous: edges are numbered by first
// encounter, mesh.cpp:116-137).  Its MINRES vectors hold [own edges | own cells | ghosts]; the
// saddle operator's local Q, D, D^T are the global rows with columns mapped to that layout
// (host/partition.hpp), so every row sums exactly the reference's terms in its order.  J and H
// are the m x N_r column slices of the own cells.  Per MINRES iteration the exchanges are:
//   * one halo exchange of zhat (ghost edges and cells: one mesh row) before the operator;
//   * the partitioned V-cycle's halos (part_amg.cuh: two per fine level) and the allgather of
//     the replicated tail's residual;
//   * an allgather + fixed-order sum of the m-partials of H^T v2 (and of J zhat2 on the
//     reference schedule) -- the "capacitance columns by observation" reduction;
//   * packed-scalar reductions: delta, (<z,v>, <z,z>, <v,v>), ||r||^2 -- allgather of the
//     rank partials and a fixed-order sum, so every rank holds the same bits and takes the same
//     control-flow decisions without a broadcast.
// The setup's H = S^-1 J^T runs the partitioned multi-RHS V-cycle on the own columns, and
// C = I + (sum_r J_r H_r^T)/beta sums the ranks' DMMA partials in rank order.
#include "context.cuh"
#include "part_amg.cuh"

namespace gnw {

void Context::set_comm(std::shared_ptr<Comm> c) {
  if (c && c->world < 1) throw std::invalid_argument("partition: world size must be >= 1");
  destroy_graph();
  comm_ = std::move(c);
  assembled_ = false;  // the partition is fixed by the next assemble
  jmem_.reset();
  jm_m_ = -1;
  dJ_ = nullptr;
  m_ = 0;
  pa_.m = 0;
}

void Context::reduce_m(const double* part, double* out, long long n, cudaStream_t s) {
  comm_->allgather(part, gath_, n, s);
  comm_tally().calls += 1;
  comm_tally().bytes += 8.0 * static_cast<double>(n) * comm_->world;
  sum_partials(gath_, comm_->world, n, out, s);
}

void Context::reduce_scratch(MinresState* st, int k0, int cnt) {
  comm_->allgather(st->scratch + k0, sgath_, cnt, stream_);
  comm_tally().calls += 1;
  comm_tally().bytes += 8.0 * cnt * comm_->world;
  sum_scratch(sgath_, comm_->world, cnt, st, k0, stream_);
}

void Context::exchange_saddle(double* v) { halo_exchange(*comm_, *sh_, v, 1, rpmem_, stream_); }

// Partition, halos and local operators (after the replicated host setup of assemble()).
void Context::setup_rowpart() {
  const cudaStream_t s = stream_;
  const int P = comm_->world, me = comm_->rank;
  part_lo_ = partition_cells(N_, P);
  for (int r = 0; r < P; ++r)
    if (part_lo_[r + 1] == part_lo_[r])
      throw std::invalid_argument("partition: a rank would own no cells (fewer than 64 cells per rank)");
  c_lo_ = part_lo_[me];
  c_hi_ = part_lo_[me + 1];
  const host::SaddlePartition sp = host::partition_saddle(mesh_, Q_, D_, part_lo_, me);
  const host::Halo& h = sp.halo;
  const std::vector<int32_t>& cell_own = sp.cell_owner;
  Kl_ = sp.K_l;
  Nl_ = sp.N_l;
  nloc_ = h.n_local();
  part_e_ = sp.edge_lo;
  e_lo_ = part_e_[me];
  e_hi_ = part_e_[me + 1];
  rpmem_.release_all();
  sh_ = std::make_unique<DHalo>(upload_halo(rpmem_, h, s));
  op_ = OperatorArgs{};
  op_.Q = upload_csr(mem_, sp.Q, s);
  op_.D = upload_csr(mem_, sp.D, s);
  op_.Dt = upload_csr(mem_, sp.Dt, s);
  op_.Qs = upload_sell(mem_, sp.Q, s, 2);
  op_.Ds = upload_sell(mem_, sp.D, s, 1);
  op_.Dts = upload_sell(mem_, sp.Dt, s, 1);
  op_.K = Kl_;
  op_.N = Nl_;
  // local -> global maps: the saddle layout (own + ghosts) and the cell vector of the rhs
  std::vector<int> l2g(static_cast<size_t>(nloc_)), cell_l2g(static_cast<size_t>(Nl_ + nloc_ - Kl_ - Nl_));
  for (long long k = 0; k < h.n_own; ++k) l2g[k] = static_cast<int>(h.own_global[k]);
  for (size_t k = 0; k < h.ghost_global.size(); ++k) l2g[h.n_own + k] = static_cast<int>(h.ghost_global[k]);
  for (long long j = 0; j < Nl_; ++j) cell_l2g[j] = static_cast<int>(c_lo_ + j);
  for (size_t k = 0; k < h.ghost_global.size(); ++k)
    cell_l2g[Nl_ + k] = h.ghost_global[k] >= K_ ? static_cast<int>(h.ghost_global[k] - K_) : -1;
  sad_l2g_ = rpmem_.alloc<int>(l2g.size());
  cell_l2g_ = rpmem_.alloc<int>(std::max<size_t>(cell_l2g.size(), 1));
  n_cell_l2g_ = static_cast<long long>(cell_l2g.size());
  GNW_CUDA_CHECK(cudaMemcpyAsync(sad_l2g_, l2g.data(), l2g.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(cell_l2g_, cell_l2g.data(), cell_l2g.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  // own-edge 1/diag(Q)
  std::vector<double> qd = host::diagonal(Q_);
  std::vector<double> qinv(static_cast<size_t>(Kl_));
  for (long long k = 0; k < Kl_; ++k) qinv[k] = 1.0 / qd[e_lo_ + k];  // inversion.cpp:210-211
  dnib_ = mem_.alloc<double>(1);
  op_.neg_inv_beta = dnib_;
  pa_ = PrecArgs{};
  double* dq = mem_.alloc<double>(std::max<long long>(Kl_, 1));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dq, qinv.data(), qinv.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  pa_.qinv = dq;
  pa_.K = Kl_;
  pa_.N = Nl_;
  pa_.neg_inv_beta = dnib_;
  alloc_vectors(nloc_, Kl_, Nl_);
  // global-size staging for the public entry points (global vectors in and out)
  gio_a_ = rpmem_.alloc<double>(K_ + N_);
  gio_b_ = rpmem_.alloc<double>(K_ + N_);
  gio_c_ = rpmem_.alloc<double>(std::max<long long>(N_, 1));
  gio_d_ = rpmem_.alloc<double>(std::max<long long>(N_, 1));
  sgath_ = rpmem_.alloc<double>(static_cast<size_t>(P) * 8);
  gath_ = rpmem_.alloc<double>(static_cast<size_t>(P) * 16);
  gath_cap_ = 16;
  // the partitioned V-cycle (level 0 = cells, same owners)
  long long rows_rep = 32768;
  if (const char* e = std::getenv("GNW_PART_REPLICATE_ROWS")) rows_rep = std::atoll(e);
  pamg_ = std::make_unique<PartAmg>();
  pamg_->build(amg_, cell_own, comm_.get(), rows_rep, s);
  svc_ = mem_.alloc<double>(std::max<long long>(Nl_, 1));
  fork_ = false;  // the exchanges run on the main stream
  sync();
}

// global vector (device) -> this rank's local saddle layout: own entries and, when `ghosts`,
// the ghost entries too (read straight from the global input: no exchange needed)
void Context::global_to_local(const double* g, double* l, bool ghosts) {
  gather_rows(sad_l2g_, ghosts ? nloc_ : Kl_ + Nl_, g, l, 1, stream_);
}

// own entries of a local saddle vector -> the full global vector on every rank
void Context::local_to_global(const double* l, double* g) {
  const cudaStream_t s = stream_;
  if (Kl_) GNW_CUDA_CHECK(cudaMemcpyAsync(g + e_lo_, l, Kl_ * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (Nl_) GNW_CUDA_CHECK(cudaMemcpyAsync(g + K_ + c_lo_, l + Kl_, Nl_ * sizeof(double), cudaMemcpyDeviceToDevice, s));
  const int P = comm_->world;
  std::vector<long long> off(P), cnt(P);
  for (int r = 0; r < P; ++r) {
    off[r] = part_e_[r];
    cnt[r] = part_e_[r + 1] - part_e_[r];
  }
  comm_->allgatherv(g, off, cnt, s);
  for (int r = 0; r < P; ++r) {
    off[r] = K_ + part_lo_[r];
    cnt[r] = part_lo_[r + 1] - part_lo_[r];
  }
  comm_->allgatherv(g, off, cnt, s);
}

// a global input vector of the public API (host or device pointer) on the device
const double* Context::global_in(const double* p, size_t n, double* dev) {
  if (ptr_mode == 1) return p;
  GNW_CUDA_CHECK(cudaMemcpyAsync(dev, p, n * sizeof(double), cudaMemcpyHostToDevice, stream_));
  return dev;
}
void Context::global_out(double* p, const double* dev, size_t n) {
  GNW_CUDA_CHECK(cudaMemcpyAsync(p, dev, n * sizeof(double), ptr_mode == 1 ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 stream_));
  sync();
}

// H = S_hat^-1 J^T on the own cells: the partitioned multi-RHS V-cycle over column batches
void Context::build_h_rowpart() {
  const cudaStream_t s = stream_;
  const int b = static_cast<int>(std::min<int64_t>(64, m_));  // identical on every rank
  if (!hx_ || hx_b_ < b) {
    hx_mem_ = std::make_unique<DeviceMemory>();
    hx_ = hx_mem_->alloc<double>(static_cast<size_t>(std::max<long long>(Nl_, 1)) * b);
    hy_ = hx_mem_->alloc<double>(static_cast<size_t>(std::max<long long>(Nl_, 1)) * b);
    hx_b_ = b;
  }
  for (int64_t i0 = 0; i0 < m_; i0 += b) {
    const int bb = static_cast<int>(std::min<int64_t>(b, m_ - i0));
    transpose_rows_to_batch(dJ_, Nl_, ldj_, static_cast<int>(i0), bb, hx_, s);
    pamg_->vcycle_batch(hx_, bb, hy_, st_plain_, s);
    transpose_batch_to_rows(hy_, Nl_, ldh_, static_cast<int>(i0), bb, dHt_, s);
  }
}

}  // namespace gnw
