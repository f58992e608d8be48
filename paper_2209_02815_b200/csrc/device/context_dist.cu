// context_dist.cu -- the cell-partitioned (multi-GPU) mode of the context (comm.cuh).
//
// Per MINRES iteration the partitioned context runs the same kernels as one GPU, plus:
//   J x    : row GEMV over the own column slice -> m-partial -> allgather + fixed-order sum
//   J^T u  : column sweep over the own cells inside k_saddle -> allgatherv of the cell part
//   delta  : k_dist_delta over the (now complete, replicated) vectors
//   H^T y  : as J x;  H t: own cells inside k_finish_prec -> allgatherv;  Givens: k_dist_givens
// so every rank holds bitwise-identical MINRES vectors and scalars, and takes the same
// control-flow decisions (verification, exhaustion, maxit) without a scalar broadcast.
#include "context.cuh"

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

void Context::gather_cells(double* full, cudaStream_t s) {
  const int P = comm_->world;
  std::vector<long long> off(P), cnt(P);
  for (int r = 0; r < P; ++r) {
    off[r] = K_ + part_lo_[r];
    cnt[r] = part_lo_[r + 1] - part_lo_[r];
  }
  comm_->allgatherv(full, off, cnt, s);
}

void Context::reduce_m(const double* part, double* out, long long n, cudaStream_t s) {
  comm_->allgather(part, gath_, n, s);
  sum_partials(gath_, comm_->world, n, out, s);
}

}  // namespace gnw
