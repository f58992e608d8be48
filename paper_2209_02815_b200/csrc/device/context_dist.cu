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

// H = S_hat^-1 J^T (inversion.cpp:107-114), partitioned.  The m rows of J are cut into
// column batches of width b; in round t rank q owns batch k = tP + q.  Per round:
//   1. all-to-all: every rank sends its column slice of each batch's J rows to the batch's
//      owner, which assembles the full rows (interleaved, cells contiguous per rank);
//   2. the owner runs the batched V-cycle on its batch (full N, replicated hierarchy);
//   3. all-to-all back: the owner sends each rank that rank's cells of the H rows.
// So each batch is computed once (t_H / P per rank) and each rank ends with Ht[:, own].
void Context::build_h_partitioned(int b) {
  const cudaStream_t s = stream_;
  const int P = comm_->world, me = comm_->rank;
  const long long Nme = c_hi_ - c_lo_;
  const int m = static_cast<int>(m_);
  const int nb = (m + b - 1) / b;
  const size_t na = static_cast<size_t>(P) * b * Nme, nbuf = static_cast<size_t>(b) * N_;
  if (!a2a_mem_ || a2a_na_ < na || a2a_nb_ < nbuf) {
    a2a_mem_.reset();
    a2a_mem_ = std::make_unique<DeviceMemory>();
    a2a_a_ = a2a_mem_->alloc<double>(na);
    a2a_b_ = a2a_mem_->alloc<double>(nbuf);
    a2a_na_ = na;
    a2a_nb_ = nbuf;
  }
  auto width = [&](int k) { return k < nb ? std::min(b, m - k * b) : 0; };
  auto ncells = [&](int q) { return part_lo_[q + 1] - part_lo_[q]; };
  std::vector<const double*> send(P);
  std::vector<double*> recv(P);
  std::vector<long long> sc(P), rc(P);
  for (int t0 = 0; t0 < nb; t0 += P) {
    const int bm = width(t0 + me);  // my batch this round (0: none)
    // 1. my columns of every batch of the round -> its owner
    for (int q = 0; q < P; ++q) {
      const int bq = width(t0 + q);
      double* chunk = a2a_a_ + static_cast<size_t>(q) * b * Nme;
      if (bq > 0)
        GNW_CUDA_CHECK(cudaMemcpy2DAsync(chunk, Nme * sizeof(double), dJ_ + static_cast<long long>(t0 + q) * b * ldj_,
                                         ldj_ * sizeof(double), Nme * sizeof(double), bq, cudaMemcpyDeviceToDevice, s));
      send[q] = chunk;
      sc[q] = bq * Nme;
      recv[q] = a2a_b_ + static_cast<size_t>(bm) * part_lo_[q];
      rc[q] = bm * ncells(q);
    }
    comm_->alltoallv(send, sc, recv, rc, s);
    if (bm > 0) {
      // 2. full rows of my batch -> interleaved batch, V-cycles, then each rank's cells of H rows
      for (int q = 0; q < P; ++q)
        transpose_rows_to_batch(recv[q], ncells(q), ncells(q), 0, bm, damg_.batch_in() + part_lo_[q] * bm, s);
      damg_.vcycle_batch(damg_.batch_in(), bm, damg_.batch_out(), coarse_mode == 1, st_plain_, s);
      for (int q = 0; q < P; ++q)
        transpose_batch_to_rows(damg_.batch_out() + part_lo_[q] * bm, ncells(q), ncells(q), 0, bm, recv[q], s);
    }
    // 3. H rows of every batch of the round, my cells <- the batch's owner
    for (int q = 0; q < P; ++q) {
      send[q] = recv[q];
      sc[q] = bm * ncells(q);
      recv[q] = a2a_a_ + static_cast<size_t>(q) * b * Nme;
      rc[q] = width(t0 + q) * Nme;
    }
    comm_->alltoallv(send, sc, recv, rc, s);
    for (int q = 0; q < P; ++q) {
      const int bq = width(t0 + q);
      if (bq > 0)
        GNW_CUDA_CHECK(cudaMemcpy2DAsync(dHt_ + static_cast<long long>(t0 + q) * b * ldh_, ldh_ * sizeof(double),
                                         recv[q], Nme * sizeof(double), Nme * sizeof(double), bq,
                                         cudaMemcpyDeviceToDevice, s));
    }
  }
}

}  // namespace gnw
