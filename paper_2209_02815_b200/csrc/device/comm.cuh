// comm.cuh -- the exchange layer of the cell-partitioned (multi-GPU) GN-step solve
// (SURVEY.md 8(e)).
//
// One rank per GPU.  Every rank holds the whole mesh, the sparse operators, the AMG
// hierarchy and the MINRES vectors (replicated, bitwise identical on all ranks); the
// dense m x N operands J and H^T are split by cell columns, rank r owning [lo[r], lo[r+1]).
// Each pass over a dense operand is therefore followed by exactly one exchange:
//
//   * a column-sweep result (J^T u, H t, J^T dg) lives only on the owner of each cell
//     -> in-place allgatherv of the cell slices;
//   * a row-GEMV result (J x, H^T y) is a sum of per-rank partials -> allgather of the
//     m-vector partials, then a fixed-order sum (rank 0, 1, ...) on every rank, so that
//     every rank (and every run) gets the same bits;
//   * the capacitance partials J_r H_r^T (m x m) -> the same allgather + fixed-order sum.
//
// Two implementations of the exchanges, with identical results:
//   * NcclComm: NCCL over NVLink/NVSwitch (ncclAllGather; grouped ncclBroadcast for the
//     variable slices), all on the context's stream; libnccl is opened at run time.
//   * LocalComm: `world` ranks as host threads of ONE process sharing one device; an
//     exchange is a host barrier plus device-to-device copies.  The kernels of different
//     ranks never wait on each other on the device, so one GPU can run a P-rank solve
//     (the test and single-GPU stand-in for P GPUs).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace gnw {

// Contiguous cell ranges, boundaries multiples of 64 cells (16-byte aligned J/H column
// slices, even widths for the DMMA capacitance kernel).  lo has world + 1 entries.
std::vector<long long> partition_cells(long long N, int world);

class Comm {
 public:
  virtual ~Comm() = default;
  int rank = 0, world = 1;
  // in place: rank r's slice buf[off[r], off[r] + cnt[r]) is copied into every rank's buf
  virtual void allgatherv(double* buf, const std::vector<long long>& off, const std::vector<long long>& cnt,
                          cudaStream_t s) = 0;
  // out[r * n, (r + 1) * n) = rank r's in[0, n)
  virtual void allgather(const double* in, double* out, long long n, cudaStream_t s) = 0;
  // personalised exchange: send[q] (scnt[q] doubles) goes to rank q, recv[q] (rcnt[q]) comes from q
  virtual void alltoallv(const std::vector<const double*>& send, const std::vector<long long>& scnt,
                         const std::vector<double*>& recv, const std::vector<long long>& rcnt, cudaStream_t s) = 0;
  virtual const char* kind() const = 0;
};

// Shared state of the in-process ranks.
class LocalHub {
 public:
  explicit LocalHub(int world) : world_(world), ptr_(world, nullptr) {}
  int world() const { return world_; }
  // all ranks arrive; throws if a rank has abandoned the group
  void barrier();
  void abandon();  // a rank failed: wake and fail the others instead of hanging
  std::vector<const double*>& ptrs() { return ptr_; }
  std::vector<std::vector<const double*>>& table() { return table_; }  // [from][to] send pointers

 private:
  int world_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  long long generation_ = 0;
  bool broken_ = false;
  std::vector<const double*> ptr_;
  std::vector<std::vector<const double*>> table_ = std::vector<std::vector<const double*>>(world_, std::vector<const double*>(world_));
};

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalHub> hub, int rank);
  ~LocalComm() override;
  void allgatherv(double* buf, const std::vector<long long>& off, const std::vector<long long>& cnt,
                  cudaStream_t s) override;
  void allgather(const double* in, double* out, long long n, cudaStream_t s) override;
  void alltoallv(const std::vector<const double*>& send, const std::vector<long long>& scnt,
                 const std::vector<double*>& recv, const std::vector<long long>& rcnt, cudaStream_t s) override;
  const char* kind() const override { return "local"; }
  LocalHub& hub() { return *hub_; }

 private:
  std::shared_ptr<LocalHub> hub_;
};

class NcclComm final : public Comm {
 public:
  // id: 128-byte ncclUniqueId from nccl_unique_id() on one rank, shared by the caller
  NcclComm(const unsigned char* id, int rank, int world, int device);
  ~NcclComm() override;
  void allgatherv(double* buf, const std::vector<long long>& off, const std::vector<long long>& cnt,
                  cudaStream_t s) override;
  void allgather(const double* in, double* out, long long n, cudaStream_t s) override;
  void alltoallv(const std::vector<const double*>& send, const std::vector<long long>& scnt,
                 const std::vector<double*>& recv, const std::vector<long long>& rcnt, cudaStream_t s) override;
  const char* kind() const override { return "nccl"; }

 private:
  void* comm_ = nullptr;  // ncclComm_t
};

// 128-byte ncclUniqueId (rank 0 creates it; the caller broadcasts it, e.g. over torch.distributed)
void nccl_unique_id(unsigned char out[128]);
bool nccl_available(std::string* why);

}  // namespace gnw
