// part_amg.cuh -- the row-partitioned pieces of the multi-GPU GN-step solve:
// halo exchanges of partitioned vectors and the partitioned V-cycle.
//
// Layout (host/partition.hpp): a rank's copy of a partitioned vector holds its owned entries
// first, then its ghosts grouped by owning rank.  A halo exchange packs the entries other ranks
// read into one buffer (send lists grouped by destination) and lands every rank's ghosts
// straight in the ghost region (Comm::alltoallv: NCCL send/recv over NVLink, or device copies
// between in-process ranks).
//
// The V-cycle (amg.cpp:90-111, the one-pass-per-level form of vcycle_fused.cu) runs the fine
// levels on owned rows with one halo exchange per level on the way down (r_l, read by
// T_l^T and S_l) and one on the way up (e_{l+1}, read by T_l).  From the first level with at
// most `rows_rep` rows the rest of the cycle is replicated: the level's residual is allgathered
// (padded per rank, scattered to global order), every rank runs the same single-GPU tail
// (DeviceAmg on the sub-hierarchy: fused levels, collapsed dense map) and keeps the entries it
// owns or reads.  Every rank computes the same tail bits.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "../host/partition.hpp"
#include "amg_device.cuh"
#include "comm.cuh"

namespace gnw {

struct DHalo {
  long long n_own = 0, n_local = 0;
  int* send_idx = nullptr;  // device
  long long n_send = 0;
  std::vector<long long> send_off, recv_off;  // host, P + 1
  double* sendbuf = nullptr;                  // device, n_send * bmax
  int bmax = 0;
};

DHalo upload_halo(DeviceMemory& mem, const host::Halo& h, cudaStream_t s);
// ghosts of v (b interleaved columns per entry: v[local * b + q]) from their owners
void halo_exchange(Comm& comm, DHalo& h, double* v, int b, DeviceMemory& mem, cudaStream_t s);
// exchanges issued and bytes sent by this process's partitioned solves (all contexts)
struct CommTally {
  unsigned long long calls = 0;
  double bytes = 0.0;
};
CommTally& comm_tally();
// out[k * b + q] = in[idx[k] * b + q], k < n  (gathers / extractions through an index map)
void gather_rows(const int* idx, long long n, const double* in, double* out, int b, cudaStream_t s);
// out[idx[k] * b + q] = in[k * b + q], k < n
void scatter_rows(const int* idx, long long n, const double* in, double* out, int b, cudaStream_t s);

class PartAmg {
 public:
  // h: the global hierarchy (identical on every rank); cell_owner: level-0 owners.  Levels
  // [0, lt) are partitioned, lt = the first level >= 1 with at most rows_rep rows (or the
  // coarsest), and the cycle from lt on is replicated.
  void build(const host::AmgHierarchy& h, const std::vector<int32_t>& cell_owner, Comm* comm, long long rows_rep,
             cudaStream_t s);
  // out0 (owned level-0 rows) = B r0 (owned rows of r0; ghosts are exchanged here)
  void vcycle(VSel r0, double* out0, const MinresState* st, cudaStream_t s);
  // Y = B X on b interleaved columns (owned rows, ld = b)
  void vcycle_batch(const double* X, int b, double* Y, const MinresState* st_plain, cudaStream_t s);
  long long n_own() const { return lv_.empty() ? tail_n_own_ : lv_[0].halo.n_own; }
  int partitioned_levels() const { return static_cast<int>(lv_.size()); }
  int tail_level() const { return lt_; }
  size_t bytes() const { return mem_.bytes + (bmem_ ? bmem_->bytes : 0) + tail_.bytes(); }
  long long exchanges_per_cycle() const { return 2 * static_cast<long long>(lv_.size()) + 1; }

 private:
  struct Level {
    DLevel d;    // local S (own rows; level-l local columns), T (own rows; level-(l+1) local), Tt (own rows of l+1)
    DHalo halo;  // level-l space
    double *r = nullptr, *e = nullptr;  // single RHS, n_local
    double *mr = nullptr, *me = nullptr;  // b columns, n_local * b
  };
  void ensure_batch(int b);
  void tail_gather(const double* own, int b, double* full, cudaStream_t s);  // -> global order, replicated
  Comm* comm_ = nullptr;
  DeviceMemory mem_;
  std::unique_ptr<DeviceMemory> bmem_;
  int bcap_ = 0;
  std::vector<Level> lv_;
  int lt_ = 0;
  // replicated tail at level lt
  DeviceAmg tail_;
  long long tail_n_ = 0, tail_n_own_ = 0, tail_maxown_ = 0;
  int* tail_gidx_ = nullptr;      // P x maxown: every rank's owned global indices (padded)
  long long tail_gidx_n_ = 0;
  int* tail_l2g_ = nullptr;       // my level-lt local (own + ghost) -> global
  long long tail_nlocal_ = 0;
  double *tail_r_ = nullptr, *tail_e_ = nullptr;       // level lt, single RHS: own (r), local (e)
  double *tail_pad_ = nullptr, *tail_gath_ = nullptr;  // allgather staging
  double *tail_rf_ = nullptr, *tail_ef_ = nullptr;     // full global vectors
  double *btail_r_ = nullptr, *btail_e_ = nullptr, *btail_pad_ = nullptr, *btail_gath_ = nullptr,
         *btail_rf_ = nullptr, *btail_ef_ = nullptr;
  double* r0_ = nullptr;  // level-0 input with ghost space (single RHS)
  double* br0_ = nullptr;
};

}  // namespace gnw
