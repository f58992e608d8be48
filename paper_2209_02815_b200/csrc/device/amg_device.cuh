// amg_device.cuh -- a device-resident SA-AMG hierarchy (amg.hpp:25-42) and its
// V-cycles (amg.cpp:90-111): single right-hand side (MINRES loop, graph-safe:
// level-0 input may be a device ring slot) and batched (b interleaved columns,
// per column bit-identical to the single-RHS cycle).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../host/setup.hpp"
#include "kernels.cuh"

namespace gnw {

struct DeviceError : std::runtime_error {
  DeviceError(const char* expr, cudaError_t e, const char* file, int line)
      : std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + expr + " (" + file + ":" +
                           std::to_string(line) + ")") {}
  explicit DeviceError(const std::string& s) : std::runtime_error(s) {}
};

// Device allocations with byte accounting; freed together.
struct DeviceMemory {
  std::vector<void*> ptrs;
  size_t bytes = 0;
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    const size_t nb = std::max<size_t>(count, 1) * sizeof(T);
    GNW_CUDA_CHECK(cudaMalloc(&p, nb));
    ptrs.push_back(p);
    bytes += nb;
    return static_cast<T*>(p);
  }
  void release_all();
  ~DeviceMemory() { release_all(); }
};

DCsr upload_csr(DeviceMemory& mem, const host::Csr& A, cudaStream_t s);
// SELL-32 copy of A (common.cuh); width 0 (nothing allocated) if a row exceeds kSellMaxWidth.
// encode: 0 values as doubles; 1 signs in the columns (all values +-1, else falls back to 2);
// 2 one-byte value codes (at most 256 distinct values, else falls back to 0)
DSell upload_sell(DeviceMemory& mem, const host::Csr& A, cudaStream_t s, int encode = 0);
// lane-ELL copy for G lanes per row with coded values (common.cuh DLell); words == nullptr when
// the padding would be excessive or an entry does not fit 32 bits
DLell upload_lell(DeviceMemory& mem, const host::Csr& A, int G, cudaStream_t s);
// sparse_matmul on the device, bit-identical to host::spgemm (spgemm.cu)
host::Csr device_spgemm(const host::Csr& A, const host::Csr& B, cudaStream_t s);

struct DevFusedOps;  // sparse_device.cuh

class DeviceAmg {
 public:
  // min_collapse_level: the first level the dense collapsed tail may start at (1 for a whole
  // hierarchy; 0 for the replicated tail of a partitioned cycle that starts at the collapse level)
  // fused_dev: the leading levels' one-pass operators where the device setup already formed
  // them; they are adopted (the vector's matrices are left empty)
  void upload(const host::AmgHierarchy& h, cudaStream_t s, int min_collapse_level = 1,
              std::vector<DevFusedOps>* fused_dev = nullptr);
  void reset();
  bool empty() const { return lv_.empty(); }
  int n() const { return lv_.empty() ? 0 : lv_[0].n; }
  size_t bytes() const { return mem_.bytes + (bmem_ ? bmem_->bytes : 0); }

  // z = B r, one V-cycle (exact = the reference's thread-per-row order and Cholesky coarse solve)
  void vcycle(VSel r0, double* out0, const MinresState* st, int exact, cudaStream_t s);
  // b columns interleaved: r0 / out0 are n x b (ld = b)
  // With ht != nullptr the result may instead be stored transposed into Ht rows
  // (ht[q * ldh + i], see mvc2_up2_rows); returns true when it was (out0 untouched).
  bool vcycle_batch(const double* r0, int b, double* out0, int exact, const MinresState* st_plain, cudaStream_t s,
                    double* ht = nullptr, long long ldh = 0);
  void ensure_batch(int b);
  int batch_capacity() const { return bmem_b_; }
  double* batch_in() const { return bR0_; }
  double* batch_out() const { return bX0_; }

  int collapse_level() const { return collapse_l_; }
  // the V-cycle part of the persistent MINRES kernel's arguments (one-pass lane-ELL levels above
  // the dense tail); false when a level has no lane-ELL copy or there are too many levels
  bool fill_persist(struct PersistArgs& a) const;
  bool fused() const { return fused_; }
  // the dense collapsed tail starts at the first level with at most this many rows (env
  // GNW_VC_COLLAPSE_MAX, default 3072); the dense map is L2-resident up to that (72 MB)
  static int collapse_max();

 private:
  DLevel level(int l, int exact) const;
  // Levels [l0, L) of the cycle: r / out live at level l0.  With `collapse`, the levels from
  // collapse_l_ down are replaced by the dense operator collapse_M_ (default mode only).
  void cycle_levels(int l0, VSel r, double* out, const MinresState* st, int exact, bool collapse, cudaStream_t s);
  void build_collapse(cudaStream_t s);
  double* collapse_matrix(int lc, cudaStream_t s);  // the sub-cycle from level lc as one dense matrix

  bool fused_ = false;             // fused per-level operators built (vcycle_fused.cu)
  int min_collapse_ = 1;
  int collapse_l_ = -1;           // first level with n <= kCollapseMax above the coarsest, or -1
  double* collapse_M_ = nullptr;  // n x n row-major: column j = the sub-cycle applied to e_j
  int pstop_ = -1;                // the persistent kernel's deeper tail level (small hierarchies), or -1
  double* pcollapse_M_ = nullptr;
  DeviceMemory mem_;
  std::vector<DLevel> lv_;
  double* coarse_inv_ = nullptr;
  double* coarse_L_ = nullptr;
  int nc_ = 0;
  std::vector<double*> vr_, ve_, vres_, vx_;
  std::unique_ptr<DeviceMemory> bmem_;
  int bmem_b_ = 0;
  std::vector<double*> mr_, me_, mres_, mx_;
  double *bR0_ = nullptr, *bX0_ = nullptr;
};

}  // namespace gnw
