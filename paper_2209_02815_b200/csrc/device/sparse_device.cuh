// sparse_device.cuh -- device-resident CSR matrices and the sparse building blocks of the
// SA-AMG setup: sparse_matmul (sparse.cpp:118-154), transpose
// (sparse.cpp:97-116), and the level pipeline of amg_setup (amg.cpp:115-187) around the host's
// sequential greedy aggregation.  Every result is bit-identical to the host / reference code:
// the products keep the reference's accumulation order (spgemm.cu), the per-row loops are the
// reference's loops with one thread per row, and the library is built with --fmad=false.
#pragma once

#include <cuda_runtime.h>

#include <utility>
#include <vector>

#include "../host/setup.hpp"
#include "amg_device.cuh"

namespace gnw {

// CSR on the device, stream-ordered allocations (cudaMallocAsync), int64 rowptr like the host.
struct DevCsr {
  long long n_rows = 0, n_cols = 0, nnz = 0;
  long long* rp = nullptr;
  int* col = nullptr;
  double* val = nullptr;
  cudaStream_t s = nullptr;
  DevCsr() = default;
  DevCsr(const DevCsr&) = delete;
  DevCsr& operator=(const DevCsr&) = delete;
  DevCsr(DevCsr&& o) noexcept { *this = std::move(o); }
  DevCsr& operator=(DevCsr&& o) noexcept {
    if (this != &o) {
      release();
      n_rows = o.n_rows, n_cols = o.n_cols, nnz = o.nnz, rp = o.rp, col = o.col, val = o.val, s = o.s;
      o.rp = nullptr, o.col = nullptr, o.val = nullptr, o.nnz = 0;
    }
    return *this;
  }
  ~DevCsr() { release(); }
  void release() {
    if (rp) cudaFreeAsync(rp, s);
    if (col) cudaFreeAsync(col, s);
    if (val) cudaFreeAsync(val, s);
    rp = nullptr, col = nullptr, val = nullptr;
  }
};

// host <-> device through a pinned double buffer (the host matrices live in pageable vectors)
DevCsr dev_upload(const host::Csr& A, cudaStream_t s);
host::Csr dev_download(const DevCsr& A, cudaStream_t s);
void dev_upload_array(void* dst, const void* src, size_t bytes, cudaStream_t s);
void dev_download_array(void* dst, const void* src, size_t bytes, cudaStream_t s);

// C = A B with the reference's accumulation order (spgemm.cu)
DevCsr dev_spgemm(const DevCsr& A, const DevCsr& B, cudaStream_t s);
// A^T with each row's entries in ascending original-row order (sparse.cpp:97-116)
DevCsr dev_transpose(const DevCsr& A, cudaStream_t s);

// The one-pass V-cycle operators of a level (host::FusedCycleOps), device resident
struct DevFusedOps {
  DevCsr S, T, Tt;
};

// amg_setup (amg.cpp:115-187) with the level products, the filtering, the prolongator merge
// and the transposes on the device; the greedy aggregation (amg.cpp:13-68, sequential) runs on
// the host on each level's downloaded matrix.  Bit-identical to host::amg_setup.  When
// `fused` is given, the one-pass V-cycle operators (host::fused_cycle_ops) of the levels above
// the collapsed tail are formed on the device too (reusing the Galerkin product's A P) and
// STAY there: DeviceAmg::upload adopts them and builds their lane-ELL copies on the device.
// Levels with at most `host_rows` rows (env GNW_DEVICE_SETUP_MIN_ROWS, default 100000) are
// finished by host::amg_setup: their expand-sort-compress products are slower than 16 cores.
host::AmgHierarchy device_amg_setup(const host::Csr& S, const host::AmgOptions& o, cudaStream_t s,
                                    std::vector<DevFusedOps>* fused, int collapse_max);
// DCsr (int32 rowptr) owned by `mem` from a DevCsr, whose arrays are adopted (A is left empty)
DCsr adopt_csr(DeviceMemory& mem, DevCsr& A, cudaStream_t s);
// upload_lell on the device: same layout, codes numbered by ascending value bits
DLell build_lell_device(DeviceMemory& mem, const DCsr& A, int G, cudaStream_t s);
// returns the setup's cached stream-ordered blocks to the driver (after the hierarchy is uploaded)
void device_setup_trim();
// assemble_lumped_schur (fem_mixed.cpp:84-94) on the device: D diag(Q)^-1 D^T
host::Csr device_lumped_schur(const host::Csr& Q, const host::Csr& D, cudaStream_t s);

}  // namespace gnw
