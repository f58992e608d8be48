// kernels.cu -- gnw device kernels (sm_100a, FP64).  See kernels.cuh.
//
// Bit-exactness notes (compiled with --fmad=false):
//  * sparse row sums run one thread per row in CSR column order, starting from
//    0.0, so they round exactly like spmv_add (sparse.cpp:73-83);
//  * restriction gathers through R = P^T whose rows list fine indices in
//    ascending order: the same additions as spmv_transpose's scatter
//    (sparse.cpp:85-95; adding a zero product never changes a sum that
//    started at +0.0, so the reference's zero-skip is immaterial);
//  * J^T u, H t, the rhs and all vector recurrences use the reference's
//    per-element operation order (linalg.cpp:33-54, minres.cpp:11-16).
// Reductions (dots, J x, H^T y) are deterministic fixed-order trees, not the
// reference's sequential sums.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <mutex>
#include <set>
#include <string>

#include "kernels.cuh"
#include "minres_scalars.cuh"

namespace gnw {

namespace {

// Column sweeps (J^T u, H t): loads in flight per thread.  One thread per column walks all m
// rows.  Batch = loads in flight per thread: 8 keeps k_finish_prec at 32 registers (8 CTAs
// per SM) for small m; at large m the t staging (30 KB smem at m = 3780) caps residency at
// 6-7 CTAs per SM anyway and a batch of 16 carries the bytes in flight (C5 shapes:
// 5.96 -> 7.08 TB/s; C2 with 16: 6.31 -> 6.05 TB/s, hence the switch).
constexpr int kSweepBatchWideM = 1024;

// Eight strided 8-byte loads issued back to back as one asm statement, so all eight
// results are live at once (ptxas would otherwise interleave them with the add chain and
// keep only ~4 in flight).
__device__ __forceinline__ void ld8_strided(double* v, const double* p, long long stride_bytes) {
  asm volatile(
      "{\n\t.reg .u64 a;\n\t"
      "mov.u64 a, %8;\n\t"
      "ld.global.nc.f64 %0, [a];\n\tadd.u64 a, a, %9;\n\t"
      "ld.global.nc.f64 %1, [a];\n\tadd.u64 a, a, %9;\n\t"
      "ld.global.nc.f64 %2, [a];\n\tadd.u64 a, a, %9;\n\t"
      "ld.global.nc.f64 %3, [a];\n\tadd.u64 a, a, %9;\n\t"
      "ld.global.nc.f64 %4, [a];\n\tadd.u64 a, a, %9;\n\t"
      "ld.global.nc.f64 %5, [a];\n\tadd.u64 a, a, %9;\n\t"
      "ld.global.nc.f64 %6, [a];\n\tadd.u64 a, a, %9;\n\t"
      "ld.global.nc.f64 %7, [a];\n\t}"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
      : "l"(p), "l"(stride_bytes));
}

// Sixteen at once: ptxas may schedule adds between two 8-load statements (the adds wait for
// the first eight), so a 16-deep batch needs one statement.
__device__ __forceinline__ void ld16_strided(double* v, const double* p, long long stride_bytes) {
  asm volatile(
      "{\n\t.reg .u64 a;\n\t"
      "mov.u64 a, %16;\n\t"
      "ld.global.nc.f64 %0, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %1, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %2, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %3, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %4, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %5, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %6, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %7, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %8, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %9, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %10, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %11, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %12, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %13, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %14, [a];\n\tadd.u64 a, a, %17;\n\t"
      "ld.global.nc.f64 %15, [a];\n\t}"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7]),
        "=d"(v[8]), "=d"(v[9]), "=d"(v[10]), "=d"(v[11]), "=d"(v[12]), "=d"(v[13]), "=d"(v[14]), "=d"(v[15])
      : "l"(p), "l"(stride_bytes));
}

// sum_{i < m} p[i * ld] * s[i], accumulated in ascending i (the reference's matvec order):
// the loads of a batch are issued before its sequential adds, so every thread keeps
// kSweepBatch 8-byte loads in flight.
template <int B>
__device__ __forceinline__ double col_dot(const double* __restrict__ p, long long ld, const double* s, int m) {
  static_assert(B % 8 == 0, "batch is a multiple of 8");
  double acc = 0.0;
  int i = 0;
  for (; i + B <= m; i += B) {
    double v[B];
    if constexpr (B % 16 == 0) {
#pragma unroll
      for (int k = 0; k < B; k += 16) ld16_strided(v + k, p + static_cast<long long>(i + k) * ld, ld * 8);
    } else {
#pragma unroll
      for (int k = 0; k < B; k += 8) ld8_strided(v + k, p + static_cast<long long>(i + k) * ld, ld * 8);
    }
#pragma unroll
    for (int k = 0; k < B; ++k) acc = acc + v[k] * s[i + k];
  }
  for (; i < m; ++i) acc = acc + __ldg(p + static_cast<long long>(i) * ld) * s[i];
  return acc;
}
// Two column dots over the same s in one sweep (fused loop: w = (H t')_c and q_c = (J^T t')_c),
// each in ascending i; the batch's loads of both columns are issued before the adds.
template <int B>
__device__ __forceinline__ void col_dot2(const double* __restrict__ p, long long ldp, const double* __restrict__ r,
                                         long long ldr, const double* s, int m, double& accp, double& accr) {
  static_assert(B % 8 == 0, "batch is a multiple of 8");
  double ap = 0.0, ar = 0.0;
  int i = 0;
  for (; i + B <= m; i += B) {
    double v[B], w[B];
    if constexpr (B % 16 == 0) {
#pragma unroll
      for (int k = 0; k < B; k += 16) {
        ld16_strided(v + k, p + static_cast<long long>(i + k) * ldp, ldp * 8);
        ld16_strided(w + k, r + static_cast<long long>(i + k) * ldr, ldr * 8);
      }
    } else {
#pragma unroll
      for (int k = 0; k < B; k += 8) {
        ld8_strided(v + k, p + static_cast<long long>(i + k) * ldp, ldp * 8);
        ld8_strided(w + k, r + static_cast<long long>(i + k) * ldr, ldr * 8);
      }
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      ap = ap + v[k] * s[i + k];
      ar = ar + w[k] * s[i + k];
    }
  }
  for (; i < m; ++i) {
    ap = ap + __ldg(p + static_cast<long long>(i) * ldp) * s[i];
    ar = ar + __ldg(r + static_cast<long long>(i) * ldr) * s[i];
  }
  accp = ap;
  accr = ar;
}

constexpr int kTpb = 256;

inline unsigned grid_for(long long n, int tpb = kTpb) {
  return static_cast<unsigned>((n + tpb - 1) / tpb);
}

std::atomic<uint64_t> g_launches{0};

inline void check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch failed (") + what + "): " + cudaGetErrorString(e));
}

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

}  // namespace

uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

void smem_optin(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;  // (kernel, device)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (e == cudaSuccess && done.count({fn, dev})) return;
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch failed: ") + cudaGetErrorString(e));
  done.insert({fn, dev});
}

bool g_pdl = [] {
  const char* e = std::getenv("GNW_PDL");
  return e == nullptr || std::atoi(e) != 0;
}();

// ======================================================================
// V-cycle, single right-hand side (amg.cpp:90-111)
// ======================================================================

// resid = r - A (wd .* r)        amg.cpp:98-101
__global__ void __launch_bounds__(kTpb) k_vc_down(DCsr A, const double* __restrict__ wd, VSel rs,
                                                  double* __restrict__ resid, const MinresState* st) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_rows) return;
  double s = 0.0;
  const int k1 = A.rowptr[i + 1];
#pragma unroll 4
  for (int k = A.rowptr[i]; k < k1; ++k) {
    const int c = __ldg(&A.cols[k]);
    s = s + ldg(&A.vals[k]) * (ldg(&wd[c]) * r[c]);
  }
  resid[i] = r[i] + (-1.0 * s);
}

// rc = P^T resid (gather through R)        amg.cpp:103
__global__ void __launch_bounds__(kTpb) k_vc_restrict(DCsr R, const double* __restrict__ resid,
                                                      double* __restrict__ rc) {
  griddep_wait();
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= R.n_rows) return;
  double s = 0.0;
  const int k1 = R.rowptr[a + 1];
#pragma unroll 4
  for (int k = R.rowptr[a]; k < k1; ++k) s = s + ldg(&R.vals[k]) * resid[__ldg(&R.cols[k])];
  rc[a] = s;
}

// x = wd .* r + P ec        amg.cpp:98, :105
__global__ void __launch_bounds__(kTpb) k_vc_up1(DCsr P, const double* __restrict__ wd, VSel rs,
                                                 const double* __restrict__ ec, double* __restrict__ x,
                                                 const MinresState* st) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n_rows) return;
  double s = 0.0;
  const int k1 = P.rowptr[i + 1];
#pragma unroll 4
  for (int k = P.rowptr[i]; k < k1; ++k) s = s + ldg(&P.vals[k]) * ec[__ldg(&P.cols[k])];
  x[i] = ldg(&wd[i]) * r[i] + 1.0 * s;
}

// out = x + wd .* (r - A x)        amg.cpp:107-109
__global__ void __launch_bounds__(kTpb) k_vc_up2(DCsr A, const double* __restrict__ wd, VSel rs,
                                                 const double* __restrict__ x, double* __restrict__ out,
                                                 const MinresState* st) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_rows) return;
  double s = 0.0;
  const int k1 = A.rowptr[i + 1];
#pragma unroll 4
  for (int k = A.rowptr[i]; k < k1; ++k) s = s + ldg(&A.vals[k]) * x[__ldg(&A.cols[k])];
  const double res = r[i] + (-1.0 * s);
  out[i] = x[i] + ldg(&wd[i]) * res;
}

// x[:, q] = Ainv r[:, q]; one warp per (row, rhs), lane-strided partials + xor tree
__global__ void k_coarse_inverse(const double* __restrict__ Ainv, int n, VSel rs, double* __restrict__ x,
                                 const MinresState* st, int nrhs) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= static_cast<long long>(n) * nrhs) return;
  const int i = static_cast<int>(w / nrhs), q = static_cast<int>(w % nrhs);
  double acc[1] = {0.0};
  for (int j = lane; j < n; j += 32) acc[0] = acc[0] + ldg(&Ainv[static_cast<long long>(i) * n + j]) * r[static_cast<long long>(j) * nrhs + q];
  warp_reduce<1>(acc);
  if (lane == 0) x[static_cast<long long>(i) * nrhs + q] = acc[0];
}

// Single right-hand side (the MINRES V-cycle's coarse / collapsed-tail apply, C2: n = 1147):
// one 128-thread CTA per row.  Thread t owns columns t, t + 128, ...; the first 16 of its
// matrix entries (all of them for n <= 2048) are loaded BEFORE the grid-dependency wait -- the
// matrix is fixed per hierarchy, so under programmatic dependent launch these loads overlap the
// predecessor's drain -- and the products are added in column order, then lanes (xor tree),
// then the four warps in order.  One warp per row walked 72 dependent loads per lane in
// batches (14.1, later 10.3 us at C2 for a 10.5 MB L2-resident matrix).  Deterministic; not
// the reference order (the reference solves with the Cholesky factor, k_coarse_cholesky, in
// exact mode).
constexpr int kCoarseTpb = 128;
__global__ void __launch_bounds__(kCoarseTpb) k_coarse_inverse1(const double* __restrict__ Ainv, int n, VSel rs,
                                                                double* __restrict__ x, const MinresState* st) {
  const int i = blockIdx.x, t = threadIdx.x;
  const double* __restrict__ row = Ainv + static_cast<long long>(i) * n;
  double mm[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) mm[u] = t + kCoarseTpb * u < n ? ldg(&row[t + kCoarseTpb * u]) : 0.0;
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  double rr[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) rr[u] = t + kCoarseTpb * u < n ? r[t + kCoarseTpb * u] : 0.0;
  double a = 0.0;
#pragma unroll
  for (int u = 0; u < 16; ++u) a = a + mm[u] * rr[u];
  for (int j = t + 16 * kCoarseTpb; j < n; j += kCoarseTpb) a = a + ldg(&row[j]) * r[j];
  double acc[1] = {a};
  warp_reduce<1>(acc);
  __shared__ double part[kCoarseTpb / 32];
  if ((t & 31) == 0) part[t >> 5] = acc[0];
  __syncthreads();
  if (t == 0) x[i] = ((part[0] + part[1]) + part[2]) + part[3];
}

// cholesky_solve (linalg.cpp:107-123) replayed exactly, one thread per rhs column
__global__ void k_coarse_cholesky(const double* __restrict__ L, int n, VSel rs, double* __restrict__ x,
                                  const MinresState* st, int nrhs, int ld) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nrhs) return;
  for (int i = 0; i < n; ++i) x[static_cast<long long>(i) * ld + q] = r[static_cast<long long>(i) * ld + q];
  for (int i = 0; i < n; ++i) {
    double s = x[static_cast<long long>(i) * ld + q];
    for (int k = 0; k < i; ++k) s = s - L[static_cast<long long>(i) * n + k] * x[static_cast<long long>(k) * ld + q];
    x[static_cast<long long>(i) * ld + q] = s / L[static_cast<long long>(i) * n + i];
  }
  for (int ii = n - 1; ii >= 0; --ii) {
    double s = x[static_cast<long long>(ii) * ld + q];
    for (int k = ii + 1; k < n; ++k) s = s - L[static_cast<long long>(k) * n + ii] * x[static_cast<long long>(k) * ld + q];
    x[static_cast<long long>(ii) * ld + q] = s / L[static_cast<long long>(ii) * n + ii];
  }
}

// The same four level kernels on the SELL-32 copies (common.cuh): every entry load of a row
// is issued at once and coalesced across the warp; the row sums add the same terms in the
// same order as the CSR loops above (bit-identical).
template <int W>
__global__ void __launch_bounds__(kTpb) k_vcs_down(DSell A, const double* __restrict__ wd, VSel rs,
                                                   double* __restrict__ resid, const MinresState* st) {
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_rows) return;
  int c[W];
  double v[W];
  sell_load<W>(A, i, c, v);
  const double* __restrict__ r = vsel(rs, st);
  const double s = sell_finish_f<W>(c, v, [&](int j) { return ldg(&wd[j]) * r[j]; });
  resid[i] = r[i] + (-1.0 * s);
}

template <int W>
__global__ void __launch_bounds__(kTpb) k_vcs_restrict(DSell R, const double* __restrict__ resid,
                                                       double* __restrict__ rc) {
  griddep_wait();
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= R.n_rows) return;
  int c[W];
  double v[W];
  sell_load<W>(R, a, c, v);
  rc[a] = sell_finish_f<W>(c, v, [&](int j) { return resid[j]; });
}

template <int W>
__global__ void __launch_bounds__(kTpb) k_vcs_up1(DSell P, const double* __restrict__ wd, VSel rs,
                                                  const double* __restrict__ ec, double* __restrict__ x,
                                                  const MinresState* st) {
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n_rows) return;
  int c[W];
  double v[W];
  sell_load<W>(P, i, c, v);
  const double* __restrict__ r = vsel(rs, st);
  const double s = sell_finish_f<W>(c, v, [&](int j) { return ec[j]; });
  x[i] = ldg(&wd[i]) * r[i] + 1.0 * s;
}

template <int W>
__global__ void __launch_bounds__(kTpb) k_vcs_up2(DSell A, const double* __restrict__ wd, VSel rs,
                                                  const double* __restrict__ x, double* __restrict__ out,
                                                  const MinresState* st) {
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n_rows) return;
  int c[W];
  double v[W];
  sell_load<W>(A, i, c, v);
  const double* __restrict__ r = vsel(rs, st);
  const double s = sell_finish_f<W>(c, v, [&](int j) { return x[j]; });
  const double res = r[i] + (-1.0 * s);
  out[i] = x[i] + ldg(&wd[i]) * res;
}

#define GNW_SELL_SWITCH(width, KER, ...)          \
  switch (width) {                                \
    case 1: KER(1, __VA_ARGS__); break;           \
    case 2: KER(2, __VA_ARGS__); break;           \
    case 3: KER(3, __VA_ARGS__); break;           \
    case 4: KER(4, __VA_ARGS__); break;           \
    case 5: KER(5, __VA_ARGS__); break;           \
    case 6: KER(6, __VA_ARGS__); break;           \
    case 7: KER(7, __VA_ARGS__); break;           \
    default: KER(8, __VA_ARGS__); break;          \
  }
#define GNW_VCS_LAUNCH(W, ker, n, ...) GNW_LAUNCH(launch_k(ker<W>, grid_for(n), kTpb, 0, __VA_ARGS__))

void note_launch(const char* what) { check_launch(what); }

void vc_down(const DLevel& L, VSel r, double* resid, const MinresState* st, cudaStream_t s) {
  if (L.gA > 1) return vcg_down(L, r, resid, st, s);
  if (L.As.width > 0) {
    GNW_SELL_SWITCH(L.As.width, GNW_VCS_LAUNCH, k_vcs_down, L.n, s, L.As, L.wd, r, resid, st);
    return check_launch("vcs_down");
  }
  GNW_LAUNCH(launch_k(k_vc_down, grid_for(L.n), kTpb, 0, s, L.A, L.wd, r, resid, st));
  check_launch("vc_down");
}
void vc_restrict(const DLevel& L, const double* resid, double* rc, cudaStream_t s) {
  if (L.gR > 1) return vcg_restrict(L, resid, rc, s);
  if (L.Rs.width > 0) {
    GNW_SELL_SWITCH(L.Rs.width, GNW_VCS_LAUNCH, k_vcs_restrict, L.R.n_rows, s, L.Rs, resid, rc);
    return check_launch("vcs_restrict");
  }
  GNW_LAUNCH(launch_k(k_vc_restrict, grid_for(L.R.n_rows), kTpb, 0, s, L.R, resid, rc));
  check_launch("vc_restrict");
}
void vc_up1(const DLevel& L, VSel r, const double* ec, double* x, const MinresState* st, cudaStream_t s) {
  if (L.gP > 1) return vcg_up1(L, r, ec, x, st, s);
  if (L.Ps.width > 0) {
    GNW_SELL_SWITCH(L.Ps.width, GNW_VCS_LAUNCH, k_vcs_up1, L.n, s, L.Ps, L.wd, r, ec, x, st);
    return check_launch("vcs_up1");
  }
  GNW_LAUNCH(launch_k(k_vc_up1, grid_for(L.n), kTpb, 0, s, L.P, L.wd, r, ec, x, st));
  check_launch("vc_up1");
}
void vc_up2(const DLevel& L, VSel r, const double* x, double* out, const MinresState* st, cudaStream_t s) {
  if (L.gA > 1) return vcg_up2(L, r, x, out, st, s);
  if (L.As.width > 0) {
    GNW_SELL_SWITCH(L.As.width, GNW_VCS_LAUNCH, k_vcs_up2, L.n, s, L.As, L.wd, r, x, out, st);
    return check_launch("vcs_up2");
  }
  GNW_LAUNCH(launch_k(k_vc_up2, grid_for(L.n), kTpb, 0, s, L.A, L.wd, r, x, out, st));
  check_launch("vc_up2");
}
void coarse_inverse(const double* Ainv, int n, VSel r, double* x, const MinresState* st, int nrhs,
                    cudaStream_t s) {
  const long long threads = static_cast<long long>(n) * nrhs * 32;
  if (nrhs == 1) {
    GNW_LAUNCH(launch_k(k_coarse_inverse1, n, kCoarseTpb, 0, s, Ainv, n, r, x, st));
    return check_launch("coarse_inverse1");
  }
  GNW_LAUNCH(launch_k(k_coarse_inverse, grid_for(threads), kTpb, 0, s, Ainv, n, r, x, st, nrhs));
  check_launch("coarse_inverse");
}
void coarse_cholesky(const double* L, int n, VSel r, double* x, const MinresState* st, int nrhs, int ld,
                     cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_coarse_cholesky, grid_for(nrhs, 64), 64, 0, s, L, n, r, x, st, nrhs, ld));
  check_launch("coarse_cholesky");
}

// ======================================================================
// V-cycle, multiple right-hand sides (X[row * ld + q]); thread (row, q)
// performs exactly the single-RHS operation sequence on column q.
// block = (32 q-lanes, 8 rows); grid = (rows/8, b/32)
// ======================================================================
__global__ void __launch_bounds__(256) k_mvc_down(DCsr A, const double* __restrict__ wd,
                                                  const double* __restrict__ r, int ldr,
                                                  double* __restrict__ resid, int b) {
  griddep_wait();
  const int i = blockIdx.x * 8 + threadIdx.y;
  const int q = blockIdx.y * 32 + threadIdx.x;
  if (i >= A.n_rows || q >= b) return;
  double s = 0.0;
  const int k1 = A.rowptr[i + 1];
  for (int k = A.rowptr[i]; k < k1; ++k) {
    const int c = A.cols[k];
    s = s + ldg(&A.vals[k]) * (ldg(&wd[c]) * r[static_cast<long long>(c) * ldr + q]);
  }
  resid[static_cast<long long>(i) * b + q] = r[static_cast<long long>(i) * ldr + q] + (-1.0 * s);
}

__global__ void __launch_bounds__(256) k_mvc_restrict(DCsr R, const double* __restrict__ resid,
                                                      double* __restrict__ rc, int b) {
  griddep_wait();
  const int a = blockIdx.x * 8 + threadIdx.y;
  const int q = blockIdx.y * 32 + threadIdx.x;
  if (a >= R.n_rows || q >= b) return;
  double s = 0.0;
  const int k1 = R.rowptr[a + 1];
  for (int k = R.rowptr[a]; k < k1; ++k) s = s + ldg(&R.vals[k]) * resid[static_cast<long long>(R.cols[k]) * b + q];
  rc[static_cast<long long>(a) * b + q] = s;
}

__global__ void __launch_bounds__(256) k_mvc_up1(DCsr P, const double* __restrict__ wd,
                                                 const double* __restrict__ r, int ldr,
                                                 const double* __restrict__ ec, double* __restrict__ x, int b) {
  griddep_wait();
  const int i = blockIdx.x * 8 + threadIdx.y;
  const int q = blockIdx.y * 32 + threadIdx.x;
  if (i >= P.n_rows || q >= b) return;
  double s = 0.0;
  const int k1 = P.rowptr[i + 1];
  for (int k = P.rowptr[i]; k < k1; ++k) s = s + ldg(&P.vals[k]) * ec[static_cast<long long>(P.cols[k]) * b + q];
  x[static_cast<long long>(i) * b + q] = ldg(&wd[i]) * r[static_cast<long long>(i) * ldr + q] + 1.0 * s;
}

__global__ void __launch_bounds__(256) k_mvc_up2(DCsr A, const double* __restrict__ wd,
                                                 const double* __restrict__ r, int ldr,
                                                 const double* __restrict__ x, double* __restrict__ out,
                                                 int ldo, int b) {
  griddep_wait();
  const int i = blockIdx.x * 8 + threadIdx.y;
  const int q = blockIdx.y * 32 + threadIdx.x;
  if (i >= A.n_rows || q >= b) return;
  double s = 0.0;
  const int k1 = A.rowptr[i + 1];
  for (int k = A.rowptr[i]; k < k1; ++k) s = s + ldg(&A.vals[k]) * x[static_cast<long long>(A.cols[k]) * b + q];
  const double res = r[static_cast<long long>(i) * ldr + q] + (-1.0 * s);
  out[static_cast<long long>(i) * ldo + q] = x[static_cast<long long>(i) * b + q] + ldg(&wd[i]) * res;
}

void mvc_down(const DLevel& L, const double* r, int ldr, double* resid, int b, cudaStream_t s) {
  if (b % 2 == 0 && ldr % 2 == 0) return mvc2_down(L, r, ldr, resid, b, s);
  dim3 grid((L.n + 7) / 8, (b + 31) / 32), block(32, 8);
  GNW_LAUNCH(launch_k(k_mvc_down, grid, block, 0, s, L.A, L.wd, r, ldr, resid, b));
  check_launch("mvc_down");
}
void mvc_restrict(const DLevel& L, const double* resid, double* rc, int b, cudaStream_t s) {
  if (b % 2 == 0) return mvc2_restrict(L, resid, rc, b, s);
  dim3 grid((L.R.n_rows + 7) / 8, (b + 31) / 32), block(32, 8);
  GNW_LAUNCH(launch_k(k_mvc_restrict, grid, block, 0, s, L.R, resid, rc, b));
  check_launch("mvc_restrict");
}
void mvc_up1(const DLevel& L, const double* r, int ldr, const double* ec, double* x, int b, cudaStream_t s) {
  if (b % 2 == 0 && ldr % 2 == 0) return mvc2_up1(L, r, ldr, ec, x, b, s);
  dim3 grid((L.n + 7) / 8, (b + 31) / 32), block(32, 8);
  GNW_LAUNCH(launch_k(k_mvc_up1, grid, block, 0, s, L.P, L.wd, r, ldr, ec, x, b));
  check_launch("mvc_up1");
}
void mvc_up2(const DLevel& L, const double* r, int ldr, const double* x, double* out, int ldo, int b,
             cudaStream_t s) {
  if (b % 2 == 0 && ldr % 2 == 0 && ldo % 2 == 0) return mvc2_up2(L, r, ldr, x, out, ldo, b, s);
  dim3 grid((L.n + 7) / 8, (b + 31) / 32), block(32, 8);
  GNW_LAUNCH(launch_k(k_mvc_up2, grid, block, 0, s, L.A, L.wd, r, ldr, x, out, ldo, b));
  check_launch("mvc_up2");
}
void mcoarse_inverse(const double* Ainv, int n, const double* r, double* x, int b, cudaStream_t s) {
  const long long threads = static_cast<long long>(n) * b * 32;
  GNW_LAUNCH(launch_k(k_coarse_inverse, grid_for(threads), kTpb, 0, s, Ainv, n, vfixed(const_cast<double*>(r)), x, nullptr, b));
  check_launch("mcoarse_inverse");
}

// rows [r0, r0+b) of A (row-major, `cols` columns) -> X[c * b + q]; and back.  Tiles of
// 32 rows (q) x 64 columns (c): the row side moves 16-byte pairs (512 B per warp row), so
// every thread has 4 x 16 B in flight on that side (the 32 x 32 tiles with 8-byte accesses
// ran at 4.6-4.8 TB/s).  `vec` = both the row stride and the tile start are even.
__global__ void __launch_bounds__(256) k_transpose_rows_to_batch(const double* __restrict__ A, long long cols,
                                                                 long long ld, int r0, int b,
                                                                 double* __restrict__ X) {
  griddep_wait();
  __shared__ double tile[32][65];
  const long long c0 = static_cast<long long>(blockIdx.x) * 64;
  const int q0 = blockIdx.y * 32;
  const bool vec = (ld & 1) == 0;
#pragma unroll
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int q = q0 + y;
    const long long c = c0 + 2 * threadIdx.x;
    double2 v = make_double2(0.0, 0.0);
    if (q < b) {
      const double* row = A + static_cast<long long>(r0 + q) * ld;
      if (vec && c + 1 < cols) {
        v = __ldg(reinterpret_cast<const double2*>(row + c));
      } else {
        if (c < cols) v.x = __ldg(row + c);
        if (c + 1 < cols) v.y = __ldg(row + c + 1);
      }
    }
    tile[y][2 * threadIdx.x] = v.x;
    tile[y][2 * threadIdx.x + 1] = v.y;
  }
  __syncthreads();
#pragma unroll
  for (int y = threadIdx.y; y < 64; y += 8) {
    const long long c = c0 + y;
    const int q = q0 + threadIdx.x;
    if (c < cols && q < b) X[c * b + q] = tile[threadIdx.x][y];
  }
}

__global__ void __launch_bounds__(256) k_transpose_batch_to_rows(const double* __restrict__ X, long long cols,
                                                                 long long ld, int r0, int b,
                                                                 double* __restrict__ A) {
  griddep_wait();
  __shared__ double tile[32][65];
  const long long c0 = static_cast<long long>(blockIdx.x) * 64;
  const int q0 = blockIdx.y * 32;
  const bool vec = (ld & 1) == 0;
#pragma unroll
  for (int y = threadIdx.y; y < 64; y += 8) {
    const long long c = c0 + y;
    const int q = q0 + threadIdx.x;
    tile[threadIdx.x][y] = (c < cols && q < b) ? X[c * b + q] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int q = q0 + y;
    const long long c = c0 + 2 * threadIdx.x;
    if (q >= b) continue;
    double* row = A + static_cast<long long>(r0 + q) * ld;
    const double2 v = make_double2(tile[y][2 * threadIdx.x], tile[y][2 * threadIdx.x + 1]);
    if (vec && c + 1 < cols) {
      *reinterpret_cast<double2*>(row + c) = v;
    } else {
      if (c < cols) row[c] = v.x;
      if (c + 1 < cols) row[c + 1] = v.y;
    }
  }
}

void transpose_rows_to_batch(const double* A, long long cols, long long ld, int r0, int b, double* X,
                             cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((cols + 63) / 64), (b + 31) / 32), block(32, 8);
  GNW_LAUNCH(launch_k(k_transpose_rows_to_batch, grid, block, 0, s, A, cols, ld, r0, b, X));
  check_launch("transpose_rows_to_batch");
}
void transpose_batch_to_rows(const double* X, long long cols, long long ld, int r0, int b, double* A,
                             cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((cols + 63) / 64), (b + 31) / 32), block(32, 8);
  GNW_LAUNCH(launch_k(k_transpose_batch_to_rows, grid, block, 0, s, X, cols, ld, r0, b, A));
  check_launch("transpose_batch_to_rows");
}

// ======================================================================
// Row GEMV with chunked columns: out[i] = sum_c A[i, c] x[c] (deterministic)
// ======================================================================
// One wave, no tail: the grid is (column spans) x (groups of 32 rows) with
// spans x groups = SMs x resident CTAs per SM, each CTA streaming one contiguous
// column span of its 32 rows.  (A 2-D grid of short tiles left a 1.6-wave tail at
// C2 -- 78% of HBM bandwidth; one full wave has no tail.)  x is read through L1:
// the 8 warps of a CTA share each x line.

// R row segments A[row_r, 0 : len] dotted with x[0 : len], one warp, lanes take
// 2-column steps; R independent rows keep R x 2 x 16-byte loads in flight per lane.
template <int R, int U = 4>
__device__ __forceinline__ void warp_rows_dot(const double* __restrict__ a, long long ld, int nrows,
                                              const double* __restrict__ x, int scaled, double sc, int len,
                                              bool vec_ok, int lane, double (&out)[R]) {
  double acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0.0;
  auto xv = [&](int t) { return scaled ? __ldg(x + t) * sc : __ldg(x + t); };
  if (vec_ok) {
    const int len2 = len & ~1;
#pragma unroll U
    for (int t = lane * 2; t < len2; t += 64) {
      const double x0 = xv(t), x1 = xv(t + 1);
      double2 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        v[r] = r < nrows ? __ldg(reinterpret_cast<const double2*>(a + r * ld + t)) : make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc[r] = acc[r] + v[r].x * x0;
        acc[r] = acc[r] + v[r].y * x1;
      }
    }
    if ((len & 1) && lane == 0) {
      const double xl = xv(len - 1);
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r < nrows) acc[r] = acc[r] + __ldg(a + r * ld + len - 1) * xl;
    }
  } else {
    for (int t = lane; t < len; t += 32) {
      const double xt = xv(t);
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r < nrows) acc[r] = acc[r] + __ldg(a + r * ld + t) * xt;
    }
  }
  warp_reduce<R>(acc);
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = acc[r];
}

// Register budget of 4 CTAs per SM: with it ptxas keeps the unrolled 16-byte row loads in
// flight (64 registers; C2 0.173 -> 0.165 ms); at the default budget it interleaves them.
// R rows per warp (8 warps): R = 4 below m = 1024; R = 8 (64 rows per CTA) at large m, where
// the one-wave plan otherwise rounds 119 row groups x 4 spans = 476 of 592 CTA slots (C5).
template <int R, int U, int MINB>
__global__ void __launch_bounds__(kTpb, MINB) k_row_gemv(const double* __restrict__ A, int m, long long N, long long ld, VSel xs,
                                                   long long xoff, int scaled, const MinresState* st,
                                                   double* __restrict__ partial, unsigned* counter,
                                                   double* __restrict__ out, int span) {
  griddep_wait();
  const double* __restrict__ x = vsel(xs, st) + xoff;
  const double sc = scaled ? st->inv_gamma : 1.0;
  const long long c0 = static_cast<long long>(blockIdx.x) * span;
  const int len = static_cast<int>(min(static_cast<long long>(span), N - c0));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec_ok = ((ld & 1) == 0);  // span is even, so every row segment starts 16-byte aligned
  {
    const int row = blockIdx.y * (R * (kTpb / 32)) + warp * R;
    if (row < m) {
      double d[R];
      const int nr = min(R, m - row);
      warp_rows_dot<R, U>(A + static_cast<long long>(row) * ld + c0, ld, nr, x + c0, scaled, sc, len, vec_ok, lane, d);
      if (lane == 0)
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (r < nr) partial[static_cast<long long>(blockIdx.x) * m + row + r] = d[r];
    }
  }
  // last block reduces over spans in index order
  __shared__ bool am_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    am_last = (atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  for (int row = threadIdx.x; row < m; row += blockDim.x) {
    double s = 0.0;
    // unrolled: the partial loads are independent, so 8 L2 round trips overlap
#pragma unroll 8
    for (unsigned b = 0; b < gridDim.x; ++b) s += __ldcg(&partial[static_cast<long long>(b) * m + row]);
    out[row] = s;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

static int g_rg_wide_m = [] {  // env GNW_RG_WIDE_M: m from which the 8-rows-per-warp variant runs
  const char* e = std::getenv("GNW_RG_WIDE_M");
  return e ? std::atoi(e) : 1024;
}();
static inline bool rg_wide(int m) { return m >= g_rg_wide_m; }
#define K_ROW_GEMV_NARROW k_row_gemv<4, 4, 4>
#define K_ROW_GEMV_WIDE k_row_gemv<8, 2, 3>

RowGemv row_gemv_plan(long long N, int m, int reserve) {
  static int sms = 0, occ = 0, occw = 0;  // SMs, resident k_row_gemv CTAs per SM (narrow, wide)
  if (sms == 0) {
    int dev = 0;
    sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, K_ROW_GEMV_NARROW, kTpb, 0) != cudaSuccess || occ < 1) occ = 4;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occw, K_ROW_GEMV_WIDE, kTpb, 0) != cudaSuccess || occw < 1) occw = 3;
    cudaGetLastError();
  }
  const bool wide = rg_wide(m);
  const int rows_cta = (wide ? 8 : 4) * (kTpb / 32);
  // reserve: CTA slots per SM left free for a concurrent graph branch (the V-cycle)
  const int slots = sms * std::max(1, (wide ? occw : occ) - reserve);
  RowGemv p;
  p.ngroups = std::max(1, (m + rows_cta - 1) / rows_cta);
  const long long spans = std::max(1, slots / p.ngroups);
  long long span = (N + spans - 1) / spans;
  span = std::max<long long>(64, (span + 63) / 64 * 64);
  p.chunk = static_cast<int>(span);
  p.nchunks = static_cast<int>((N + span - 1) / span);
  return p;
}

void row_gemv(const double* A, int m, long long N, long long ld, VSel x, long long x_off, int scaled,
              const MinresState* st, double* partial, unsigned* counter, double* out, const RowGemv& plan,
              cudaStream_t s) {
  const bool wide = rg_wide(m);
  const int rows_cta = (wide ? 8 : 4) * (kTpb / 32);
  const dim3 grid(plan.nchunks, (m + rows_cta - 1) / rows_cta);
  GNW_LAUNCH(launch_k(wide ? K_ROW_GEMV_WIDE : K_ROW_GEMV_NARROW, grid, kTpb, 0, s, A, m, N, ld, x, x_off, scaled, st,
                      partial, counter, out, plan.chunk));
  check_launch("row_gemv");
}

// ======================================================================
// Saddle operator  y = [Q x1 + D^T x2 ; D x1 - (1/beta) J^T (J x2)]
// ======================================================================
// B = 16 (m >= 1024): the register budget of 5 CTAs per SM lets ptxas keep the 16 loads of a
// batch in flight (with the default budget it interleaves them with the add chain at 32 registers)
template <int B>
__global__ void __launch_bounds__(kTpb, B >= 16 ? 5 : 8) k_saddle(OperatorArgs op, VSel xs, int scaled, const double* __restrict__ u,
                                                 VSel ys, MinresState* st, int loop, int nb_edge,
                                                 double* part, unsigned* counter) {
  // the operator's entries are fixed per assembly: their loads are issued BEFORE the
  // grid-dependency wait, so they overlap the predecessor's drain (its last-block reduction)
  extern __shared__ double usm[];
  __shared__ double red[kTpb / 32];
  double dotv[1] = {0.0};
  if (static_cast<int>(blockIdx.x) < nb_edge) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    // unit-square RT0 rows (5 Q entries, 2 D^T entries; boundary rows padded): every entry
    // load of the row is issued before the state load that selects z
    const bool fast = e < op.K && op.Qs.width == 5 && op.Dts.width == 2;
    int cq[5], ct[2];
    double vq[5], vt[2];
    if (fast) {
      sell_load<5>(op.Qs, e, cq, vq);
      sell_load<2>(op.Dts, e, ct, vt);
    }
    griddep_wait();
    const double* __restrict__ z = vsel(xs, st);
    double* __restrict__ y = vsel(ys, st);
    const double sc = scaled ? st->inv_gamma : 1.0;
    if (e < op.K) {
      double sq = 0.0, sd = 0.0;
      if (fast) {
        sq = sell_finish<5>(cq, vq, z, 0, scaled, sc);
        sd = sell_finish<2>(ct, vt, z, op.K, scaled, sc);
      } else if (op.Qs.width > 0 && op.Dts.width > 0) {  // SELL-32: independent, coalesced entry loads
        sq = sell_row(op.Qs, e, z, 0, scaled, sc);
        sd = sell_row(op.Dts, e, z, op.K, scaled, sc);
      } else {
        for (int k = op.Q.rowptr[e]; k < op.Q.rowptr[e + 1]; ++k) {
          const int c = op.Q.cols[k];
          sq = sq + __ldg(&op.Q.vals[k]) * (scaled ? z[c] * sc : z[c]);
        }
        for (int k = op.Dt.rowptr[e]; k < op.Dt.rowptr[e + 1]; ++k) {
          const long long c = op.K + op.Dt.cols[k];
          sd = sd + __ldg(&op.Dt.vals[k]) * (scaled ? z[c] * sc : z[c]);
        }
      }
      double o = 0.0;
      o = o + 1.0 * sq;  // spmv_add(*Q, zeta, 1.0, out1)
      o = o + 1.0 * sd;  // axpy(1.0, dt, out1)
      y[e] = o;
      dotv[0] = o * (scaled ? z[e] * sc : z[e]);
    }
  } else {
    const long long c = static_cast<long long>(blockIdx.x - nb_edge) * blockDim.x + threadIdx.x;
    const bool fast = c < op.N && op.Ds.width == 3;
    int cd[3];
    double vd[3];
    if (fast) sell_load<3>(op.Ds, c, cd, vd);
    griddep_wait();
    const double* __restrict__ z = vsel(xs, st);
    double* __restrict__ y = vsel(ys, st);
    const double sc = scaled ? st->inv_gamma : 1.0;
    if (op.m > 0 && op.q == nullptr) {  // the fused/lean loops read q instead of J^T (J zhat2)
      for (int t = threadIdx.x; t < op.m; t += blockDim.x) usm[t] = u[t];
      __syncthreads();
    }
    if (c < op.N) {
      double sd = 0.0;
      if (fast) {
        sd = sell_finish<3>(cd, vd, z, 0, scaled, sc);
      } else if (op.Ds.width > 0) {
        sd = sell_row(op.Ds, c, z, 0, scaled, sc);
      } else {
        for (int k = op.D.rowptr[c]; k < op.D.rowptr[c + 1]; ++k) {
          const int e = op.D.cols[k];
          sd = sd + __ldg(&op.D.vals[k]) * (scaled ? z[e] * sc : z[e]);
        }
      }
      double o = 0.0;
      o = o + 1.0 * sd;  // spmv_add(*D, zeta, 1.0, out2)
      if (op.m > 0 && op.q != nullptr) {  // fused: J^T (J zhat2) = J^T (t' * ig) ~ q * ig (Woodbury identity J z2 = t')
        o = o + *op.neg_inv_beta * (op.q[c] * sc);
      } else if (op.m > 0) {  // matvec_transpose(J, J dm), linalg.cpp:45-54
        const double jt = col_dot<B>(op.J + c, op.ldj, usm, op.m);
        o = o + *op.neg_inv_beta * jt;  // axpy(-1.0 / beta, jtjdm, out2)
      }
      y[op.K + c] = o;
      dotv[0] = o * (scaled ? z[op.K + c] * sc : z[op.K + c]);
    }
  }
  double tot[1];
  if (grid_reduce_last<1>(dotv, part, counter, red, tot) && threadIdx.x == 0) {
    const double delta = tot[0];
    if (loop) {
      st->delta = delta;
      st->coef_v1 = -delta / st->gamma_cur;
      st->coef_v2 = -st->gamma_cur / st->gamma_prev;
    } else {
      st->scratch[0] = delta;
    }
  }
}

void saddle_operator(const OperatorArgs& op, VSel x, int scaled, const double* u, VSel y, MinresState* st,
                     int loop, double* partial, unsigned* counter, cudaStream_t s) {
  // u staged in shared memory for the J^T u column dot: m <= kMaxStageM doubles
  smem_optin(reinterpret_cast<const void*>(k_saddle<8>), kMaxStageM * 8);
  smem_optin(reinterpret_cast<const void*>(k_saddle<16>), kMaxStageM * 8);
  const int nbe = static_cast<int>(grid_for(op.K)), nbc = static_cast<int>(grid_for(op.N));
  GNW_LAUNCH(launch_k((op.m >= kSweepBatchWideM && op.q == nullptr) ? k_saddle<16> : k_saddle<8>, nbe + nbc, kTpb, op.q != nullptr ? 0 : std::max(op.m, 1) * sizeof(double), s, op, x, scaled, u, y, st, loop, nbe,
                                                                       partial, counter));
  check_launch("saddle_operator");
}

// ======================================================================
// Preconditioner (inversion.cpp:71-89) fused with the v-combination
// ======================================================================
// v_next = Az + c1 v_cur + c2 v_prev (combine, minres.cpp:76-77; `loop`) or v = y
// (plain preconditioner input); z1 = qinv .* v1 on the edge part (inversion.cpp:79);
// per-block partial dots <z, v>, <z, z> (edge part) and <v, v> (all) -> dots_part.
__global__ void __launch_bounds__(kTpb) k_combine_elem(PrecArgs pa, VSel azs, VSel vcs, VSel vps, VSel vns,
                                                       VSel zns, int loop, const MinresState* st,
                                                       double* dots_part) {
  __shared__ double red[3 * (kTpb / 32)];
  const long long n = pa.K + pa.N;
  // two consecutive elements per thread, 16-byte loads (all vectors are separate allocations)
  const long long i0 = 2 * (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x);
  // v_cur and v_prev (and the iteration index that selects their ring slots) were written before
  // the predecessor (the operator) started: loaded BEFORE the grid-dependency wait, under the
  // operator's last-block reduction
  const double* __restrict__ vc = loop ? vsel(vcs, st) : nullptr;
  const double* __restrict__ vp = loop ? vsel(vps, st) : nullptr;
  double2 pb = make_double2(0.0, 0.0), pc = make_double2(0.0, 0.0);
  if (loop && i0 + 1 < n) {
    pb = *reinterpret_cast<const double2*>(vc + i0);
    pc = *reinterpret_cast<const double2*>(vp + i0);
  }
  griddep_wait();
  const double* __restrict__ az = vsel(azs, st);
  double* __restrict__ vn = vsel(vns, st);
  double* __restrict__ zn = vsel(zns, st);
  const double c1 = loop ? st->coef_v1 : 0.0, c2 = loop ? st->coef_v2 : 0.0;
  double d[3] = {0.0, 0.0, 0.0};  // <z, v>, <z, z>, <v, v>
  auto one = [&](long long i, double a, double b, double c) {
    double v;
    if (loop) {
      v = a + c1 * b;  // combine: ca*a + cb*b + cc*c, ca = 1
      v = v + c2 * c;
    } else {
      v = a;
    }
    if (i < pa.K) {
      const double z = __ldg(&pa.qinv[i]) * v;
      zn[i] = z;
      d[0] = d[0] + z * v;
      d[1] = d[1] + z * z;
    }
    d[2] = d[2] + v * v;
    return v;
  };
  if (i0 + 1 < n) {
    const double2 a = *reinterpret_cast<const double2*>(az + i0);
    const double2 b = pb, c = pc;
    const double v0 = one(i0, a.x, b.x, c.x);
    const double v1 = one(i0 + 1, a.y, b.y, c.y);
    if (loop) *reinterpret_cast<double2*>(vn + i0) = make_double2(v0, v1);
  } else if (i0 < n) {
    const double v0 = one(i0, az[i0], loop ? vc[i0] : 0.0, loop ? vp[i0] : 0.0);
    if (loop) vn[i0] = v0;
  }
  block_reduce<3>(d, red);
  if (threadIdx.x == 0)
    for (int k = 0; k < 3; ++k) dots_part[blockIdx.x * 3 + k] = d[k];
}

int combine_blocks(long long K, long long N) { return static_cast<int>(grid_for((K + N + 1) / 2)); }

// the combine kernel's per-block dot partials (n triples) summed in a fixed order by one CTA:
// run on a side graph branch beside the dense sweeps, so the finish kernel's last block adds
// one triple instead of thousands (its serial L2 round trips were on the critical path)
__global__ void __launch_bounds__(1024) k_sum_triples(const double* __restrict__ parts, int n, double* __restrict__ out) {
  griddep_wait();
  __shared__ double red[3 * 32];
  double a[3] = {0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < n; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < 3; ++k) a[k] += __ldcg(&parts[b * 3 + k]);
  block_reduce<3>(a, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] = a[k];
}

void sum_triples(const double* parts, int n, double* out, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_sum_triples, 1, 1024, 0, s, parts, n, out));
  check_launch("sum_triples");
}

void combine_elem(const PrecArgs& pa, VSel az, VSel vcur, VSel vprev, VSel vnext, VSel znext, int loop,
                  MinresState* st, double* dots_part, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_combine_elem, combine_blocks(pa.K, pa.N), kTpb, 0, s, pa, az, vcur, vprev, vnext, znext, loop, st, dots_part));
  check_launch("combine_elem");
}

void combine_precondition(const PrecArgs& pa, VSel az, VSel vcur, VSel vprev, VSel vnext, VSel znext, int loop,
                          MinresState* st, double* /*vcopy*/, double* dots_part, double* t_part,
                          unsigned* counter, double* t_out, const RowGemv& plan, cudaStream_t s) {
  combine_elem(pa, az, vcur, vprev, vnext, znext, loop, st, dots_part, s);
  if (pa.m > 0)  // t = H^T v2 (matvec_transpose(h_hat, y2), inversion.cpp:82): row GEMV over Ht
    row_gemv(pa.Ht, pa.m, pa.N, pa.ldh, vnext, pa.K, 0, st, t_part, counter, t_out, plan, s);
}

// t2 = Cinv t, warp per row
__global__ void k_cinv_apply(const double* __restrict__ Cinv, const double* __restrict__ t, double* __restrict__ t2,
                             int m) {
  griddep_wait();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= m) return;
  double acc[1] = {0.0};
  for (int j = lane; j < m; j += 32) acc[0] = acc[0] + __ldg(&Cinv[static_cast<long long>(w) * m + j]) * t[j];
  warp_reduce<1>(acc);
  if (lane == 0) t2[w] = acc[0];
}

// r = t - C t2 (warp per row, C full and symmetric)
__global__ void k_cap_residual(const double* __restrict__ C, const double* __restrict__ t,
                               const double* __restrict__ t2, double* __restrict__ r, int m) {
  griddep_wait();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= m) return;
  double acc[1] = {0.0};
  for (int j = lane; j < m; j += 32) acc[0] = acc[0] + __ldg(&C[static_cast<long long>(w) * m + j]) * t2[j];
  warp_reduce<1>(acc);
  if (lane == 0) r[w] = t[w] - acc[0];
}

// t2 += Cinv r (warp per row)
__global__ void k_cinv_refine(const double* __restrict__ Cinv, const double* __restrict__ r, double* __restrict__ t2,
                              int m) {
  griddep_wait();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= m) return;
  double acc[1] = {0.0};
  for (int j = lane; j < m; j += 32) acc[0] = acc[0] + __ldg(&Cinv[static_cast<long long>(w) * m + j]) * r[j];
  warp_reduce<1>(acc);
  if (lane == 0) t2[w] = t2[w] + acc[0];
}

// t2 = L^-T L^-1 t in one CTA (x in shared memory, L read from L2): right-looking forward and
// backward substitution, each step's updates spread over the threads.  The fallback for an
// ill-conditioned capacitance matrix (PrecArgs::cap_tri); O(m) barriers, ~0.1 ms at m ~ 1000.
__global__ void __launch_bounds__(1024) k_cap_tri_solve(const double* __restrict__ L, const double* __restrict__ t,
                                                        double* __restrict__ t2, int m) {
  griddep_wait();
  extern __shared__ double xs[];
  for (int i = threadIdx.x; i < m; i += blockDim.x) xs[i] = t[i];
  __syncthreads();
  for (int i = 0; i < m; ++i) {  // L y = t
    if (threadIdx.x == 0) xs[i] = xs[i] / L[static_cast<long long>(i) * m + i];
    __syncthreads();
    const double yi = xs[i];
    for (int j = i + 1 + threadIdx.x; j < m; j += blockDim.x) xs[j] = xs[j] - L[static_cast<long long>(j) * m + i] * yi;
    __syncthreads();
  }
  for (int i = m - 1; i >= 0; --i) {  // L^T x = y
    if (threadIdx.x == 0) xs[i] = xs[i] / L[static_cast<long long>(i) * m + i];
    __syncthreads();
    const double xi = xs[i];
    for (int j = threadIdx.x; j < i; j += blockDim.x) xs[j] = xs[j] - L[static_cast<long long>(i) * m + j] * xi;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) t2[i] = xs[i];
}

void capacitance_solve(const PrecArgs& pa, const double* t, double* t2, cudaStream_t s) {
  if (pa.m == 0) return;
  if (pa.cap_tri && !pa.exact) {
    smem_optin(reinterpret_cast<const void*>(k_cap_tri_solve), kMaxStageM * 8);
    GNW_LAUNCH(launch_k(k_cap_tri_solve, 1, 1024, static_cast<size_t>(pa.m) * sizeof(double), s, pa.Lc, t, t2, pa.m));
    return check_launch("capacitance_solve");
  }
  if (pa.exact) {
    GNW_LAUNCH(launch_k(k_coarse_cholesky, 1, 64, 0, s, pa.Lc, pa.m, vfixed(const_cast<double*>(t)), t2, nullptr, 1, 1));
  } else {
    const unsigned g = grid_for(static_cast<long long>(pa.m) * 32);
    GNW_LAUNCH(launch_k(k_cinv_apply, g, kTpb, 0, s, pa.Cinv, t, t2, pa.m));
    if (pa.Cfull && pa.cres) {
      // one step of iterative refinement: the fused/lean loops use J z2 = t2 = C^-1 t, which
      // holds only as far as C t2 = t does; the explicit inverse alone leaves a residual
      // ~ eps kappa(C) |t|, refinement brings it to ~ eps |C| |t2| (backward stable)
      check_launch("capacitance_solve");
      GNW_LAUNCH(launch_k(k_cap_residual, g, kTpb, 0, s, pa.Cfull, t, const_cast<const double*>(t2), pa.cres, pa.m));
      check_launch("capacitance_solve");
      GNW_LAUNCH(launch_k(k_cinv_refine, g, kTpb, 0, s, pa.Cinv, const_cast<const double*>(pa.cres), t2, pa.m));
    }
  }
  check_launch("capacitance_solve");
}

// upper triangle of C from its lower triangle (the capacitance DGEMM computes the lower tiles)
__global__ void k_mirror_lower(double* C, int n) {
  griddep_wait();
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(n) * n) return;
  const int i = static_cast<int>(t / n), j = static_cast<int>(t % n);
  if (j <= i) return;
  C[static_cast<long long>(i) * n + j] = C[static_cast<long long>(j) * n + i];
}

void mirror_lower(double* C, int n, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_mirror_lower, grid_for(static_cast<long long>(n) * n), kTpb, 0, s, C, n));
  check_launch("mirror_lower");
}


template <int B>
__global__ void __launch_bounds__(kTpb, B >= 16 ? 5 : 8) k_finish_prec(PrecArgs pa, const double* __restrict__ svc,
                                                      const double* __restrict__ t2, VSel vns, VSel zns, int loop,
                                                      MinresState* st, const double* __restrict__ dots_edge,
                                                      int n_edge_blocks, double* part, unsigned* counter) {
  griddep_wait();
  extern __shared__ double tsm[];
  __shared__ double red[3 * (kTpb / 32)];
  const double* __restrict__ vn = vsel(vns, st);
  double* __restrict__ zn = vsel(zns, st);
  if (pa.m > 0) {
    for (int t = threadIdx.x; t < pa.m; t += blockDim.x) tsm[t] = t2[t];
    __syncthreads();
  }
  double d[3] = {0.0, 0.0, 0.0};
  const long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c < pa.N) {
    double z = svc[c];
    if (pa.m > 0) {  // w = matvec(h_hat, t) row c (linalg.cpp:33-43); s += (-1/beta) w
      double w = 0.0;
      const double* __restrict__ Hc = pa.Ht + c;
      if (pa.q != nullptr) {  // one sweep over H and J: w = (H t')_c, q_c = (J^T t')_c
        double qq = 0.0;
        col_dot2<8>(Hc, pa.ldh, pa.J + c, pa.ldj, tsm, pa.m, w, qq);  // 16 loads in flight (32 at B = 16 spill residency)
        pa.q[c] = qq;
      } else {
        w = col_dot<B>(Hc, pa.ldh, tsm, pa.m);
      }
      z = z + *pa.neg_inv_beta * w;
    }
    zn[pa.K + c] = z;
    const double v = vn[pa.K + c];
    d[0] = z * v;
    d[1] = z * z;
  }
  double tot[3];
  if (!grid_reduce_last<3>(d, part, counter, red, tot)) return;
  finish_scalars(tot, dots_edge, n_edge_blocks, loop, st, red);
}

__global__ void k_givens_from_scratch(MinresState* st) {
  griddep_wait();
  givens_step(st->scratch[0], st->scratch[1], st->scratch[2], st);
}
void givens_from_scratch(MinresState* st, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_givens_from_scratch, 1, 1, 0, s, st));
  check_launch("givens_from_scratch");
}

template <int B>
__global__ void __launch_bounds__(kTpb, B >= 16 ? 5 : 8) k_col_sweep(const double* __restrict__ A, long long ld,
                                                    const double* __restrict__ t, int m, long long n,
                                                    double* __restrict__ q, VSel ys, long long yoff,
                                                    const MinresState* st, const double* __restrict__ coef,
                                                    double* __restrict__ yout) {
  griddep_wait();
  extern __shared__ double tsm[];
  for (int i = threadIdx.x; i < m; i += blockDim.x) tsm[i] = t[i];
  __syncthreads();
  const long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const double qc = col_dot<B>(A + c, ld, tsm, m);
  q[c] = qc;
  if (yout) yout[c] = vsel(ys, st)[yoff + c] + *coef * qc;  // y' = v2 + (-1/beta) q
}

void col_sweep(const double* A, long long ld, const double* t, int m, long long n, double* q, cudaStream_t s,
               VSel ys, long long yoff, const MinresState* st, const double* coef, double* yout) {
  // t staged in shared memory: m <= kMaxStageM doubles
  smem_optin(reinterpret_cast<const void*>(k_col_sweep<8>), kMaxStageM * 8);
  smem_optin(reinterpret_cast<const void*>(k_col_sweep<16>), kMaxStageM * 8);
  static const int wide_m = [] {  // env GNW_COL_SWEEP_WIDE_M: batch-16 threshold (experiments)
    const char* e = std::getenv("GNW_COL_SWEEP_WIDE_M");
    return e ? std::atoi(e) : kSweepBatchWideM;
  }();
  GNW_LAUNCH(launch_k(m >= wide_m ? k_col_sweep<16> : k_col_sweep<8>, grid_for(n), kTpb,
                      std::max(m, 1) * sizeof(double), s, A, ld, t, m, n, q, ys, yoff, st, coef, yout));
  check_launch("col_sweep");
}

int finish_blocks(const PrecArgs& pa) {
  return static_cast<int>(grid_for(pa.N));
}

void finish_precondition(const PrecArgs& pa, const double* svc, const double* t2, VSel vnext, VSel znext, int loop,
                         MinresState* st, const double* dots_edge, int n_edge_blocks, double* part,
                         unsigned* counter, cudaStream_t s) {
  smem_optin(reinterpret_cast<const void*>(k_finish_prec<8>), kMaxStageM * 8);
  smem_optin(reinterpret_cast<const void*>(k_finish_prec<16>), kMaxStageM * 8);
  GNW_LAUNCH(launch_k(pa.m >= kSweepBatchWideM ? k_finish_prec<16> : k_finish_prec<8>, finish_blocks(pa), kTpb,
                      std::max(pa.m, 1) * sizeof(double), s, pa, svc, t2, vnext, znext, loop, st, dots_edge,
                      n_edge_blocks, part, counter));
  check_launch("finish_precondition");
}

// ======================================================================
// Partitioned (multi-GPU) solve: fixed-order sums of the ranks' partials and the scalar steps
// that follow them (context_rowpart.cu).  Every rank sums the same gathered partials in rank
// order, so every rank holds the same bits.
// ======================================================================
__global__ void k_sum_scratch(const double* __restrict__ parts, int P, int cnt, MinresState* st, int k0) {
  griddep_wait();
  const int i = threadIdx.x;
  if (i >= cnt) return;
  double s = 0.0;
  for (int r = 0; r < P; ++r) s += parts[r * cnt + i];
  st->scratch[k0 + i] = s;
}

void sum_scratch(const double* parts, int P, int cnt, MinresState* st, int k0, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_sum_scratch, 1, 32, 0, s, parts, P, cnt, st, k0));
  check_launch("sum_scratch");
}

// the saddle kernel's loop epilogue from the reduced delta (scratch[0])
__global__ void k_delta_coef(MinresState* st) {
  griddep_wait();
  const double delta = st->scratch[0];
  st->delta = delta;
  st->coef_v1 = -delta / st->gamma_cur;
  st->coef_v2 = -st->gamma_cur / st->gamma_prev;
}
void delta_coef(MinresState* st, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_delta_coef, 1, 1, 0, s, st));
  check_launch("delta_coef");
}

__global__ void k_sum_partials(const double* __restrict__ parts, int P, long long n, double* __restrict__ out) {
  griddep_wait();
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int r = 0; r < P; ++r) s += parts[static_cast<long long>(r) * n + i];
  out[i] = s;
}

void sum_partials(const double* parts, int P, long long n, double* out, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_sum_partials, grid_for(n), kTpb, 0, s, parts, P, n, out));
  check_launch("sum_partials");
}

__global__ void k_capacitance_reduce(const double* __restrict__ parts, int P, int m, double beta,
                                     double* __restrict__ C) {
  griddep_wait();
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long mm = static_cast<long long>(m) * m;
  if (k >= mm) return;
  double s = 0.0;
  for (int r = 0; r < P; ++r) s += parts[r * mm + k];
  double v = s / beta;
  if (k / m == k % m) v += 1.0;
  C[k] = v;
}

void capacitance_reduce(const double* parts, int P, int m, double beta, double* C, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_capacitance_reduce, grid_for(static_cast<long long>(m) * m), kTpb, 0, s, parts, P, m, beta, C));
  check_launch("capacitance_reduce");
}

// ======================================================================
// MINRES vector recurrences (minres.cpp:93-106) and loop control
// ======================================================================

__global__ void __launch_bounds__(kTpb) k_minres_update(long long n, VSel zs, VSel azs, VSel wps, VSel wcs, VSel wns,
                                                        VSel ups, VSel ucs, VSel uns, double* __restrict__ x,
                                                        double* __restrict__ r, MinresState* st,
                                                        double* hist_e, double* hist_p, long long hist_cap,
                                                        double* part, unsigned* counter,
                                                        cudaGraphConditionalHandle handle, int use_cond) {
  griddep_wait();
  __shared__ double red[kTpb / 32];
  if (use_cond != 2 && st->status != kRunning) {  // use_cond == 2: isolated timing, no loop control
    if (use_cond == 1 && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(handle, 0);
    return;
  }
  const double* __restrict__ z = vsel(zs, st);
  const double* __restrict__ az = vsel(azs, st);
  const double* __restrict__ wp = vsel(wps, st);
  const double* __restrict__ wc = vsel(wcs, st);
  double* __restrict__ wn = vsel(wns, st);
  const double* __restrict__ up = vsel(ups, st);
  const double* __restrict__ uc = vsel(ucs, st);
  double* __restrict__ un = vsel(uns, st);
  const double ig = st->inv_gamma, na3 = -st->alpha3, na2 = -st->alpha2, ia = st->inv_alpha1;
  const double tau = st->tau, ntau = -tau;
  double rr[1] = {0.0};
  // minres.cpp:93-106 per element; pairs of elements with 16-byte loads/stores
  auto elem = [&](double zv, double wpv, double wcv, double azv, double upv, double ucv, double xv, double rv,
                  double& wo, double& uo, double& xo, double& ro) {
    const double zh = zv * ig;
    double w = zh + na3 * wpv;
    w = w + na2 * wcv;
    w = w * ia;
    double uu = azv + na3 * upv;
    uu = uu + na2 * ucv;
    uu = uu * ia;
    wo = w;
    uo = uu;
    xo = xv + tau * w;
    ro = rv + ntau * uu;
    rr[0] = rr[0] + ro * ro;
  };
  const long long np = n / 2;
  auto ld2 = [](const double* p, long long k) { return *reinterpret_cast<const double2*>(p + 2 * k); };
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < np;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double2 zv = ld2(z, k), wpv = ld2(wp, k), wcv = ld2(wc, k), azv = ld2(az, k), upv = ld2(up, k),
                  ucv = ld2(uc, k), xv = ld2(x, k), rv = ld2(r, k);
    double2 wo, uo, xo, ro;
    elem(zv.x, wpv.x, wcv.x, azv.x, upv.x, ucv.x, xv.x, rv.x, wo.x, uo.x, xo.x, ro.x);
    elem(zv.y, wpv.y, wcv.y, azv.y, upv.y, ucv.y, xv.y, rv.y, wo.y, uo.y, xo.y, ro.y);
    *reinterpret_cast<double2*>(wn + 2 * k) = wo;
    *reinterpret_cast<double2*>(un + 2 * k) = uo;
    *reinterpret_cast<double2*>(x + 2 * k) = xo;
    *reinterpret_cast<double2*>(r + 2 * k) = ro;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long i = n - 1;
    elem(z[i], wp[i], wc[i], az[i], up[i], uc[i], x[i], r[i], wn[i], un[i], x[i], r[i]);
  }
  double tot[1];
  if (!grid_reduce_last<1>(rr, part, counter, red, tot) || threadIdx.x != 0 || use_cond == 2) return;
  if (use_cond == 3) {  // partitioned: this rank's ||r||^2 only; update_tail_from_scratch finishes
    st->scratch[6] = tot[0];
    return;
  }
  update_tail(tot[0], st, hist_e, hist_p, hist_cap);
  if (use_cond == 1) cudaGraphSetConditional(handle, st->status == kRunning ? 1u : 0u);
}

__global__ void k_update_tail_from_scratch(MinresState* st, double* hist_e, double* hist_p, long long hist_cap) {
  griddep_wait();
  if (st->status != kRunning) return;
  update_tail(st->scratch[6], st, hist_e, hist_p, hist_cap);
}
void update_tail_from_scratch(MinresState* st, double* hist_e, double* hist_p, long long hist_cap, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_update_tail_from_scratch, 1, 1, 0, s, st, hist_e, hist_p, hist_cap));
  check_launch("update_tail_from_scratch");
}

void minres_update(long long n, VSel z, VSel az, VSel wprev, VSel wcur, VSel wnext, VSel uprev, VSel ucur, VSel unext,
                   double* x, double* r, MinresState* st, double* hist_e, double* hist_p, long long hist_cap,
                   double* part, unsigned* counter, unsigned long long cond_handle, int use_cond, cudaStream_t s) {
  const unsigned grid = std::min<unsigned>(grid_for((n + 1) / 2), 148u * 8u);
  GNW_LAUNCH(launch_k(k_minres_update, grid, kTpb, 0, s, n, z, az, wprev, wcur, wnext, uprev, ucur, unext, x, r, st, hist_e, hist_p,
                                        hist_cap, part, counter,
                                        static_cast<cudaGraphConditionalHandle>(cond_handle), use_cond));
  check_launch("minres_update");
}

__global__ void k_minres_rotate(MinresState* st) {
  griddep_wait();
  st->gamma_prev = st->gamma_cur;
  st->gamma_cur = st->gamma_next;
  st->c_prev = st->c_cur;
  st->c_cur = st->c_next;
  st->s_prev = st->s_cur;
  st->s_cur = st->s_next;
  st->inv_gamma = 1.0 / st->gamma_cur;
  st->j = st->j + 1;
  st->status = (st->j > st->maxit) ? kMaxit : kRunning;
}

void minres_rotate(MinresState* st, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_minres_rotate, 1, 1, 0, s, st));
  check_launch("minres_rotate");
}

__global__ void __launch_bounds__(kTpb) k_residual(long long n, const double* __restrict__ b,
                                                   const double* __restrict__ y, double* __restrict__ r,
                                                   MinresState* st, int want_b, double* part, unsigned* counter) {
  griddep_wait();
  __shared__ double red[2 * (kTpb / 32)];
  double v[2] = {0.0, 0.0};
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double ri = b[i] - y[i];
    r[i] = ri;
    v[0] = v[0] + ri * ri;
    if (want_b) v[1] = v[1] + b[i] * b[i];
  }
  double tot[2];
  if (grid_reduce_last<2>(v, part, counter, red, tot) && threadIdx.x == 0) {
    st->scratch[4] = tot[0];
    if (want_b) st->scratch[5] = tot[1];
  }
}

void residual(long long n, const double* b, const double* y, double* r, MinresState* st, int want_b, double* part,
              unsigned* counter, cudaStream_t s) {
  const unsigned grid = std::min<unsigned>(grid_for(n), 148u * 8u);
  GNW_LAUNCH(launch_k(k_residual, grid, kTpb, 0, s, n, b, y, r, st, want_b, part, counter));
  check_launch("residual");
}

__global__ void __launch_bounds__(kTpb) k_dot(long long n, const double* __restrict__ a, const double* __restrict__ b,
                                              double* out, double* part, unsigned* counter) {
  griddep_wait();
  __shared__ double red[kTpb / 32];
  double v[1] = {0.0};
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    v[0] = v[0] + a[i] * b[i];
  double tot[1];
  if (grid_reduce_last<1>(v, part, counter, red, tot) && threadIdx.x == 0) *out = tot[0];
}

void dot(long long n, const double* a, const double* b, double* out, double* part, unsigned* counter, cudaStream_t s) {
  const unsigned grid = std::min<unsigned>(grid_for(n), 148u * 8u);
  GNW_LAUNCH(launch_k(k_dot, grid, kTpb, 0, s, n, a, b, out, part, counter));
  check_launch("dot");
}

// rhs = [-D^T (m - m_ref); J^T (g - g_obs) / beta]   inversion.cpp:126-146
__global__ void __launch_bounds__(kTpb) k_rhs(OperatorArgs op, double beta, const double* __restrict__ mdl,
                                              const double* __restrict__ mref, const double* __restrict__ g,
                                              const double* __restrict__ gobs, double* __restrict__ rhs,
                                              int nb_edge) {
  griddep_wait();
  extern __shared__ double gsm[];
  if (static_cast<int>(blockIdx.x) < nb_edge) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= op.K) return;
    double s = 0.0;
    for (int k = op.Dt.rowptr[e]; k < op.Dt.rowptr[e + 1]; ++k) {
      const int c = op.Dt.cols[k];
      s = s + __ldg(&op.Dt.vals[k]) * (mdl[c] - mref[c]);
    }
    rhs[e] = -s;
  } else {
    for (int t = threadIdx.x; t < op.m; t += blockDim.x) gsm[t] = g[t] - gobs[t];  // inversion.cpp:137-138
    __syncthreads();
    const long long c = static_cast<long long>(blockIdx.x - nb_edge) * blockDim.x + threadIdx.x;
    if (c >= op.N) return;
    double jt = 0.0;
    const double* __restrict__ Jc = op.J + c;
#pragma unroll 8
    for (int i = 0; i < op.m; ++i) jt = jt + __ldg(Jc + static_cast<long long>(i) * op.ldj) * gsm[i];
    rhs[op.K + c] = jt / beta;
  }
}

void assemble_rhs(const OperatorArgs& op, double beta, const double* mdl, const double* mref, const double* g,
                  const double* gobs, double* rhs, cudaStream_t s) {
  const int nbe = static_cast<int>(grid_for(op.K)), nbc = static_cast<int>(grid_for(op.N));
  smem_optin(reinterpret_cast<const void*>(k_rhs), kMaxStageM * 8);
  GNW_LAUNCH(launch_k(k_rhs, nbe + nbc, kTpb, std::max(op.m, 1) * sizeof(double), s, op, beta, mdl, mref, g, gobs,
                      rhs, nbe));
  check_launch("assemble_rhs");
}

// ======================================================================
// Capacitance DGEMM: C = I + (J Ht^T)/beta via split-K FP64 tensor-core DMMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA; tcgen05 has no kind::f64 on sm_100a).
// CTA tile 128x128, 8 warps (2 x 4), warp tile 64x32 = 8x4 DMMA tiles,
// K staged 16 at a time through a 3-stage cp.async ring.
// ======================================================================
namespace dg {
constexpr int BM = 128, BN = 128, BK = 16, LDS = BK + 4, STAGES = 3;
constexpr int SMEM = STAGES * (BM + BN) * LDS * 8;
}  // namespace dg

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256, 1) k_dgemm_nt(const double* __restrict__ A, long long lda,
                                                     const double* __restrict__ B, long long ldb, int m,
                                                     long long N, long long kchunk, const int2* __restrict__ pairs,
                                                     int npairs, double* __restrict__ part) {
  griddep_wait();
  using namespace dg;
  extern __shared__ __align__(16) double sm[];
  double* As = sm;                            // [STAGES][BM][LDS]
  double* Bs = sm + STAGES * BM * LDS;        // [STAGES][BN][LDS]
  const int2 pr = pairs[blockIdx.x];
  const int i0 = pr.x * BM, j0 = pr.y * BN;
  const long long k0 = static_cast<long long>(blockIdx.y) * kchunk;
  const long long k1 = min(N, k0 + kchunk);
  const int nkt = static_cast<int>((k1 - k0 + BK - 1) / BK);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps

  auto load_stage = [&](int stage, int kt) {
    const long long kb = k0 + static_cast<long long>(kt) * BK;
    // 128 rows x 16 doubles = 1024 16-byte chunks per operand; 4 per thread
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int chunk = tid + it * 256;
      const int row = chunk >> 3, kc = (chunk & 7) * 2;
      const long long kk = kb + kc;
      {
        const int gr = i0 + row;
        const bool ok = gr < m && kk < k1;
        const double* src = ok ? A + static_cast<long long>(gr) * lda + kk : A;
        cp_async16(As + (stage * BM + row) * LDS + kc, src, ok ? 16 : 0);
      }
      {
        const int gr = j0 + row;
        const bool ok = gr < m && kk < k1;
        const double* src = ok ? B + static_cast<long long>(gr) * ldb + kk : B;
        cp_async16(Bs + (stage * BN + row) * LDS + kc, src, ok ? 16 : 0);
      }
    }
  };

  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkt) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = kt + STAGES - 1;
    if (nxt < nkt) load_stage(nxt % STAGES, nxt);
    cp_async_commit();
    const int st = kt % STAGES;
    const double* as = As + st * BM * LDS;
    const double* bs = Bs + st * BN * LDS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) af[a] = as[(wm * 64 + a * 8 + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = bs[(wn * 32 + b * 8 + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();
  // partial tile out: part[(split * npairs + pair)][BM][BN]
  double* out = part + (static_cast<long long>(blockIdx.y) * npairs + blockIdx.x) * (BM * BN);
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = wm * 64 + a * 8 + (lane >> 2);
      const int c = wn * 32 + b * 8 + (lane & 3) * 2;
      *reinterpret_cast<double2*>(out + r * BN + c) = make_double2(acc[a][b][0], acc[a][b][1]);
    }
}

// C[i][j] = (sum_split part) / beta (+1 on the diagonal)   inversion.cpp:37-43
__global__ void k_dgemm_finalize(const double* __restrict__ part, const int2* __restrict__ pairs, int npairs,
                                 int splits, int m, double beta, double* __restrict__ C) {
  griddep_wait();
  using namespace dg;
  const int p = blockIdx.y;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= BM * BN) return;
  const int2 pr = pairs[p];
  const int i = pr.x * BM + e / BN, j = pr.y * BN + e % BN;
  if (i >= m || j >= m) return;
  double s = 0.0;
  for (int k = 0; k < splits; ++k) s += part[(static_cast<long long>(k) * npairs + p) * (BM * BN) + e];
  if (beta <= 0.0) {  // raw partial J_g H_g^T of one rank (partitioned capacitance)
    C[static_cast<long long>(i) * m + j] = s;
    return;
  }
  double v = s / beta;
  if (i == j) v += 1.0;
  C[static_cast<long long>(i) * m + j] = v;
}

DgemmPlan dgemm_plan(int m, long long N, int full, int sm_count) {
  DgemmPlan p;
  p.tile = dg::BM;
  p.ntiles = (m + dg::BM - 1) / dg::BM;
  p.npairs = full ? p.ntiles * p.ntiles : p.ntiles * (p.ntiles + 1) / 2;
  p.full = full;
  const long long kblocks = (N + dg::BK - 1) / dg::BK;
  // one CTA per SM (123 KB smem).  Split K so that the tile pairs x splits fill whole waves:
  // the smallest split count with >= 95 % wave efficiency and >= 2 waves (C5, 465 pairs:
  // 1 split = 3.14 waves of 0.27 s CTAs, 78 % efficient; 7 splits = 21.99 waves).
  int splits = 1;
  double best = -1.0;
  const int max_splits = static_cast<int>(std::max<long long>(1, std::min<long long>(kblocks / 8, 1024)));
  for (int sp = 1; sp <= max_splits; ++sp) {
    const long long ctas = static_cast<long long>(p.npairs) * sp;
    const long long waves = (ctas + sm_count - 1) / sm_count;
    if (waves < 2 && sp < max_splits) continue;
    const double eff = static_cast<double>(ctas) / static_cast<double>(waves * sm_count);
    if (eff > best + 0.01) {  // more splits only for a real gain (each costs a partial tile)
      best = eff;
      splits = sp;
    }
  }
  splits = static_cast<int>(std::max<long long>(1, std::min<long long>(splits, kblocks)));
  long long kchunk = ((kblocks + splits - 1) / splits) * dg::BK;
  p.splits = static_cast<int>((N + kchunk - 1) / kchunk);
  p.kchunk = kchunk;
  return p;
}

void capacitance_dgemm(const double* J, long long ldj, const double* Ht, long long ldh, int m, long long N,
                       double beta, const DgemmPlan& plan, double* part, double* C, cudaStream_t s) {
  if (N % 2 != 0 || ldj % 2 != 0 || ldh % 2 != 0)
    throw std::invalid_argument("capacitance_dgemm: N and leading dimensions must be even (16-byte rows)");
  // pair list lives at the end of the partial buffer
  int2 hp[4096];
  int np = 0;
  for (int i = 0; i < plan.ntiles; ++i)
    for (int j = 0; j < plan.ntiles; ++j)
      if (plan.full || j <= i) hp[np++] = make_int2(i, j);
  int2* dpairs = reinterpret_cast<int2*>(part + static_cast<long long>(plan.splits) * plan.npairs * dg::BM * dg::BN);
  cudaMemcpyAsync(dpairs, hp, np * sizeof(int2), cudaMemcpyHostToDevice, s);
  // TMA-staged, warp-specialised kernel (dgemm_tma.cu); the cp.async kernel is the fallback
  if (!capacitance_dgemm_tma(J, ldj, Ht, ldh, m, N, plan, dpairs, part, s)) {
    smem_optin(reinterpret_cast<const void*>(k_dgemm_nt), dg::SMEM);
    dim3 grid(plan.npairs, plan.splits);
    GNW_LAUNCH(launch_k(k_dgemm_nt, grid, 256, dg::SMEM, s, J, ldj, Ht, ldh, m, N, plan.kchunk, dpairs, plan.npairs, part));
    check_launch("dgemm_nt");
  }
  dim3 g2((dg::BM * dg::BN + 255) / 256, plan.npairs);
  GNW_LAUNCH(launch_k(k_dgemm_finalize, g2, 256, 0, s, part, dpairs, plan.npairs, plan.splits, m, beta, C));
  check_launch("dgemm_finalize");
}

// ======================================================================
// Dense Cholesky (linalg.cpp:88-105), single CTA, reference operation order
// ======================================================================
__global__ void __launch_bounds__(1024) k_cholesky(const double* __restrict__ C, double* __restrict__ L, int n,
                                                   int* fail) {
  griddep_wait();
  __shared__ double ljj_s;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (long long t = threadIdx.x; t < static_cast<long long>(n) * n; t += blockDim.x) L[t] = 0.0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      double d = C[static_cast<long long>(j) * n + j];
      for (int k = 0; k < j; ++k) {
        const double l = L[static_cast<long long>(j) * n + k];
        d = d - l * l;
      }
      if (!(d > 0.0)) {
        bad = 1;
      } else {
        const double ljj = sqrt(d);
        L[static_cast<long long>(j) * n + j] = ljj;
        ljj_s = ljj;
      }
    }
    __syncthreads();
    if (bad) break;
    const double ljj = ljj_s;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      double s = C[static_cast<long long>(i) * n + j];
      double* Li = L + static_cast<long long>(i) * n;
      const double* Lj = L + static_cast<long long>(j) * n;
      for (int k = 0; k < j; ++k) s = s - Li[k] * Lj[k];
      Li[j] = s / ljj;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *fail = bad;
}

void cholesky(const double* C, double* L, int n, int* fail, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_cholesky, 1, 1024, 0, s, C, L, n, fail));
  check_launch("cholesky");
}

__global__ void k_symmetrize(double* C, int n) {
  griddep_wait();
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(n) * n) return;
  const int i = static_cast<int>(t / n), j = static_cast<int>(t % n);
  if (j <= i) return;
  const double v = 0.5 * (C[static_cast<long long>(i) * n + j] + C[static_cast<long long>(j) * n + i]);
  C[static_cast<long long>(i) * n + j] = v;
  C[static_cast<long long>(j) * n + i] = v;
}

void symmetrize(double* C, int n, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_symmetrize, grid_for(static_cast<long long>(n) * n), kTpb, 0, s, C, n));
  check_launch("symmetrize");
}

// Y = L^-1 (thread per column), then Cinv = Y^T Y
__global__ void k_trinv(const double* __restrict__ L, double* __restrict__ Y, int n) {
  griddep_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int i = 0; i < j; ++i) Y[static_cast<long long>(i) * n + j] = 0.0;
  for (int i = j; i < n; ++i) {
    double s = (i == j) ? 1.0 : 0.0;
    for (int k = j; k < i; ++k) s = s - L[static_cast<long long>(i) * n + k] * Y[static_cast<long long>(k) * n + j];
    Y[static_cast<long long>(i) * n + j] = s / L[static_cast<long long>(i) * n + i];
  }
}

__global__ void k_syrk_tn(const double* __restrict__ Y, double* __restrict__ Cinv, int n) {
  griddep_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (j >= n || j > i) return;
  double s = 0.0;
#pragma unroll 8
  for (int k = i; k < n; ++k)
    s = s + __ldg(&Y[static_cast<long long>(k) * n + i]) * __ldg(&Y[static_cast<long long>(k) * n + j]);
  Cinv[static_cast<long long>(i) * n + j] = s;
  Cinv[static_cast<long long>(j) * n + i] = s;
}

void cholesky_inverse(const double* L, double* Y, double* Cinv, int n, cudaStream_t s) {
  trinv_blocked(L, Y, n, s);
  dim3 grid(grid_for(n, 128), n);
  GNW_LAUNCH(launch_k(k_syrk_tn, grid, 128, 0, s, Y, Cinv, n));
  check_launch("syrk_tn");
}

__global__ void k_fill_zero(double* p, long long n) {
  griddep_wait();
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = 0.0;
}

void fill_zero(double* p, long long n, cudaStream_t s) {
  if (n <= 0) return;
  GNW_LAUNCH(launch_k(k_fill_zero, std::min<unsigned>(grid_for(n), 148u * 16u), kTpb, 0, s, p, n));
  check_launch("fill_zero");
}

}  // namespace gnw
