// common.cuh -- shared device-side definitions for the gnw kernels (sm_100a).
//
// Floating point: the library is compiled with --fmad=false so that every
// a*b+c written in the reference's evaluation order rounds exactly like the
// reference's x86-64 build (no FMA contraction).  Kernels that do not need
// reference-order rounding (tensor-core DGEMM, reductions) say so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

namespace gnw {

constexpr int kWarp = 32;
// largest m whose m-vector is staged in shared memory by the dense sweeps (gnw_set_jacobian cap)
constexpr int kMaxStageM = 8192;

// Programmatic dependent launch: every kernel starts with griddep_wait(), so a
// launch may be issued (and its CTAs made resident) while its predecessor on the
// stream drains; the wait returns once the predecessor has completed and its
// memory is visible.  Without the launch attribute the wait is a no-op.
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  // allow the next kernel's CTAs to be scheduled once every CTA of this grid has started
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

extern bool g_pdl;  // launch with programmatic stream serialization (env GNW_PDL, default on)

// Opts `fn` in to `bytes` of dynamic shared memory on the CURRENT device, once per
// (kernel, device) pair; thread-safe (kernels.cu).  Throws on failure.
void smem_optin(const void* fn, int bytes);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// MINRES loop status codes (device -> host).
enum : int {
  kRunning = 0,
  kVerify = 1,      // recurred residual <= tol: host verifies with the true residual
  kExhausted = 2,   // gamma_{j+1} <= 1e-13 gamma_1 (minres.cpp:122)
  kMaxit = 3,
  kErrNotPD = 4,    // "minres: preconditioner is not positive definite"
  kErrStagnated = 5 // "minres: breakdown (stagnated rotation)"
};

// Scalar state of the MINRES recurrence (minres.cpp:61-68), device resident.
struct MinresState {
  double gamma_prev, gamma_cur, gamma_next;
  double c_prev, c_cur, c_next;
  double s_prev, s_cur, s_next;
  double eta, gamma1, bnorm, tol, exhausted_tol;
  double delta;          // <A zhat, zhat>
  double inv_gamma;      // 1 / gamma_cur  (zhat = z * inv_gamma)
  double coef_v1, coef_v2; // -delta/gamma_cur, -gamma_cur/gamma_prev
  double alpha2, alpha3, inv_alpha1, tau;
  double rel;            // ||r|| / ||b|| after the update
  double scratch[8];
  long long j;           // iteration index (1-based)
  long long maxit;
  long long iterations;  // report.iterations
  int status;
  int pad;
};

// A vector argument that is either a fixed buffer or a slot of a device ring
// indexed by the MINRES iteration counter: p[(j + off) % mod].
struct VSel {
  double* p[3];
  int mod;
  int off;
};

__host__ inline VSel vfixed(double* x) {
  VSel s;
  s.p[0] = s.p[1] = s.p[2] = x;
  s.mod = 1;
  s.off = 0;
  return s;
}
__host__ inline VSel vring(double* const* ring, int mod, int off) {
  VSel s;
  for (int k = 0; k < 3; ++k) s.p[k] = ring[k < mod ? k : 0];
  s.mod = mod;
  s.off = off;
  return s;
}

__device__ __forceinline__ double* vsel(const VSel& s, const MinresState* st) {
  if (s.mod == 1) return s.p[0];
  const int idx = (int)((st->j + s.off) % s.mod);
  // select without dynamic indexing (keeps the struct in registers, no stack frame)
  double* p = s.p[0];
  if (idx == 1) p = s.p[1];
  if (idx == 2) p = s.p[2];
  return p;
}

// Device CSR (int32 indices).
struct DCsr {
  int n_rows = 0, n_cols = 0, nnz = 0;
  int* rowptr = nullptr;
  int* cols = nullptr;
  double* vals = nullptr;
};

// Device sliced-ELL copy of a CSR matrix (SELL-32): rows in slices of 32, each slice stores
// `width` entries per row column-major, entry k of row r at
// (r / 32) * 32 * width + k * 32 + r % 32.  A warp's k-th loads of cols/vals are then one
// contiguous 128 B / 256 B segment, and every entry load of a row is independent of the
// others (no rowptr -> cols -> x chain per entry).  Entries keep the CSR order of their row;
// padding has col = -1 and is skipped, so a row sum adds exactly the CSR terms in the CSR
// order (bit-identical to the CSR loop).  width = 0: not built (row longer than kSellMaxWidth).
constexpr int kSellMaxWidth = 8;
// Compact encodings of the VALUES (the saddle operator's Q, D, D^T; context.cu):
//   signed_cols: every value is +1 or -1 (D, D^T: cell_edge_signs) -- no value array; entry
//     (c, -1) is stored as column -c - 2 (padding keeps -1);
//   codes: at most 256 distinct values (Q of a unit-square mesh has four: 2/3, 1/3, -1/6, 0) --
//     one byte per entry indexing `table`.
// The decoded value is the same double, so every product and sum is bit-identical; the saddle
// kernel then streams 4-5 bytes per entry instead of 12.
struct DSell {
  int n_rows = 0, width = 0;
  const int* cols = nullptr;
  const double* vals = nullptr;
  const unsigned char* codes = nullptr;
  const double* table = nullptr;
  int signed_cols = 0;
};

// Lane-ELL copy of a CSR matrix for the G-lanes-per-row kernels of the loop's V-cycle
// (vcycle_fused.cu).  A warp holds 32 / G rows; lane (row % (32 / G)) * G + j sums entries
// j, j + G, ... of its row, exactly like the CSR kernels, so entry e of row r sits at
//   ((r / (32 / G)) * width + e / G) * 32 + (r % (32 / G)) * G + e % G
// with `width` entries per lane (the longest row, rounded up).  The k-th load of a warp is one
// contiguous 128-byte segment and no rowptr is read first.  Padding (0xffffffff) comes last in
// its lane, so every lane adds the CSR terms in the CSR order: bit-identical sums.
// Each entry is ONE 32-bit word: the level operators of a structured mesh hold few distinct
// doubles (C2: 11 in S_0, 79 in T_0, 4172 in T_3), so the value is a code into `table` (the
// decoded double is the same bits) packed above the column: word = code << shift | col.
// Built only when column bits + code bits <= 31; otherwise the level keeps its CSR kernels.
// Slices are allocated for every warp of the launch grid (multiples of 8 warps).
struct DLell {
  int n_rows = 0, width = 0, lanes = 0, shift = 0;
  unsigned mask = 0;
  const unsigned* words = nullptr;
  const double* table = nullptr;
};

// sum_k vals[k] * (x[off + cols[k]] * sc)  (sc applied only when scaled), in CSR order
template <int W>
__device__ __forceinline__ void sell_load(const DSell& A, long long row, int (&c)[W], double (&v)[W]);

template <int W>
__device__ __forceinline__ double sell_row_w(const DSell& A, long long row, const double* __restrict__ x,
                                             long long off, bool scaled, double sc) {
  int c[W];
  double v[W];
  sell_load<W>(A, row, c, v);
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const double xv = c[k] >= 0 ? x[off + c[k]] : 0.0;
    v[k] = v[k] * (scaled ? xv * sc : xv);  // --fmad=false: same rounding as the CSR loop
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < W; ++k)
    if (c[k] >= 0) s = s + v[k];
  return s;
}

// the two halves of sell_row_w, so that the entry loads of several matrices (and of the
// MINRES state) are all in flight before the first gather
template <int W>
__device__ __forceinline__ void sell_load(const DSell& A, long long row, int (&c)[W], double (&v)[W]) {
  const long long base = (row >> 5) * 32LL * W + (row & 31);
  if (A.signed_cols) {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int q = __ldg(A.cols + base + 32 * k);
      c[k] = q >= -1 ? q : -q - 2;
      v[k] = q >= -1 ? 1.0 : -1.0;
    }
  } else if (A.codes) {
    unsigned char h[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
      c[k] = __ldg(A.cols + base + 32 * k);
      h[k] = __ldg(A.codes + base + 32 * k);
    }
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = __ldg(A.table + h[k]);
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      c[k] = __ldg(A.cols + base + 32 * k);
      v[k] = __ldg(A.vals + base + 32 * k);
    }
  }
}
template <int W>
__device__ __forceinline__ double sell_finish(const int (&c)[W], double (&v)[W], const double* __restrict__ x,
                                              long long off, bool scaled, double sc) {
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const double xv = c[k] >= 0 ? x[off + c[k]] : 0.0;
    v[k] = v[k] * (scaled ? xv * sc : xv);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < W; ++k)
    if (c[k] >= 0) s = s + v[k];
  return s;
}

// sell_finish with the multiplicand of entry (row, c) given by f(c)
template <int W, class F>
__device__ __forceinline__ double sell_finish_f(const int (&c)[W], double (&v)[W], F f) {
#pragma unroll
  for (int k = 0; k < W; ++k) v[k] = v[k] * (c[k] >= 0 ? f(c[k]) : 0.0);
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < W; ++k)
    if (c[k] >= 0) s = s + v[k];
  return s;
}

__device__ __forceinline__ double sell_row(const DSell& A, long long row, const double* __restrict__ x, long long off,
                                           bool scaled, double sc) {
  switch (A.width) {
    case 1: return sell_row_w<1>(A, row, x, off, scaled, sc);
    case 2: return sell_row_w<2>(A, row, x, off, scaled, sc);
    case 3: return sell_row_w<3>(A, row, x, off, scaled, sc);
    case 4: return sell_row_w<4>(A, row, x, off, scaled, sc);
    case 5: return sell_row_w<5>(A, row, x, off, scaled, sc);
    case 6: return sell_row_w<6>(A, row, x, off, scaled, sc);
    case 7: return sell_row_w<7>(A, row, x, off, scaled, sc);
    default: return sell_row_w<8>(A, row, x, off, scaled, sc);
  }
}

// ---------------------------------------------------------------- reductions
// Deterministic block reduction: warp xor-tree, then warps in index order.
template <int NV>
__device__ __forceinline__ void warp_reduce(double (&v)[NV]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
}

// Reduces NV values over the block; result valid in thread 0.  smem needs
// NV * (blockDim/32) doubles.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double* smem) {
  warp_reduce<NV>(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) smem[warp * NV + k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += smem[w * NV + k];
      v[k] = s;
    }
  }
  __syncthreads();
}

// Grid-wide deterministic reduction via the last-arriving block.  Each block
// writes its NV partials to part[blockIdx.x * NV + k]; the last block sums
// the partials in block-index order (fixed tree, independent of arrival
// order) and returns true in ALL its threads with `out` (thread 0) holding
// the totals.  `counter` must be zero at launch; it is reset by the last block.
template <int NV>
__device__ bool grid_reduce_last(double (&v)[NV], double* part, unsigned int* counter, double* smem,
                                 double (&out)[NV]) {
  block_reduce<NV>(v, smem);
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) part[blockIdx.x * NV + k] = v[k];
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  // U strided partials per thread loaded at once, then added in the same order as the plain
  // strided loop (same bits): the last block no longer pays one L2 round trip per partial
  // while every other SM idles (k_saddle at n = 1024: 20488 blocks -> 80 round trips)
  constexpr int U = NV >= 3 ? 2 : 8;  // NV = 3 kernels run at 32 registers
  const int G = static_cast<int>(gridDim.x), bs = static_cast<int>(blockDim.x);
  for (int b0 = threadIdx.x; b0 < G; b0 += U * bs) {
    double t[U][NV];
#pragma unroll
    for (int j = 0; j < U; ++j)
#pragma unroll
      for (int k = 0; k < NV; ++k) t[j][k] = b0 + j * bs < G ? __ldcg(&part[(b0 + j * bs) * NV + k]) : 0.0;
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (b0 + j * bs < G)
#pragma unroll
        for (int k = 0; k < NV; ++k) acc[k] += t[j][k];
  }
  block_reduce<NV>(acc, smem);
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = acc[k];
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

}  // namespace gnw

#define GNW_LAUNCH(expr)                                                                        \
  do {                                                                                          \
    cudaError_t e__ = (expr);                                                                   \
    if (e__ != cudaSuccess)                                                                     \
      throw std::runtime_error(std::string("kernel launch failed: ") + cudaGetErrorString(e__)); \
  } while (0)

#define GNW_CUDA_CHECK(expr)                                                  \
  do {                                                                           \
    cudaError_t e__ = (expr);                                                    \
    if (e__ != cudaSuccess) throw ::gnw::DeviceError(#expr, e__, __FILE__, __LINE__); \
  } while (0)
