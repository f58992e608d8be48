// vcycle_wide.cu -- V-cycle kernels for levels with several nonzeros per row.
//
// Thread-per-row CSR (kernels.cu) reproduces the reference's sequential row sums
// bit for bit, but a thread walking a row of 10..400 entries serialises its
// dependent loads and its loads are strided across the warp (C3, ncu cold-cache:
// level 1 of the hierarchy, 13 entries per row, ran at 3.9 TB/s; warp-per-row on
// level 2, 26 per row, at 1.5 TB/s because 6 of 32 lanes idled and every warp
// carried a whole row's latency chain for 26 entries).  Here a group of G lanes
// (G = 2..32, picked per matrix from its mean row length, DLevel::gA/gP/gR) owns
// a row: lane j accumulates the entries k = start + j, start + j + G, ... in
// order, then the group combines through the xor butterfly (G/2, ..., 1).
// That order is deterministic but not the reference's; GNW_COARSE_CHOLESKY
// ("exact") mode never uses these kernels.
//
// The multi-RHS kernels (H = S^-1 J^T, b interleaved columns) run one thread per
// (row, column) in the reference's sequential order (kernels.cu, vcycle_batch.cu).
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {

// G lanes own a row (G = 2..32, a power of two): lane j of the group accumulates the entries
// k = start + j, start + j + G, ... in order, then the group combines through the xor
// butterfly (G/2, ..., 1).  G = 32 is the warp-per-row order.  Rows outside the matrix
// still join the shuffles (full mask) with a zero partial.
template <int G, class F>
__device__ __forceinline__ double group_row(const DCsr& A, int i, int sub, bool valid, F f) {
  double acc = 0.0;
  if (valid) {
    const int k1 = A.rowptr[i + 1];
    // unrolled so several (index -> value) load chains are in flight per lane
#pragma unroll 4
    for (int k = A.rowptr[i] + sub; k < k1; k += G) acc = acc + __ldg(&A.vals[k]) * f(__ldg(&A.cols[k]));
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

constexpr int kGroupTpb = 256;

template <int G>
struct GroupIdx {
  int i, sub;
  __device__ GroupIdx() : i(blockIdx.x * (kGroupTpb / G) + threadIdx.x / G), sub(threadIdx.x % G) {}
};

}  // namespace

// --------------------------------------------------------------- single RHS
template <int G>
__global__ void __launch_bounds__(kGroupTpb) k_vcg_down(DCsr A, const double* __restrict__ wd, VSel rs,
                                                        double* __restrict__ resid, const MinresState* st) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const GroupIdx<G> g;
  const bool ok = g.i < A.n_rows;
  const double s = group_row<G>(A, g.i, g.sub, ok, [&](int c) { return __ldg(&wd[c]) * r[c]; });
  if (ok && g.sub == 0) resid[g.i] = r[g.i] + (-1.0 * s);
}

template <int G>
__global__ void __launch_bounds__(kGroupTpb) k_vcg_restrict(DCsr R, const double* __restrict__ resid,
                                                            double* __restrict__ rc) {
  griddep_wait();
  const GroupIdx<G> g;
  const bool ok = g.i < R.n_rows;
  const double s = group_row<G>(R, g.i, g.sub, ok, [&](int c) { return resid[c]; });
  if (ok && g.sub == 0) rc[g.i] = s;
}

template <int G>
__global__ void __launch_bounds__(kGroupTpb) k_vcg_up1(DCsr P, const double* __restrict__ wd, VSel rs,
                                                       const double* __restrict__ ec, double* __restrict__ x,
                                                       const MinresState* st) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const GroupIdx<G> g;
  const bool ok = g.i < P.n_rows;
  const double s = group_row<G>(P, g.i, g.sub, ok, [&](int c) { return ec[c]; });
  if (ok && g.sub == 0) x[g.i] = __ldg(&wd[g.i]) * r[g.i] + 1.0 * s;
}

template <int G>
__global__ void __launch_bounds__(kGroupTpb) k_vcg_up2(DCsr A, const double* __restrict__ wd, VSel rs,
                                                       const double* __restrict__ x, double* __restrict__ out,
                                                       const MinresState* st) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const GroupIdx<G> g;
  const bool ok = g.i < A.n_rows;
  const double s = group_row<G>(A, g.i, g.sub, ok, [&](int c) { return x[c]; });
  if (ok && g.sub == 0) {
    const double res = r[g.i] + (-1.0 * s);
    out[g.i] = x[g.i] + __ldg(&wd[g.i]) * res;
  }
}

// ------------------------------------------------------- collapsed coarse tail
// Y = M X for the batched V-cycle (X, Y: n x b row-major = b interleaved columns).  A plain
// shared-memory tiled FP64 GEMM: 32 x 64 output tiles (2 x 4 per thread), 32-deep k steps.
// (The previous one-thread-per-output loop ran at 2.7 TFLOP/s: 248 us at C2, n = 1147, b = 256.)
namespace {
constexpr int kDti = 32, kDtq = 64, kDtk = 32;
}
__global__ void __launch_bounds__(256) k_dense_apply_batch(const double* __restrict__ M, int n,
                                                           const double* __restrict__ X, double* __restrict__ Y,
                                                           int b) {
  griddep_wait();
  __shared__ double Ms[kDtk][kDti + 2];  // Ms[k][i] = M[i0 + i][k0 + k]
  __shared__ __align__(16) double Xs[kDtk][kDtq];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int i0 = blockIdx.x * kDti, q0 = blockIdx.y * kDtq;
  double acc[2][4] = {};
  for (int k0 = 0; k0 < n; k0 += kDtk) {
#pragma unroll
    for (int u = 0; u < (kDti * kDtk) / 256; ++u) {
      const int e = tid + 256 * u, r = e / kDtk, c = e % kDtk;
      Ms[c][r] = (i0 + r < n && k0 + c < n) ? __ldg(&M[static_cast<long long>(i0 + r) * n + k0 + c]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < (kDtk * kDtq) / 256; ++u) {
      const int e = tid + 256 * u, r = e / kDtq, c = e % kDtq;
      Xs[r][c] = (k0 + r < n && q0 + c < b) ? X[static_cast<long long>(k0 + r) * b + q0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < kDtk; ++k) {
      const double a0 = Ms[k][2 * ty], a1 = Ms[k][2 * ty + 1];
      const double2 x01 = *reinterpret_cast<const double2*>(&Xs[k][4 * tx]);
      const double2 x23 = *reinterpret_cast<const double2*>(&Xs[k][4 * tx + 2]);
      const double xv[4] = {x01.x, x01.y, x23.x, x23.y};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[0][c] = __fma_rn(a0, xv[c], acc[0][c]);
        acc[1][c] = __fma_rn(a1, xv[c], acc[1][c]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int i = i0 + 2 * ty + a;
    if (i >= n) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int q = q0 + 4 * tx + c;
      if (q < b) Y[static_cast<long long>(i) * b + q] = acc[a][c];
    }
  }
}

__global__ void k_identity_rows(double* __restrict__ I, int n) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < static_cast<long long>(n) * n) I[k] = (k / n == k % n) ? 1.0 : 0.0;
}

__global__ void k_transpose_square(const double* __restrict__ A, double* __restrict__ T, int n) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < static_cast<long long>(n) * n) T[k] = A[(k % n) * n + k / n];
}

// ------------------------------------------------------------------ launchers
// G = the largest power of two <= (mean entries per row) / T, in [1, 32]; T = 4 by default
// (C3 hierarchy: 4 -> 1, 10 -> 2, 13 -> 2, 26 -> 4, 72 -> 16, 150+ -> 32; standalone V-cycle
// T = 2 / 3 / 4 / 6: C3 0.951 / 0.906 / 0.856 / 0.872 ms, C5 0.294 / 0.287 / 0.285 / 0.300 ms,
// C2 0.105 / 0.108 / 0.109 / 0.118 ms; warp-per-row on every level >= 24 per row: 1.04 / 0.40 / 0.12).
int vc_group_lanes(long long nnz, long long rows) {
  static const double T = [] {
    const char* e = std::getenv("GNW_VC_T");
    return e ? std::atof(e) : 4.0;
  }();
  if (rows <= 0) return 1;
  const double per = static_cast<double>(nnz) / static_cast<double>(rows) / T;
  int g = 1;
  while (g < 32 && 2 * g <= per) g *= 2;
  return g;
}

static unsigned ggrid(int rows, int G) {
  const int per = kGroupTpb / G;
  return static_cast<unsigned>((rows + per - 1) / per);
}

#define GNW_G_DISPATCH(G, KERNEL, ROWS, ...)                                                         \
  switch (G) {                                                                                       \
    case 2: GNW_LAUNCH(launch_k(KERNEL<2>, ggrid(ROWS, 2), kGroupTpb, 0, __VA_ARGS__)); break;     \
    case 4: GNW_LAUNCH(launch_k(KERNEL<4>, ggrid(ROWS, 4), kGroupTpb, 0, __VA_ARGS__)); break;     \
    case 8: GNW_LAUNCH(launch_k(KERNEL<8>, ggrid(ROWS, 8), kGroupTpb, 0, __VA_ARGS__)); break;     \
    case 16: GNW_LAUNCH(launch_k(KERNEL<16>, ggrid(ROWS, 16), kGroupTpb, 0, __VA_ARGS__)); break;  \
    default: GNW_LAUNCH(launch_k(KERNEL<32>, ggrid(ROWS, 32), kGroupTpb, 0, __VA_ARGS__)); break;  \
  }

void vcg_down(const DLevel& L, VSel r, double* resid, const MinresState* st, cudaStream_t s) {
  GNW_G_DISPATCH(L.gA, k_vcg_down, L.n, s, L.A, L.wd, r, resid, st);
  note_launch("vcg_down");
}
void vcg_restrict(const DLevel& L, const double* resid, double* rc, cudaStream_t s) {
  GNW_G_DISPATCH(L.gR, k_vcg_restrict, L.R.n_rows, s, L.R, resid, rc);
  note_launch("vcg_restrict");
}
void vcg_up1(const DLevel& L, VSel r, const double* ec, double* x, const MinresState* st, cudaStream_t s) {
  GNW_G_DISPATCH(L.gP, k_vcg_up1, L.n, s, L.P, L.wd, r, ec, x, st);
  note_launch("vcg_up1");
}
void vcg_up2(const DLevel& L, VSel r, const double* x, double* out, const MinresState* st, cudaStream_t s) {
  GNW_G_DISPATCH(L.gA, k_vcg_up2, L.n, s, L.A, L.wd, r, x, out, st);
  note_launch("vcg_up2");
}
void dense_seq_batch(const double* M, int n, const double* X, double* Y, int b, cudaStream_t s) {
  dim3 grid((n + kDti - 1) / kDti, (b + kDtq - 1) / kDtq);
  GNW_LAUNCH(launch_k(k_dense_apply_batch, grid, 256, 0, s, M, n, X, Y, b));
  note_launch("dense_apply_batch");
}
void identity_rows(double* I, int n, cudaStream_t s) {
  const long long t = static_cast<long long>(n) * n;
  k_identity_rows<<<static_cast<unsigned>((t + 255) / 256), 256, 0, s>>>(I, n);
  note_launch("identity_rows");
}
void transpose_square(const double* A, double* T, int n, cudaStream_t s) {
  const long long t = static_cast<long long>(n) * n;
  k_transpose_square<<<static_cast<unsigned>((t + 255) / 256), 256, 0, s>>>(A, T, n);
  note_launch("transpose_square");
}

}  // namespace gnw
