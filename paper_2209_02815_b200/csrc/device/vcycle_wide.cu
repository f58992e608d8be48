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
// Y[:, q] = M X[:, q], one thread per (row, column): X loads coalesced over the columns,
// M rows broadcast within a warp.
__global__ void __launch_bounds__(256) k_dense_seq_batch(const double* __restrict__ M, int n,
                                                         const double* __restrict__ X, double* __restrict__ Y, int b) {
  griddep_wait();
  const int i = blockIdx.x * 8 + threadIdx.y;
  const int q = blockIdx.y * 32 + threadIdx.x;
  if (i >= n || q >= b) return;
  const double* __restrict__ Mi = M + static_cast<long long>(i) * n;
  // four interleaved partial sums (default mode only; four loads in flight per thread)
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int j = 0;
  for (; j + 4 <= n; j += 4) {
    a0 = a0 + __ldg(&Mi[j]) * X[static_cast<long long>(j) * b + q];
    a1 = a1 + __ldg(&Mi[j + 1]) * X[static_cast<long long>(j + 1) * b + q];
    a2 = a2 + __ldg(&Mi[j + 2]) * X[static_cast<long long>(j + 2) * b + q];
    a3 = a3 + __ldg(&Mi[j + 3]) * X[static_cast<long long>(j + 3) * b + q];
  }
  for (; j < n; ++j) a0 = a0 + __ldg(&Mi[j]) * X[static_cast<long long>(j) * b + q];
  Y[static_cast<long long>(i) * b + q] = (a0 + a1) + (a2 + a3);
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
  dim3 grid((n + 7) / 8, (b + 31) / 32), block(32, 8);
  GNW_LAUNCH(launch_k(k_dense_seq_batch, grid, block, 0, s, M, n, X, Y, b));
  note_launch("dense_seq_batch");
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
