// vcycle_wide.cu -- V-cycle kernels for WIDE levels (many nonzeros per row).
//
// Thread-per-row CSR (kernels.cu) reproduces the reference's sequential row sums
// bit for bit, but on the coarse SA-AMG levels rows hold 25..400 entries and
// only a few hundred rows exist (C2: 5541 x 72, 1147 x 150, then 396..171 dense
// rows), so one thread walking a row serialises hundreds of dependent loads.
// Here a warp owns a row: lane l accumulates the entries k = start + l,
// start + l + 32, ... in order, then the lanes combine through the xor
// butterfly (16, 8, 4, 2, 1).  That order is deterministic but not the
// reference's; GNW_COARSE_CHOLESKY ("exact") mode never uses these kernels.
//
// The multi-RHS kernels (H = S^-1 J^T, b interleaved columns) run one thread per
// (row, column) and EMULATE the same lane partition and butterfly with 32
// register partials, so every column of a batched V-cycle is bit-identical to
// the single-RHS V-cycle of the MINRES loop.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {

template <class F>
__device__ __forceinline__ double warp_row(const DCsr& A, int i, int lane, F f) {
  double acc = 0.0;
  const int k1 = A.rowptr[i + 1];
  // unrolled so several (index -> value) load chains are in flight per lane
#pragma unroll 4
  for (int k = A.rowptr[i] + lane; k < k1; k += 32) acc = acc + __ldg(&A.vals[k]) * f(__ldg(&A.cols[k]));
  double v[1] = {acc};
  warp_reduce<1>(v);
  return v[0];
}

constexpr int kRowsPerBlock = 8;  // 8 warps, one row each

}  // namespace

// --------------------------------------------------------------- single RHS
__global__ void __launch_bounds__(256) k_vcw_down(DCsr A, const double* __restrict__ wd, VSel rs,
                                                  double* __restrict__ resid, const MinresState* st) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const int i = blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= A.n_rows) return;
  const double s = warp_row(A, i, lane, [&](int c) { return __ldg(&wd[c]) * r[c]; });
  if (lane == 0) resid[i] = r[i] + (-1.0 * s);
}

__global__ void __launch_bounds__(256) k_vcw_restrict(DCsr R, const double* __restrict__ resid,
                                                      double* __restrict__ rc) {
  griddep_wait();
  const int a = blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (a >= R.n_rows) return;
  const double s = warp_row(R, a, lane, [&](int c) { return resid[c]; });
  if (lane == 0) rc[a] = s;
}

__global__ void __launch_bounds__(256) k_vcw_up1(DCsr P, const double* __restrict__ wd, VSel rs,
                                                 const double* __restrict__ ec, double* __restrict__ x,
                                                 const MinresState* st) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const int i = blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= P.n_rows) return;
  const double s = warp_row(P, i, lane, [&](int c) { return ec[c]; });
  if (lane == 0) x[i] = __ldg(&wd[i]) * r[i] + 1.0 * s;
}

__global__ void __launch_bounds__(256) k_vcw_up2(DCsr A, const double* __restrict__ wd, VSel rs,
                                                 const double* __restrict__ x, double* __restrict__ out,
                                                 const MinresState* st) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const int i = blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= A.n_rows) return;
  const double s = warp_row(A, i, lane, [&](int c) { return x[c]; });
  if (lane == 0) {
    const double res = r[i] + (-1.0 * s);
    out[i] = x[i] + __ldg(&wd[i]) * res;
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
static unsigned wgrid(int rows) { return static_cast<unsigned>((rows + kRowsPerBlock - 1) / kRowsPerBlock); }

void vcw_down(const DLevel& L, VSel r, double* resid, const MinresState* st, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_vcw_down, wgrid(L.n), 256, 0, s, L.A, L.wd, r, resid, st));
  note_launch("vcw_down");
}
void vcw_restrict(const DLevel& L, const double* resid, double* rc, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_vcw_restrict, wgrid(L.R.n_rows), 256, 0, s, L.R, resid, rc));
  note_launch("vcw_restrict");
}
void vcw_up1(const DLevel& L, VSel r, const double* ec, double* x, const MinresState* st, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_vcw_up1, wgrid(L.n), 256, 0, s, L.P, L.wd, r, ec, x, st));
  note_launch("vcw_up1");
}
void vcw_up2(const DLevel& L, VSel r, const double* x, double* out, const MinresState* st, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_vcw_up2, wgrid(L.n), 256, 0, s, L.A, L.wd, r, x, out, st));
  note_launch("vcw_up2");
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
