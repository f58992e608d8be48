// dense.cu -- m x m dense kernels of the Woodbury setup: blocked Cholesky in the
// reference's exact operation order, and the blocked triangular inverse.
//
// dense_cholesky (linalg.cpp:88-105) computes, for every lower element (i, j),
//     s = C[i][j];  for k < j:  s = s - L[i][k] * L[j][k];  then  s / L[j][j]  (or sqrt)
// i.e. one sequential subtraction chain per element in ascending k.  A right-looking
// blocked factorisation that applies the panel updates k = p .. p+31 to every trailing
// element one subtraction at a time, in ascending k, performs exactly that chain, so
// it is bit-identical to the reference while the critical path shrinks from
// O(m^2) dependent operations to O(m) (one barrier per column inside a panel).
//
//   k_chol_panel  : columns [p, p+w) of the rows i >= p.  One thread per row holds
//                   the row's w panel entries in registers; each CTA also carries the
//                   32 diagonal-block rows (redundantly), whose column k is published
//                   through shared memory once per step.  (A variant that factored the
//                   diagonal block in warp 0 first, fully unrolled, ran 2x slower: its
//                   17k-instruction body stalled on instruction fetch.)
//   k_chol_update : W[i][j] -= L[i][k] L[j][k], k = p .. p+w-1 in order, for the
//                   trailing lower triangle (32 x 32 tiles, panel columns in smem).
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {
constexpr int PW = 32;       // panel width
constexpr int PT = 256;      // panel kernel threads per CTA (32 diagonal-block rows + 224 rows below)
}  // namespace

__global__ void __launch_bounds__(PT) k_chol_panel(double* __restrict__ W, double* __restrict__ L, int n, int p,
                                                   int* fail) {
  griddep_wait();
  __shared__ double colk[PW];
  __shared__ double lcol[PW];  // L[p + t][k] of the diagonal-block rows, divided once per step
  __shared__ int bad;
  if (*fail) return;
  const int w = min(PW, n - p);
  const int t = threadIdx.x;
  // rows owned: t < 32 -> diagonal-block row p + t; else row p + 32 + blockIdx.x*(PT-32) + (t-32)
  int i;
  if (t < PW)
    i = p + t;
  else
    i = p + PW + blockIdx.x * (PT - PW) + (t - PW);
  const bool diag = t < PW;
  const bool valid = diag ? (t < w) : (i < n);
  const bool writer = valid && (diag ? blockIdx.x == 0 : true);
  double row[PW];
#pragma unroll
  for (int c = 0; c < PW; ++c) row[c] = (valid && c < w) ? W[static_cast<long long>(i) * n + p + c] : 0.0;
  if (t == 0) bad = 0;
#pragma unroll
  for (int c = 0; c < PW; ++c) {
    if (c >= w) break;
    // publish column c of the diagonal block (final: all k < p + c already applied)
    __syncthreads();
    if (diag && t < w) colk[t] = row[c];
    __syncthreads();
    const double d = colk[c];
    if (!(d > 0.0)) {
      if (t == 0 && blockIdx.x == 0) *fail = 1;
      return;
    }
    const double ljj = sqrt(d);
    const int k = p + c;
    // the panel rows' L[j][k] = W[j][k] / L[k][k]: one division each, shared by every row
    // below (the same operands, so the same bits as dividing in every thread)
    if (diag && t < w && t > c) lcol[t] = colk[t] / ljj;
    __syncthreads();
    if (!valid) continue;
    if (i == k) {
      if (writer) L[static_cast<long long>(i) * n + i] = ljj;
      row[c] = ljj;
    } else if (i > k) {
      const double lik = row[c] / ljj;
      row[c] = lik;
      if (writer) L[static_cast<long long>(i) * n + k] = lik;
      // remaining panel columns j in (k, p+w), j <= i: W[i][j] -= L[i][k] * L[j][k]
#pragma unroll
      for (int cj = 0; cj < PW; ++cj) {
        if (cj <= c || cj >= w) continue;
        const int j = p + cj;
        if (j > i) continue;
        const double ljk = lcol[cj];  // == L[j][k], bit for bit
        row[cj] = row[cj] - lik * ljk;
      }
    }
  }
}

// trailing update for panel [p, p+w): tiles (ti >= tj) of the rows/cols >= p+w
__global__ void __launch_bounds__(256) k_chol_update(double* __restrict__ W, const double* __restrict__ L, int n,
                                                     int p, int w, const int* fail) {
  griddep_wait();
  __shared__ double Li[32][PW + 1], Lj[32][PW + 1];
  if (*fail) return;
  const int q0 = p + w;
  // blockIdx.x enumerates lower tiles (ti, tj), tj <= ti
  const int t = blockIdx.x;
  int ti = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while (ti * (ti + 1) / 2 > t) --ti;
  const int tj = t - ti * (ti + 1) / 2;
  const int i0 = q0 + ti * 32, j0 = q0 + tj * 32;
  for (int e = threadIdx.x; e < 32 * PW; e += blockDim.x) {
    const int r = e / PW, c = e % PW;
    Li[r][c] = (i0 + r < n && c < w) ? L[static_cast<long long>(i0 + r) * n + p + c] : 0.0;
    Lj[r][c] = (j0 + r < n && c < w) ? L[static_cast<long long>(j0 + r) * n + p + c] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
    const int r = e / 32, c = e % 32;
    const int i = i0 + r, j = j0 + c;
    if (i >= n || j >= n || j > i) continue;
    double s = W[static_cast<long long>(i) * n + j];
    for (int k = 0; k < w; ++k) s = s - Li[r][k] * Lj[c][k];
    W[static_cast<long long>(i) * n + j] = s;
  }
}

__global__ void k_copy_lower_zero_upper(const double* __restrict__ C, double* __restrict__ W, double* __restrict__ L,
                                        int n, int* fail) {
  griddep_wait();
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e == 0) *fail = 0;
  if (e >= static_cast<long long>(n) * n) return;
  W[e] = C[e];
  L[e] = 0.0;
}

void cholesky_blocked(const double* C, double* W, double* L, int n, int* fail, cudaStream_t s) {
  const long long nn = static_cast<long long>(n) * n;
  GNW_LAUNCH(launch_k(k_copy_lower_zero_upper, static_cast<unsigned>((nn + 255) / 256), 256, 0, s, C, W, L, n, fail));
  note_launch("chol_init");
  for (int p = 0; p < n; p += PW) {
    const int w = std::min(PW, n - p);
    const int below = std::max(0, n - p - PW);
    const int ctas = std::max(1, (below + (PT - PW) - 1) / (PT - PW));
    GNW_LAUNCH(launch_k(k_chol_panel, ctas, PT, 0, s, W, L, n, p, fail));
    note_launch("chol_panel");
    const int rem = n - (p + w);
    if (rem > 0) {
      const int nt = (rem + 31) / 32;
      GNW_LAUNCH(launch_k(k_chol_update, nt * (nt + 1) / 2, 256, 0, s, W, L, n, p, w, fail));
      note_launch("chol_update");
    }
  }
}

// --------------------------------------------------------------------------
// Y = L^-1 by block rows of 32: for rows i in [p, p+32) and columns j <= i,
//   s = [i == j] - sum_{k in [j, p)} L[i][k] Y[k][j]      (previous block rows)
// then the 32 x 32 diagonal block is solved row by row through shared memory.
__global__ void __launch_bounds__(1024) k_trinv_block(const double* __restrict__ L, double* __restrict__ Y, int n,
                                                      int p) {
  griddep_wait();
  const int r = threadIdx.x;               // row within block (a warp holds one column's 32 rows)
  const int jc = threadIdx.y;              // column within chunk
  const int i = p + r;
  const int j = blockIdx.x * 32 + jc;      // global column
  const bool act = i < n && j <= i;
  // s = [i == j] - sum_{k < p} L[i][k] Y[k][j], k ascending.  Rows k < p of Y were written by
  // earlier launches.  The sum runs over 32 x 32 shared-memory tiles of L and Y (one global
  // load of each per thread per tile) instead of p dependent L2 loads per thread; Y[k][j] = 0
  // for k < j, so starting every column of the chunk at the chunk's first column only adds
  // exact zeros and leaves the rounding unchanged.
  __shared__ double Ls[32][33], Ys[32][33];
  double s = (act && i == j) ? 1.0 : 0.0;
  for (int k0 = blockIdx.x * 32; k0 < p; k0 += 32) {
    const int kk = min(32, p - k0);
    Ls[jc][r] = (p + jc < n && r < kk) ? __ldg(&L[static_cast<long long>(p + jc) * n + k0 + r]) : 0.0;
    Ys[jc][r] = (jc < kk && blockIdx.x * 32 + r < n) ? __ldg(&Y[static_cast<long long>(k0 + jc) * n + blockIdx.x * 32 + r]) : 0.0;
    __syncthreads();
    if (act)
      for (int t = 0; t < kk; ++t) s = s - Ls[r][t] * Ys[t][jc];
    __syncthreads();
  }
  // the 32 x 32 diagonal block, row by row: within a column only the warp's own lanes
  // interact, so the quotient of row rr reaches the rows below by shuffle (no CTA barrier)
  const int w = min(32, n - p);
  // the diagonal block L[p + r][p + rr] staged once (the per-step load of L[i][p + rr] was
  // 32 lines per warp instruction in this column-per-warp layout)
  Ls[jc][r] = (p + jc < n && r < w) ? L[static_cast<long long>(p + jc) * n + p + r] : 1.0;
  __syncthreads();
  for (int rr = 0; rr < w; ++rr) {
    double y = 0.0;
    if (r == rr) {
      y = act ? s / Ls[r][r] : 0.0;
      if (i < n && j < n) Y[static_cast<long long>(i) * n + j] = act ? y : 0.0;
    }
    y = __shfl_sync(0xffffffffu, y, rr);
    if (r > rr && act && j <= p + rr) s = s - Ls[r][rr] * y;
  }
}

void trinv_blocked(const double* L, double* Y, int n, cudaStream_t s) {
  for (int p = 0; p < n; p += 32) {
    const int chunks = (std::min(n, p + 32) + 31) / 32;
    GNW_LAUNCH(launch_k(k_trinv_block, chunks, dim3(32, 32), 0, s, L, Y, n, p));
    note_launch("trinv_block");
  }
}

}  // namespace gnw
