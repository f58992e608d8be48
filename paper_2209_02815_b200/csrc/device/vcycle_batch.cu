// vcycle_batch.cu -- batched (multi-RHS) V-cycle kernels for NARROW levels, two
// interleaved columns per thread (16-byte loads).  Per column the arithmetic is
// exactly the thread-per-row sequence of kernels.cu (reference order), so a
// batched V-cycle column is bit-identical to the single-RHS V-cycle.
//
// Layout X[row * ld + q]: a warp covers 64 consecutive columns of one row, so every
// gather of a neighbour row is a coalesced 512-byte segment; the CSR indices of
// the row are warp-uniform loads.  The entry loop is unrolled so the index loads
// of several entries are in flight together (level 0 carries 4-5 entries per row).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// Lanes per row: a warp covers 64V columns of one row when b allows; a narrower batch (C3
// runs b = 32 for memory) packs 32 / lanes rows into each warp instead of idling lanes.
__host__ __device__ __forceinline__ int mvc_lanes(int b, int V) {
  const int need = (b + 2 * V - 1) / (2 * V);
  int l = 1;
  while (l < 32 && l < need) l *= 2;
  return l;
}
template <int V>
struct MvcIdx {
  int row, q;
  __device__ MvcIdx(int lsh) {  // lsh = log2(lanes per row), from the launcher
    row = (((blockIdx.x * 8 + threadIdx.y) << 5) + threadIdx.x) >> lsh;
    q = 2 * V * ((blockIdx.y << lsh) + (threadIdx.x & ((1 << lsh) - 1)));
  }
};
}  // namespace

// V double2 vectors (2V consecutive columns) per thread.  V = 2 doubles the bytes each
// thread has in flight behind one (row pointer -> column index -> gather) latency chain:
// the level-0 kernels were long-scoreboard bound at 3.4 TB/s with V = 1 (C2, ncu).
template <int V>
__global__ void __launch_bounds__(256) k_mvc2_down(DCsr A, const double* __restrict__ wd,
                                                   const double* __restrict__ r, int ldr,
                                                   double* __restrict__ resid, int b, int lsh) {
  griddep_wait();
  const MvcIdx<V> ix(lsh);
  const int i = ix.row, q = ix.q;
  if (i >= A.n_rows || q >= b) return;
  double sx[V], sy[V];
#pragma unroll
  for (int v = 0; v < V; ++v) sx[v] = sy[v] = 0.0;
  const int k0 = A.rowptr[i], k1 = A.rowptr[i + 1];
#pragma unroll 4
  for (int k = k0; k < k1; ++k) {
    const int c = __ldg(&A.cols[k]);
    const double a = __ldg(&A.vals[k]), w = __ldg(&wd[c]);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double2 x = ld2(r + static_cast<long long>(c) * ldr + q + 2 * v);
      sx[v] = sx[v] + a * (w * x.x);
      sy[v] = sy[v] + a * (w * x.y);
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double2 ri = ld2(r + static_cast<long long>(i) * ldr + q + 2 * v);
    st2(resid + static_cast<long long>(i) * b + q + 2 * v, make_double2(ri.x + (-1.0 * sx[v]), ri.y + (-1.0 * sy[v])));
  }
}

template <int V>
__global__ void __launch_bounds__(256) k_mvc2_restrict(DCsr R, const double* __restrict__ resid,
                                                       double* __restrict__ rc, int b, int lsh) {
  griddep_wait();
  const MvcIdx<V> ix(lsh);
  const int a = ix.row, q = ix.q;
  if (a >= R.n_rows || q >= b) return;
  double sx[V], sy[V];
#pragma unroll
  for (int v = 0; v < V; ++v) sx[v] = sy[v] = 0.0;
  const int k0 = R.rowptr[a], k1 = R.rowptr[a + 1];
#pragma unroll 4
  for (int k = k0; k < k1; ++k) {
    const int c = __ldg(&R.cols[k]);
    const double val = __ldg(&R.vals[k]);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double2 x = ld2(resid + static_cast<long long>(c) * b + q + 2 * v);
      sx[v] = sx[v] + val * x.x;
      sy[v] = sy[v] + val * x.y;
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) st2(rc + static_cast<long long>(a) * b + q + 2 * v, make_double2(sx[v], sy[v]));
}

template <int V>
__global__ void __launch_bounds__(256) k_mvc2_up1(DCsr P, const double* __restrict__ wd,
                                                  const double* __restrict__ r, int ldr,
                                                  const double* __restrict__ ec, double* __restrict__ x, int b, int lsh) {
  griddep_wait();
  const MvcIdx<V> ix(lsh);
  const int i = ix.row, q = ix.q;
  if (i >= P.n_rows || q >= b) return;
  double sx[V], sy[V];
#pragma unroll
  for (int v = 0; v < V; ++v) sx[v] = sy[v] = 0.0;
  const int k0 = P.rowptr[i], k1 = P.rowptr[i + 1];
#pragma unroll 4
  for (int k = k0; k < k1; ++k) {
    const int c = __ldg(&P.cols[k]);
    const double val = __ldg(&P.vals[k]);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double2 e = ld2(ec + static_cast<long long>(c) * b + q + 2 * v);
      sx[v] = sx[v] + val * e.x;
      sy[v] = sy[v] + val * e.y;
    }
  }
  const double w = __ldg(&wd[i]);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double2 ri = ld2(r + static_cast<long long>(i) * ldr + q + 2 * v);
    st2(x + static_cast<long long>(i) * b + q + 2 * v, make_double2(w * ri.x + 1.0 * sx[v], w * ri.y + 1.0 * sy[v]));
  }
}

template <int V>
__global__ void __launch_bounds__(256) k_mvc2_up2(DCsr A, const double* __restrict__ wd,
                                                  const double* __restrict__ r, int ldr,
                                                  const double* __restrict__ x, double* __restrict__ out,
                                                  int ldo, int b, int lsh) {
  griddep_wait();
  const MvcIdx<V> ix(lsh);
  const int i = ix.row, q = ix.q;
  if (i >= A.n_rows || q >= b) return;
  double sx[V], sy[V];
#pragma unroll
  for (int v = 0; v < V; ++v) sx[v] = sy[v] = 0.0;
  const int k0 = A.rowptr[i], k1 = A.rowptr[i + 1];
#pragma unroll 4
  for (int k = k0; k < k1; ++k) {
    const int c = __ldg(&A.cols[k]);
    const double a = __ldg(&A.vals[k]);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double2 xv = ld2(x + static_cast<long long>(c) * b + q + 2 * v);
      sx[v] = sx[v] + a * xv.x;
      sy[v] = sy[v] + a * xv.y;
    }
  }
  const double w = __ldg(&wd[i]);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double2 ri = ld2(r + static_cast<long long>(i) * ldr + q + 2 * v);
    const double2 xi = ld2(x + static_cast<long long>(i) * b + q + 2 * v);
    const double resx = ri.x + (-1.0 * sx[v]), resy = ri.y + (-1.0 * sy[v]);
    st2(out + static_cast<long long>(i) * ldo + q + 2 * v, make_double2(xi.x + w * resx, xi.y + w * resy));
  }
}

// Level-0 up2 of the Woodbury setup with the batch -> rows transpose fused into its store:
// out(i, q) goes straight to Ht[(r0 + q) * ldh + i] instead of an n x b buffer that a second
// kernel transposes (saves a write and a read of n x b doubles, 2.1 GB at C2).  The CTA's
// 8 rows x 128 columns are staged in shared memory, then each column's 8 consecutive rows
// leave as one 64-byte run (two 16-byte stores per thread).  V = 2, one row per warp.
__global__ void __launch_bounds__(256) k_mvc2_up2_rows(DCsr A, const double* __restrict__ wd,
                                                       const double* __restrict__ r, int ldr,
                                                       const double* __restrict__ x, double* __restrict__ ht,
                                                       long long ldh, int b) {
  griddep_wait();
  __shared__ __align__(16) double tile[8][129];
  const int ty = threadIdx.y, lane = threadIdx.x;
  const int i0 = blockIdx.x * 8, i = i0 + ty;
  const int qb = blockIdx.y * 128, q = qb + 4 * lane;
  const bool ok = i < A.n_rows && q < b;
  double sx[2] = {0.0, 0.0}, sy[2] = {0.0, 0.0};
  if (ok) {
    const int k0 = A.rowptr[i], k1 = A.rowptr[i + 1];
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
      const int c = __ldg(&A.cols[k]);
      const double a = __ldg(&A.vals[k]);
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const double2 xv = ld2(x + static_cast<long long>(c) * b + q + 2 * v);
        sx[v] = sx[v] + a * xv.x;
        sy[v] = sy[v] + a * xv.y;
      }
    }
    const double w = __ldg(&wd[i]);
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const double2 ri = ld2(r + static_cast<long long>(i) * ldr + q + 2 * v);
      const double2 xi = ld2(x + static_cast<long long>(i) * b + q + 2 * v);
      const double resx = ri.x + (-1.0 * sx[v]), resy = ri.y + (-1.0 * sy[v]);
      tile[ty][4 * lane + 2 * v] = xi.x + w * resx;
      tile[ty][4 * lane + 2 * v + 1] = xi.y + w * resy;
    }
  }
  __syncthreads();
  // 128 columns x 2 halves of 4 rows: thread t writes rows 4h..4h+3 of column t / 2
  const int t = ty * 32 + lane, cq = t >> 1, h = t & 1;
  const int qq = qb + cq;
  if (qq >= b) return;
  double* dst = ht + static_cast<long long>(qq) * ldh + i0 + 4 * h;
  const int rows = min(4, A.n_rows - (i0 + 4 * h));
  if (rows == 4) {
    st2(dst, make_double2(tile[4 * h][cq], tile[4 * h + 1][cq]));
    st2(dst + 2, make_double2(tile[4 * h + 2][cq], tile[4 * h + 3][cq]));
  } else {
    for (int rr = 0; rr < rows; ++rr) dst[rr] = tile[4 * h + rr][cq];
  }
}

// 4 columns per thread (V = 2) on large short-row matrices, 2 otherwise.  C2 (ncu, V = 1 -> 2):
// level 0 up1 724 -> 475 us, up2 757 -> 586, down 646 -> 580, restrict (10 per row) 305 -> 268,
// level-1 up1 (4.7 per row) 184 -> 142; the 13+ per row levels got slower with V = 2, and also
// with warp-cooperative index loads + shuffles (t_H 4.30 -> 4.43 ms), so they keep V = 1.
// Env GNW_MVC_V=1 disables V = 2.
static int mvc_v(const DCsr& M, int b) {
  static const int vmax = [] {
    const char* e = std::getenv("GNW_MVC_V");
    return e ? std::max(1, std::min(2, std::atoi(e))) : 2;
  }();
  const bool shape = M.n_rows >= 65536 && M.nnz <= 12LL * M.n_rows;
  // and only when the wider vectors fill the warps as well (b = 160: 40 threads per row
  // leave a second warp 3/4 idle, 80 fill 2.5 warps)
  auto fill = [b](int V) {
    const int need = (b + 2 * V - 1) / (2 * V), l = mvc_lanes(b, V);
    return static_cast<double>(need) / (((need + l - 1) / l) * l);
  };
  return (vmax >= 2 && b % 4 == 0 && shape && fill(2) >= fill(1)) ? 2 : 1;
}
static int lanes_log2(int b, int V) {
  int l = mvc_lanes(b, V), sh = 0;
  while ((1 << sh) < l) ++sh;
  return sh;
}
static dim3 grid2(int rows, int b, int V) {
  const int l = mvc_lanes(b, V), rows_per_cta = 8 * (32 / l);
  const int need = (b + 2 * V - 1) / (2 * V);
  return dim3((rows + rows_per_cta - 1) / rows_per_cta, (need + l - 1) / l);
}

#define GNW_MVC_LAUNCH(KERNEL, MAT, ROWS, ...)                                                         \
  do {                                                                                                 \
    if (mvc_v(MAT, b) == 2)                                                                            \
      GNW_LAUNCH(launch_k(KERNEL<2>, grid2(ROWS, b, 2), dim3(32, 8), 0, s, __VA_ARGS__, lanes_log2(b, 2))); \
    else                                                                                               \
      GNW_LAUNCH(launch_k(KERNEL<1>, grid2(ROWS, b, 1), dim3(32, 8), 0, s, __VA_ARGS__, lanes_log2(b, 1))); \
  } while (0)

void mvc2_down(const DLevel& L, const double* r, int ldr, double* resid, int b, cudaStream_t s) {
  GNW_MVC_LAUNCH(k_mvc2_down, L.A, L.n, L.A, L.wd, r, ldr, resid, b);
  note_launch("mvc2_down");
}
void mvc2_restrict(const DLevel& L, const double* resid, double* rc, int b, cudaStream_t s) {
  GNW_MVC_LAUNCH(k_mvc2_restrict, L.R, L.R.n_rows, L.R, resid, rc, b);
  note_launch("mvc2_restrict");
}
void mvc2_up1(const DLevel& L, const double* r, int ldr, const double* ec, double* x, int b, cudaStream_t s) {
  GNW_MVC_LAUNCH(k_mvc2_up1, L.P, L.n, L.P, L.wd, r, ldr, ec, x, b);
  note_launch("mvc2_up1");
}
bool mvc2_up2_rows(const DLevel& L, const double* r, int ldr, const double* x, double* ht, long long ldh, int b,
                   cudaStream_t s) {
  if (ldr % 2 != 0 || ldh % 2 != 0 || L.n % 8 != 0 || mvc_v(L.A, b) != 2 || mvc_lanes(b, 2) != 32) return false;
  const dim3 grid((L.n + 7) / 8, (b + 127) / 128);
  GNW_LAUNCH(launch_k(k_mvc2_up2_rows, grid, dim3(32, 8), 0, s, L.A, L.wd, r, ldr, x, ht, ldh, b));
  note_launch("mvc2_up2_rows");
  return true;
}

void mvc2_up2(const DLevel& L, const double* r, int ldr, const double* x, double* out, int ldo, int b,
              cudaStream_t s) {
  GNW_MVC_LAUNCH(k_mvc2_up2, L.A, L.n, L.A, L.wd, r, ldr, x, out, ldo, b);
  note_launch("mvc2_up2");
}

}  // namespace gnw
