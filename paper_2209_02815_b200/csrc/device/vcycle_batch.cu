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

#include "kernels.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }
}  // namespace

__global__ void __launch_bounds__(256) k_mvc2_down(DCsr A, const double* __restrict__ wd,
                                                   const double* __restrict__ r, int ldr,
                                                   double* __restrict__ resid, int b) {
  griddep_wait();
  const int i = blockIdx.x * 8 + threadIdx.y;
  const int q = 2 * (blockIdx.y * 32 + threadIdx.x);
  if (i >= A.n_rows || q >= b) return;
  double sx = 0.0, sy = 0.0;
  const int k0 = A.rowptr[i], k1 = A.rowptr[i + 1];
#pragma unroll 4
  for (int k = k0; k < k1; ++k) {
    const int c = __ldg(&A.cols[k]);
    const double a = __ldg(&A.vals[k]), w = __ldg(&wd[c]);
    const double2 x = ld2(r + static_cast<long long>(c) * ldr + q);
    sx = sx + a * (w * x.x);
    sy = sy + a * (w * x.y);
  }
  const double2 ri = ld2(r + static_cast<long long>(i) * ldr + q);
  st2(resid + static_cast<long long>(i) * b + q, make_double2(ri.x + (-1.0 * sx), ri.y + (-1.0 * sy)));
}

__global__ void __launch_bounds__(256) k_mvc2_restrict(DCsr R, const double* __restrict__ resid,
                                                       double* __restrict__ rc, int b) {
  griddep_wait();
  const int a = blockIdx.x * 8 + threadIdx.y;
  const int q = 2 * (blockIdx.y * 32 + threadIdx.x);
  if (a >= R.n_rows || q >= b) return;
  double sx = 0.0, sy = 0.0;
  const int k0 = R.rowptr[a], k1 = R.rowptr[a + 1];
#pragma unroll 4
  for (int k = k0; k < k1; ++k) {
    const int c = __ldg(&R.cols[k]);
    const double v = __ldg(&R.vals[k]);
    const double2 x = ld2(resid + static_cast<long long>(c) * b + q);
    sx = sx + v * x.x;
    sy = sy + v * x.y;
  }
  st2(rc + static_cast<long long>(a) * b + q, make_double2(sx, sy));
}

__global__ void __launch_bounds__(256) k_mvc2_up1(DCsr P, const double* __restrict__ wd,
                                                  const double* __restrict__ r, int ldr,
                                                  const double* __restrict__ ec, double* __restrict__ x, int b) {
  griddep_wait();
  const int i = blockIdx.x * 8 + threadIdx.y;
  const int q = 2 * (blockIdx.y * 32 + threadIdx.x);
  if (i >= P.n_rows || q >= b) return;
  double sx = 0.0, sy = 0.0;
  const int k0 = P.rowptr[i], k1 = P.rowptr[i + 1];
#pragma unroll 4
  for (int k = k0; k < k1; ++k) {
    const int c = __ldg(&P.cols[k]);
    const double v = __ldg(&P.vals[k]);
    const double2 e = ld2(ec + static_cast<long long>(c) * b + q);
    sx = sx + v * e.x;
    sy = sy + v * e.y;
  }
  const double w = __ldg(&wd[i]);
  const double2 ri = ld2(r + static_cast<long long>(i) * ldr + q);
  st2(x + static_cast<long long>(i) * b + q, make_double2(w * ri.x + 1.0 * sx, w * ri.y + 1.0 * sy));
}

__global__ void __launch_bounds__(256) k_mvc2_up2(DCsr A, const double* __restrict__ wd,
                                                  const double* __restrict__ r, int ldr,
                                                  const double* __restrict__ x, double* __restrict__ out,
                                                  int ldo, int b) {
  griddep_wait();
  const int i = blockIdx.x * 8 + threadIdx.y;
  const int q = 2 * (blockIdx.y * 32 + threadIdx.x);
  if (i >= A.n_rows || q >= b) return;
  double sx = 0.0, sy = 0.0;
  const int k0 = A.rowptr[i], k1 = A.rowptr[i + 1];
#pragma unroll 4
  for (int k = k0; k < k1; ++k) {
    const int c = __ldg(&A.cols[k]);
    const double a = __ldg(&A.vals[k]);
    const double2 xv = ld2(x + static_cast<long long>(c) * b + q);
    sx = sx + a * xv.x;
    sy = sy + a * xv.y;
  }
  const double w = __ldg(&wd[i]);
  const double2 ri = ld2(r + static_cast<long long>(i) * ldr + q);
  const double2 xi = ld2(x + static_cast<long long>(i) * b + q);
  const double resx = ri.x + (-1.0 * sx), resy = ri.y + (-1.0 * sy);
  st2(out + static_cast<long long>(i) * ldo + q, make_double2(xi.x + w * resx, xi.y + w * resy));
}

static dim3 grid2(int rows, int b) { return dim3((rows + 7) / 8, (b / 2 + 31) / 32); }

void mvc2_down(const DLevel& L, const double* r, int ldr, double* resid, int b, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_mvc2_down, grid2(L.n, b), dim3(32, 8), 0, s, L.A, L.wd, r, ldr, resid, b));
  note_launch("mvc2_down");
}
void mvc2_restrict(const DLevel& L, const double* resid, double* rc, int b, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_mvc2_restrict, grid2(L.R.n_rows, b), dim3(32, 8), 0, s, L.R, resid, rc, b));
  note_launch("mvc2_restrict");
}
void mvc2_up1(const DLevel& L, const double* r, int ldr, const double* ec, double* x, int b, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_mvc2_up1, grid2(L.n, b), dim3(32, 8), 0, s, L.P, L.wd, r, ldr, ec, x, b));
  note_launch("mvc2_up1");
}
void mvc2_up2(const DLevel& L, const double* r, int ldr, const double* x, double* out, int ldo, int b,
              cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_mvc2_up2, grid2(L.n, b), dim3(32, 8), 0, s, L.A, L.wd, r, ldr, x, out, ldo, b));
  note_launch("mvc2_up2");
}

}  // namespace gnw
