// vcycle_fused.cu -- the default-mode V-cycle with ONE pass per level each way.
//
// amg.cpp:90-111 runs four sparse passes per level: pre-smooth + residual (A), restriction
// (P^T), prolongation (P), post-smooth (A).  Expanded (host::fused_cycle_ops), the level maps
//     r_c = T^T r   on the way down,   e = S r + T e_c   on the way up,
// with T = (I - Wd A) P and S = 2 Wd - Wd A Wd precomputed once per hierarchy.  Same linear
// operator, half the dependent launches (C2: 8 + the dense tail instead of 16 + tail) and, in
// the multi-RHS cycle of the Woodbury setup, fewer passes over the n x b work arrays (the
// level's x and residual are never stored).  The exact mode (GNW_COARSE_CHOLESKY) keeps the
// reference's level-by-level order in kernels.cu.
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"
#include "lell.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {

constexpr int kTpbF = 256;

// G lanes per row, lane j sums entries start + j, start + j + G, ..., then the xor butterfly
template <int G, class F>
__device__ __forceinline__ double grow(const DCsr& A, int i, int sub, bool valid, F f) {
  double acc = 0.0;
  if (valid) {
    const int k1 = A.rowptr[i + 1];
#pragma unroll 4
    for (int k = A.rowptr[i] + sub; k < k1; k += G) acc = acc + __ldg(&A.vals[k]) * f(__ldg(&A.cols[k]));
  }
  return acc;
}
template <int G>
__global__ void __launch_bounds__(kTpbF) k_vcf_restrict(DCsr Tt, VSel rs, const MinresState* st,
                                                        double* __restrict__ rc) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const int i = blockIdx.x * (kTpbF / G) + threadIdx.x / G, sub = threadIdx.x % G;
  const bool ok = i < Tt.n_rows;
  const double s = gsum<G>(grow<G>(Tt, i, sub, ok, [&](int c) { return r[c]; }));
  if (ok && sub == 0) rc[i] = s;
}

template <int G>
__global__ void __launch_bounds__(kTpbF) k_vcf_up(DCsr S, DCsr T, VSel rs, const double* __restrict__ ec,
                                                  double* __restrict__ out, const MinresState* st) {
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  const int i = blockIdx.x * (kTpbF / G) + threadIdx.x / G, sub = threadIdx.x % G;
  const bool ok = i < S.n_rows;
  // both rows' loads are issued before either butterfly
  const double a = grow<G>(S, i, sub, ok, [&](int c) { return r[c]; });
  const double b = grow<G>(T, i, sub, ok, [&](int c) { return ec[c]; });
  const double sa = gsum<G>(a), sb = gsum<G>(b);
  if (ok && sub == 0) out[i] = sa + sb;
}


// ---------------------------------------------- lane-ELL levels with coded values (DLell, lell.cuh)
template <int G>
__global__ void __launch_bounds__(kTpbF) k_vcl_restrict(DLell Tt, VSel rs, const MinresState* st,
                                                        double* __restrict__ rc) {
  const unsigned warp = blockIdx.x * (kTpbF / 32) + threadIdx.x / 32;
  const unsigned* __restrict__ p = Tt.words + warp * static_cast<unsigned>(Tt.width * 32) + (threadIdx.x & 31);
  LellBatch b0;
  b0.load(p, 0, Tt.width);  // the matrix does not depend on the predecessor kernel
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  double acc = b0.add(Tt, 0.0, [&](int c) { return r[c]; });
  for (int k = 4; k < Tt.width; k += 4) {
    LellBatch b;
    b.load(p, k, Tt.width);
    acc = b.add(Tt, acc, [&](int c) { return r[c]; });
  }
  const double s = gsum<G>(acc);
  const int i = blockIdx.x * (kTpbF / G) + threadIdx.x / G;
  if (i < Tt.n_rows && threadIdx.x % G == 0) rc[i] = s;
}

template <int G>
__global__ void __launch_bounds__(kTpbF) k_vcl_up(DLell S, DLell T, VSel rs, const double* __restrict__ ec,
                                                  double* __restrict__ out, const MinresState* st) {
  const unsigned warp = blockIdx.x * (kTpbF / 32) + threadIdx.x / 32;
  const unsigned* __restrict__ ps = S.words + warp * static_cast<unsigned>(S.width * 32) + (threadIdx.x & 31);
  const unsigned* __restrict__ pt = T.words + warp * static_cast<unsigned>(T.width * 32) + (threadIdx.x & 31);
  LellBatch s0, t0;
  s0.load(ps, 0, S.width);
  t0.load(pt, 0, T.width);
  griddep_wait();
  const double* __restrict__ r = vsel(rs, st);
  double a = s0.add(S, 0.0, [&](int c) { return r[c]; });
  double b = t0.add(T, 0.0, [&](int c) { return ec[c]; });
  const int W = S.width > T.width ? S.width : T.width;
  for (int k = 4; k < W; k += 4) {
    LellBatch sb, tb;
    sb.load(ps, k, S.width);
    tb.load(pt, k, T.width);
    a = sb.add(S, a, [&](int c) { return r[c]; });
    b = tb.add(T, b, [&](int c) { return ec[c]; });
  }
  const double sa = gsum<G>(a), sb2 = gsum<G>(b);
  const int i = blockIdx.x * (kTpbF / G) + threadIdx.x / G;
  if (i < S.n_rows && threadIdx.x % G == 0) out[i] = sa + sb2;
}

// ------------------------------------------------------------ multi-RHS (X[row * b + q])
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// one thread per (row, 2 consecutive columns); warp = 64 columns of one row (b even)
template <class Store>
__device__ __forceinline__ void mvcf_up_row(const DCsr& S, const DCsr& T, const double* __restrict__ r,
                                            const double* __restrict__ ec, int b, int i, int q, double& ox,
                                            double& oy) {
  double sx = 0.0, sy = 0.0, tx = 0.0, ty = 0.0;
  const int s0 = S.rowptr[i], s1 = S.rowptr[i + 1];
#pragma unroll 4
  for (int k = s0; k < s1; ++k) {
    const double2 x = ld2(r + static_cast<long long>(__ldg(&S.cols[k])) * b + q);
    const double v = __ldg(&S.vals[k]);
    sx = sx + v * x.x;
    sy = sy + v * x.y;
  }
  const int t0 = T.rowptr[i], t1 = T.rowptr[i + 1];
#pragma unroll 4
  for (int k = t0; k < t1; ++k) {
    const double2 x = ld2(ec + static_cast<long long>(__ldg(&T.cols[k])) * b + q);
    const double v = __ldg(&T.vals[k]);
    tx = tx + v * x.x;
    ty = ty + v * x.y;
  }
  ox = sx + tx;
  oy = sy + ty;
}
struct NoStore {};

__global__ void __launch_bounds__(256) k_mvcf_up2(DCsr S, DCsr T, const double* __restrict__ r,
                                                  const double* __restrict__ ec, double* __restrict__ out, int b) {
  griddep_wait();
  const int i = blockIdx.x * 8 + threadIdx.y, q = 2 * (blockIdx.y * 32 + threadIdx.x);
  if (i >= S.n_rows || q >= b) return;
  double ox, oy;
  mvcf_up_row<NoStore>(S, T, r, ec, b, i, q, ox, oy);
  *reinterpret_cast<double2*>(out + static_cast<long long>(i) * b + q) = make_double2(ox, oy);
}

// odd b: one column per thread
__global__ void __launch_bounds__(256) k_mvcf_up1(DCsr S, DCsr T, const double* __restrict__ r,
                                                  const double* __restrict__ ec, double* __restrict__ out, int b) {
  griddep_wait();
  const int i = blockIdx.x * 8 + threadIdx.y, q = blockIdx.y * 32 + threadIdx.x;
  if (i >= S.n_rows || q >= b) return;
  double s = 0.0, t = 0.0;
  for (int k = S.rowptr[i]; k < S.rowptr[i + 1]; ++k) s = s + __ldg(&S.vals[k]) * r[static_cast<long long>(S.cols[k]) * b + q];
  for (int k = T.rowptr[i]; k < T.rowptr[i + 1]; ++k) t = t + __ldg(&T.vals[k]) * ec[static_cast<long long>(T.cols[k]) * b + q];
  out[static_cast<long long>(i) * b + q] = s + t;
}

// level 0 of the Woodbury setup: the result goes straight to Ht rows (ht[q * ldh + i]); the CTA's
// 8 rows x 64 columns are staged in shared memory and leave as 64-byte row runs
__global__ void __launch_bounds__(256) k_mvcf_up_rows(DCsr S, DCsr T, const double* __restrict__ r,
                                                      const double* __restrict__ ec, double* __restrict__ ht,
                                                      long long ldh, int b) {
  griddep_wait();
  __shared__ double tile[8][65];
  const int ty = threadIdx.y, lane = threadIdx.x;
  const int i0 = blockIdx.x * 8, i = i0 + ty;
  const int qb = blockIdx.y * 64, q = qb + 2 * lane;
  if (i < S.n_rows && q < b) {
    double ox, oy;
    mvcf_up_row<NoStore>(S, T, r, ec, b, i, q, ox, oy);
    tile[ty][2 * lane] = ox;
    tile[ty][2 * lane + 1] = oy;
  }
  __syncthreads();
  // 64 columns x 4 pairs of rows: thread t writes rows 2h, 2h+1 of column t / 4
  const int t = ty * 32 + lane, cq = t >> 2, h = t & 3;
  const int qq = qb + cq, rr = i0 + 2 * h;
  if (qq >= b || rr >= S.n_rows) return;
  double* dst = ht + static_cast<long long>(qq) * ldh + rr;
  if (rr + 1 < S.n_rows)
    *reinterpret_cast<double2*>(dst) = make_double2(tile[2 * h][cq], tile[2 * h + 1][cq]);
  else
    dst[0] = tile[2 * h][cq];
}

}  // namespace

#define GNW_F_DISPATCH(G, KERNEL, ROWS, ...)                                                                        \
  switch (G) {                                                                                                      \
    case 1: GNW_LAUNCH(launch_k(KERNEL<1>, (ROWS + kTpbF - 1) / kTpbF, kTpbF, 0, __VA_ARGS__)); break;              \
    case 2: GNW_LAUNCH(launch_k(KERNEL<2>, (ROWS + kTpbF / 2 - 1) / (kTpbF / 2), kTpbF, 0, __VA_ARGS__)); break;    \
    case 4: GNW_LAUNCH(launch_k(KERNEL<4>, (ROWS + kTpbF / 4 - 1) / (kTpbF / 4), kTpbF, 0, __VA_ARGS__)); break;    \
    case 8: GNW_LAUNCH(launch_k(KERNEL<8>, (ROWS + kTpbF / 8 - 1) / (kTpbF / 8), kTpbF, 0, __VA_ARGS__)); break;    \
    case 16: GNW_LAUNCH(launch_k(KERNEL<16>, (ROWS + kTpbF / 16 - 1) / (kTpbF / 16), kTpbF, 0, __VA_ARGS__)); break; \
    default: GNW_LAUNCH(launch_k(KERNEL<32>, (ROWS + kTpbF / 32 - 1) / (kTpbF / 32), kTpbF, 0, __VA_ARGS__)); break; \
  }


template <int G>
void launch_lrestrict(const DLevel& L, VSel r, double* rc, const MinresState* st, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_vcl_restrict<G>, (L.Ttl.n_rows + kTpbF / G - 1) / (kTpbF / G), kTpbF, 0, s, L.Ttl, r, st, rc));
}
template <int G>
void launch_lup(const DLevel& L, VSel r, const double* ec, double* out, const MinresState* st, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_vcl_up<G>, (L.n + kTpbF / G - 1) / (kTpbF / G), kTpbF, 0, s, L.Sl, L.Tl, r, ec, out, st));
}
#define GNW_L_DISPATCH(G, FN, ...) \
  switch (G) {                     \
    case 1: FN<1>(__VA_ARGS__); break;   \
    case 2: FN<2>(__VA_ARGS__); break;   \
    case 4: FN<4>(__VA_ARGS__); break;   \
    case 8: FN<8>(__VA_ARGS__); break;   \
    case 16: FN<16>(__VA_ARGS__); break; \
    default: FN<32>(__VA_ARGS__); break; \
  }

void vcf_restrict(const DLevel& L, VSel r, double* rc, const MinresState* st, cudaStream_t s) {
  if (L.Ttl.words != nullptr) {
    GNW_L_DISPATCH(L.gTt, launch_lrestrict, L, r, rc, st, s);
    return note_launch("vcl_restrict");
  }
  GNW_F_DISPATCH(L.gTt, k_vcf_restrict, L.Tt.n_rows, s, L.Tt, r, st, rc);
  note_launch("vcf_restrict");
}
void vcf_up(const DLevel& L, VSel r, const double* ec, double* out, const MinresState* st, cudaStream_t s) {
  if (L.Sl.words != nullptr && L.Tl.words != nullptr) {
    GNW_L_DISPATCH(L.gS, launch_lup, L, r, ec, out, st, s);
    return note_launch("vcl_up");
  }
  GNW_F_DISPATCH(L.gS, k_vcf_up, L.n, s, L.S, L.T, r, ec, out, st);
  note_launch("vcf_up");
}

void mvcf_restrict(const DLevel& L, const double* r, double* rc, int b, cudaStream_t s) {
  DLevel R = L;  // the batched restriction kernels on T^T
  R.R = L.Tt;
  R.Rs = DSell{};
  mvc_restrict(R, r, rc, b, s);
}
bool mvcf_up(const DLevel& L, const double* r, const double* ec, double* out, int b, double* ht, long long ldh,
             cudaStream_t s) {
  if (ht != nullptr && b % 2 == 0 && ldh % 2 == 0) {
    const dim3 grid((L.n + 7) / 8, (b + 63) / 64);
    GNW_LAUNCH(launch_k(k_mvcf_up_rows, grid, dim3(32, 8), 0, s, L.S, L.T, r, ec, ht, ldh, b));
    note_launch("mvcf_up_rows");
    return true;
  }
  if (b % 2 == 0) {
    GNW_LAUNCH(launch_k(k_mvcf_up2, dim3((L.n + 7) / 8, (b / 2 + 31) / 32), dim3(32, 8), 0, s, L.S, L.T, r, ec, out, b));
  } else {
    GNW_LAUNCH(launch_k(k_mvcf_up1, dim3((L.n + 7) / 8, (b + 31) / 32), dim3(32, 8), 0, s, L.S, L.T, r, ec, out, b));
  }
  note_launch("mvcf_up");
  return false;
}

}  // namespace gnw
