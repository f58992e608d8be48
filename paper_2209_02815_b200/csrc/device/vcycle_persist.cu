// vcycle_persist.cu -- the small levels of the single-RHS V-cycle (amg.cpp:90-111) as ONE
// persistent cooperative launch.
//
// Below ~64k rows a level's four kernels (down, restrict, up1, up2) are pure latency: at C2
// levels 2-3 move < 1 MB each, yet every launch costs 6-8 us (ramp, one dependent
// rowptr -> cols -> x chain, drain; profiles/r01_launches_solve_sell.json), and the collapsed
// coarse apply another 14 us.  Here those phases run back to back inside one grid of
// co-resident CTAs separated by grid barriers (a generation barrier on two global words).
// Every phase computes exactly what the launched kernel computes, in the same order:
// G-lane groups per row (vcycle_wide.cu group_row; G = 1 is kernels.cu's thread-per-row
// CSR sum, whose terms and order the SELL kernels share) and the 4-accumulator warp-per-row
// dense apply (kernels.cu k_coarse_inverse1).  So the result is bit-identical to the
// kernel chain it replaces (tests/test_gpu_vcycle_persist.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {

constexpr int kPTpb = 256;

// generation barrier over all CTAs of the (co-resident) grid; bar[0] = arrivals, bar[1] = gen
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;  // read before arriving: the last arrival cannot have bumped it yet
    __threadfence();          // this CTA's phase writes before its arrival (release)
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();  // acquire: every CTA's phase writes are visible (reads below use ld.cg)
  }
  __syncthreads();
}

template <int G, class F>
__device__ __forceinline__ double prow(const DCsr& A, int i, int sub, bool valid, F f) {
  double acc = 0.0;
  if (valid) {
    const int k1 = A.rowptr[i + 1];
#pragma unroll 4
    for (int k = A.rowptr[i] + sub; k < k1; k += G) acc = acc + __ldg(&A.vals[k]) * f(__ldg(&A.cols[k]));
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// rows [0, n) of one phase, G lanes per row, over the grid's CTAs; body(i, s) on lane 0 of each row
template <int G, class F, class B>
__device__ __forceinline__ void phase_g(const DCsr& A, int n, F f, B body) {
  constexpr int per = kPTpb / G;
  const int nvb = (n + per - 1) / per;
  for (int vb = blockIdx.x; vb < nvb; vb += gridDim.x) {  // uniform per CTA: shuffles stay full-warp
    const int i = vb * per + static_cast<int>(threadIdx.x) / G, sub = static_cast<int>(threadIdx.x) % G;
    const bool ok = i < n;
    const double s = prow<G>(A, i, sub, ok, f);
    if (ok && sub == 0) body(i, s);
  }
}

template <class F, class B>
__device__ __forceinline__ void phase(const DCsr& A, int n, int G, F f, B body) {
  switch (G) {
    case 1: phase_g<1>(A, n, f, body); break;
    case 2: phase_g<2>(A, n, f, body); break;
    case 4: phase_g<4>(A, n, f, body); break;
    case 8: phase_g<8>(A, n, f, body); break;
    case 16: phase_g<16>(A, n, f, body); break;
    default: phase_g<32>(A, n, f, body); break;
  }
}

// x = M r, one warp per row, k_coarse_inverse1's four accumulators and xor tree
__device__ __forceinline__ void phase_dense(const double* __restrict__ M, int n, const double* r, double* x) {
  const int lane = threadIdx.x & 31;
  const int wpb = kPTpb / 32;
  const int nvb = (n + wpb - 1) / wpb;
  for (int vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
    const long long i = static_cast<long long>(vb) * wpb + (threadIdx.x >> 5);
    if (i >= n) continue;  // whole warp
    const double* __restrict__ row = M + i * n;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int j = lane;
    for (; j + 96 < n; j += 128) {
      const double m0 = __ldg(&row[j]), m1 = __ldg(&row[j + 32]), m2 = __ldg(&row[j + 64]), m3 = __ldg(&row[j + 96]);
      const double r0 = __ldcg(&r[j]), r1 = __ldcg(&r[j + 32]), r2 = __ldcg(&r[j + 64]), r3 = __ldcg(&r[j + 96]);
      a0 = a0 + m0 * r0;
      a1 = a1 + m1 * r1;
      a2 = a2 + m2 * r2;
      a3 = a3 + m3 * r3;
    }
    for (; j < n; j += 32) a0 = a0 + __ldg(&row[j]) * __ldcg(&r[j]);
    double acc[1] = {(a0 + a1) + (a2 + a3)};
    warp_reduce<1>(acc);
    if (lane == 0) x[i] = acc[0];
  }
}

__global__ void __launch_bounds__(kPTpb) k_vcycle_persist(PersistTail t, VSel rs, double* __restrict__ out,
                                                          const MinresState* st) {
  griddep_wait();
  const double* r0 = vsel(rs, st);
  // down the levels: res_l = r_l - A_l (wd_l .* r_l); r_{l+1} = R_l res_l
  for (int k = 0; k < t.nlev; ++k) {
    const PersistLevel L = t.lv[k];
    const double* r = k == 0 ? r0 : L.r;
    const double* __restrict__ wd = L.wd;
    double* res = L.res;
    phase(L.A, L.n, L.gA, [&](int c) { return __ldg(&wd[c]) * __ldcg(&r[c]); },
          [&](int i, double s) { res[i] = __ldcg(&r[i]) + (-1.0 * s); });
    grid_barrier(t.bar);
    double* rn = k + 1 < t.nlev ? t.lv[k + 1].r : t.rM;
    phase(L.R, L.R.n_rows, L.gR, [&](int c) { return __ldcg(&res[c]); }, [&](int i, double s) { rn[i] = s; });
    grid_barrier(t.bar);
  }
  // the dense level (collapsed tail or coarsest explicit inverse)
  phase_dense(t.M, t.nM, t.nlev == 0 ? r0 : t.rM, t.nlev == 0 ? out : t.eM);
  // up the levels: x_l = wd .* r_l + P_l e_{l+1}; e_l = x_l + wd .* (r_l - A_l x_l)
  for (int k = t.nlev - 1; k >= 0; --k) {
    grid_barrier(t.bar);
    const PersistLevel L = t.lv[k];
    const double* r = k == 0 ? r0 : L.r;
    const double* __restrict__ wd = L.wd;
    const double* ec = k + 1 < t.nlev ? t.lv[k + 1].e : t.eM;
    double* x = L.x;
    phase(L.P, L.n, L.gP, [&](int c) { return __ldcg(&ec[c]); },
          [&](int i, double s) { x[i] = __ldg(&wd[i]) * __ldcg(&r[i]) + 1.0 * s; });
    grid_barrier(t.bar);
    double* e = k == 0 ? out : L.e;
    phase(L.A, L.n, L.gA, [&](int c) { return __ldcg(&x[c]); }, [&](int i, double s) {
      const double res = __ldcg(&r[i]) + (-1.0 * s);
      e[i] = __ldcg(&x[i]) + __ldg(&wd[i]) * res;
    });
  }
}

}  // namespace

int persist_grid() {
  static int grid = [] {
    int dev = 0, sms = 148, occ = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_vcycle_persist, kPTpb, 0) != cudaSuccess || occ < 1)
      occ = 1;
    cudaGetLastError();
    return sms * std::min(occ, 4);
  }();
  return grid;
}

void vcycle_persist(const PersistTail& t, VSel r, double* out, const MinresState* st, cudaStream_t s) {
  // CTAs: enough for the widest phase, at most what is co-resident (cooperative launch)
  int need = (t.nM + kPTpb / 32 - 1) / (kPTpb / 32);
  for (int k = 0; k < t.nlev; ++k) {
    const PersistLevel& L = t.lv[k];
    need = std::max(need, (L.n + kPTpb / L.gA - 1) / (kPTpb / L.gA));
    need = std::max(need, (L.R.n_rows + kPTpb / L.gR - 1) / (kPTpb / L.gR));
    need = std::max(need, (L.n + kPTpb / L.gP - 1) / (kPTpb / L.gP));
  }
  const int grid = std::max(1, std::min(need, persist_grid()));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPTpb);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GNW_LAUNCH(cudaLaunchKernelEx(&cfg, k_vcycle_persist, t, r, out, st));
  note_launch("vcycle_persist");
}

}  // namespace gnw
