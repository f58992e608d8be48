// vcycle_tail.cu -- the coarse tail of the single-RHS V-cycle in ONE launch.
//
// Below a few hundred thousand nonzeros per level the V-cycle is launch- and
// latency-bound: each of the 4 kernels per level (and the coarsest solve) moves a
// few MB at most, yet pays a launch gap plus a cold dependent-load chain.  This
// kernel runs levels l0 .. L-1 of amg.cpp:90-111 on one thread-block CLUSTER
// (8 CTAs x 8 warps): the phases (down, restrict, ..., coarse solve, ..., up1,
// up2) are separated by cluster barriers (barrier.cluster arrive.release /
// wait.acquire) instead of kernel boundaries, and vectors produced inside the
// launch are read with ld.global.cg so no stale L1 line can be observed.
//
// Each phase uses exactly the per-row arithmetic of the unfused kernels
// (thread-per-row reference order on narrow levels and in exact mode, the
// lane-strided warp order on wide levels, the same coarse solves), so fusing
// changes no bit of the result.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {

constexpr int kTailThreads = 256;

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
  return r;
}

__device__ __forceinline__ double ldv(const double* p) { return __ldcg(p); }

// sum_k A[i,k] f(col_k): sequential (reference order) or lane-strided warp tree
template <class F>
__device__ __forceinline__ double row_seq(const DCsr& A, int i, F f) {
  double s = 0.0;
  const int k1 = A.rowptr[i + 1];
  for (int k = A.rowptr[i]; k < k1; ++k) s = s + __ldg(&A.vals[k]) * f(A.cols[k]);
  return s;
}
template <class F>
__device__ __forceinline__ double row_warp(const DCsr& A, int i, int lane, F f) {
  double acc = 0.0;
  const int k1 = A.rowptr[i + 1];
  for (int k = A.rowptr[i] + lane; k < k1; k += 32) acc = acc + __ldg(&A.vals[k]) * f(A.cols[k]);
  double v[1] = {acc};
  warp_reduce<1>(v);
  return v[0];
}

// Apply `body(i, s)` to every row i of A with s = sum_k A[i,k] f(col_k), rows spread
// over the cluster: warps for wide matrices, threads otherwise.
template <class F, class B>
__device__ __forceinline__ void for_rows(const DCsr& A, int n, int wide, F f, B body) {
  const unsigned cr = cluster_rank(), cs = cluster_size();
  if (wide) {
    const int lane = threadIdx.x & 31;
    const int gw = static_cast<int>(cr * (kTailThreads / 32) + (threadIdx.x >> 5));
    const int nw = static_cast<int>(cs * (kTailThreads / 32));
    for (int i = gw; i < n; i += nw) {
      const double s = row_warp(A, i, lane, f);
      if (lane == 0) body(i, s);
    }
  } else {
    const int gt = static_cast<int>(cr * kTailThreads + threadIdx.x);
    const int nt = static_cast<int>(cs * kTailThreads);
    for (int i = gt; i < n; i += nt) body(i, row_seq(A, i, f));
  }
}

}  // namespace

__global__ void __launch_bounds__(kTailThreads) k_vcycle_tail(TailArgs a, VSel rin, double* out,
                                                               const MinresState* st) {
  const double* r0 = vsel(rin, st);
  auto rvec = [&](int l) -> const double* { return l == 0 ? r0 : a.r[l]; };
  // ---------------------------------------------------------------- down
  for (int l = 0; l < a.nlev; ++l) {
    const TailLevel& L = a.lv[l];
    const double* r = rvec(l);
    double* res = a.res[l];
    for_rows(L.A, L.n, L.wideA, [&](int c) { return __ldg(&L.wd[c]) * ldv(&r[c]); },
             [&](int i, double s) { res[i] = ldv(&r[i]) + (-1.0 * s); });
    cluster_sync_all();
    double* rc = a.r[l + 1];
    for_rows(L.R, L.R.n_rows, L.wideR, [&](int c) { return ldv(&res[c]); }, [&](int i, double s) { rc[i] = s; });
    cluster_sync_all();
  }
  // ------------------------------------------------------------- coarsest
  {
    const double* rc = rvec(a.nlev);
    double* ec = a.nlev == 0 ? out : a.e[a.nlev];
    const unsigned cr = cluster_rank(), cs = cluster_size();
    if (a.exact) {  // cholesky_solve replayed (linalg.cpp:107-123), one thread
      if (cr == 0 && threadIdx.x == 0) {
        const int n = a.nc;
        for (int i = 0; i < n; ++i) ec[i] = ldv(&rc[i]);
        for (int i = 0; i < n; ++i) {
          double s = ec[i];
          for (int k = 0; k < i; ++k) s = s - a.Lc[static_cast<long long>(i) * n + k] * ec[k];
          ec[i] = s / a.Lc[static_cast<long long>(i) * n + i];
        }
        for (int ii = n - 1; ii >= 0; --ii) {
          double s = ec[ii];
          for (int k = ii + 1; k < n; ++k) s = s - a.Lc[static_cast<long long>(k) * n + ii] * ec[k];
          ec[ii] = s / a.Lc[static_cast<long long>(ii) * n + ii];
        }
      }
    } else {  // explicit inverse, warp per row (k_coarse_inverse order)
      const int lane = threadIdx.x & 31;
      const int gw = static_cast<int>(cr * (kTailThreads / 32) + (threadIdx.x >> 5));
      const int nw = static_cast<int>(cs * (kTailThreads / 32));
      for (int i = gw; i < a.nc; i += nw) {
        double acc[1] = {0.0};
        for (int j = lane; j < a.nc; j += 32)
          acc[0] = acc[0] + __ldg(&a.Ainv[static_cast<long long>(i) * a.nc + j]) * ldv(&rc[j]);
        warp_reduce<1>(acc);
        if (lane == 0) ec[i] = acc[0];
      }
    }
    cluster_sync_all();
  }
  // ------------------------------------------------------------------ up
  for (int l = a.nlev - 1; l >= 0; --l) {
    const TailLevel& L = a.lv[l];
    const double* r = rvec(l);
    const double* ec = a.e[l + 1];
    double* x = a.x[l];
    for_rows(L.P, L.n, L.wideP, [&](int c) { return ldv(&ec[c]); },
             [&](int i, double s) { x[i] = __ldg(&L.wd[i]) * ldv(&r[i]) + 1.0 * s; });
    cluster_sync_all();
    double* e = l == 0 ? out : a.e[l];
    for_rows(L.A, L.n, L.wideA, [&](int c) { return ldv(&x[c]); }, [&](int i, double s) {
      const double res = ldv(&r[i]) + (-1.0 * s);
      e[i] = ldv(&x[i]) + __ldg(&L.wd[i]) * res;
    });
    cluster_sync_all();
  }
}

void vcycle_tail(const TailArgs& a, VSel rin, double* out, const MinresState* st, int cluster, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster, 1, 1);
  cfg.blockDim = dim3(kTailThreads, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static bool nonportable = false;
  if (cluster > 8 && !nonportable) {
    cudaFuncSetAttribute(k_vcycle_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    nonportable = true;
  }
  cudaLaunchKernelEx(&cfg, k_vcycle_tail, a, rin, out, st);
  note_launch("vcycle_tail");
}

}  // namespace gnw
