// lell.cuh -- device helpers of the lane-ELL level kernels (common.cuh DLell), shared by the
// per-level kernels (vcycle_fused.cu) and the persistent MINRES kernel (minres_persistent.cu).
#pragma once

#include "common.cuh"

namespace gnw {

template <int G>
__device__ __forceinline__ double gsum(double acc) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// One batch of four lane entries: the four words are loaded together, then the table look-ups
// and gathers are issued together, then the products are added in entry order (padding, which
// has the sign bit set, is skipped).
struct LellBatch {
  unsigned w[4];
  __device__ __forceinline__ void load(const unsigned* __restrict__ p, int k, int width) {
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = k + u < width ? __ldg(p + 32 * (k + u)) : 0xffffffffu;
  }
  template <class F>
  __device__ __forceinline__ double add(const DLell& A, double acc, F f) const {
    double v[4], x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = static_cast<int>(w[u]) >= 0;
      v[u] = ok ? __ldg(A.table + (w[u] >> A.shift)) : 0.0;
      x[u] = ok ? f(static_cast<int>(w[u] & A.mask)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (static_cast<int>(w[u]) >= 0) acc = acc + v[u] * x[u];
    return acc;
  }
};

}  // namespace gnw
