// dgemm_tma.cu -- the capacitance GEMM C = I + (J Ht^T) / beta (inversion.cpp:37-43 ->
// linalg.cpp:56-70) with TMA operand staging.
//
// FP64 has no tcgen05 path on sm_100a, so the math stays on the DMMA pipe
// (mma.sync.m8n8k4.f64); what Blackwell adds is the data movement.  One producer warp issues
// cp.async.bulk.tensor 2D loads (128 rows x 16 doubles of J and of Ht per stage, SWIZZLE_128B)
// into a 6-stage shared-memory ring guarded by full/empty mbarriers; eight consumer warps
// (2 x 4, 64 x 32 each) wait on the full barrier of a stage, read their DMMA fragments through
// the swizzle (conflict-free: a warp's 8 rows x 4 doubles land in 8 distinct 16-byte columns,
// two wavefronts for 256 bytes) and release the stage per warp -- no __syncthreads in the main
// loop, no per-thread address arithmetic for the loads, out-of-range rows and the K tail
// zero-filled by the TMA unit.  Same tile plan, split-K and accumulation order as the cp.async
// kernel in kernels.cu (k_dgemm_nt, kept as the fallback), so C is bit-identical to it.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "kernels.cuh"

namespace gnw {

void note_launch(const char* what);

namespace dgt {
constexpr int BM = 128, BN = 128, BK = 16, STAGES = 6;
constexpr int TILE_BYTES = BM * BK * 8;                 // 16 KB per operand per stage
constexpr int STAGE_BYTES = 2 * TILE_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;  // ring + alignment slack + barriers
constexpr int CONSUMER_WARPS = 8;
constexpr int THREADS = (CONSUMER_WARPS + 1) * 32;
}  // namespace dgt

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// element (row, k) of a 128 x 16 tile stored by TMA with SWIZZLE_128B: the 16-byte chunk index
// is xor-ed with row % 8
__device__ __forceinline__ const double* swz(const unsigned char* tile, int row, int k) {
  return reinterpret_cast<const double*>(tile + row * 128 + ((((k >> 1) ^ (row & 7)) << 4) | ((k & 1) << 3)));
}

__global__ void __launch_bounds__(dgt::THREADS, 1)
k_dgemm_tma(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, long long N,
            long long kchunk, const int2* __restrict__ pairs, int npairs, double* __restrict__ part) {
  using namespace dgt;
  extern __shared__ unsigned char smraw[];
  unsigned char* ring = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t{1023});
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ring + STAGES * STAGE_BYTES);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(bars + s), 1);                        // full: the producer's expect_tx arrival
      mbar_init(smem_u32(bars + STAGES + s), CONSUMER_WARPS);  // empty: one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  griddep_wait();  // J and Ht are written by the preceding kernels
  const int2 pr = pairs[blockIdx.x];
  const int i0 = pr.x * BM, j0 = pr.y * BN;
  const long long k0 = static_cast<long long>(blockIdx.y) * kchunk;
  const long long k1 = min(N, k0 + kchunk);
  const int nkt = static_cast<int>((k1 - k0 + BK - 1) / BK);

  if (warp == CONSUMER_WARPS) {  // producer warp: one lane drives the TMA unit
    if (lane == 0) {
      for (int kt = 0; kt < nkt; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(smem_u32(bars + STAGES + s), ((kt / STAGES) - 1) & 1);
        const unsigned full = smem_u32(bars + s);
        mbar_expect_tx(full, STAGE_BYTES);
        const int kc = static_cast<int>(k0 + static_cast<long long>(kt) * BK);
        tma_load_2d(smem_u32(ring + s * STAGE_BYTES), &mapA, kc, i0, full);
        tma_load_2d(smem_u32(ring + s * STAGE_BYTES + TILE_BYTES), &mapB, kc, j0, full);
      }
    }
    return;
  }

  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 consumer warps
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;
  for (int kt = 0; kt < nkt; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(smem_u32(bars + s), (kt / STAGES) & 1);
    const unsigned char* as = ring + s * STAGE_BYTES;
    const unsigned char* bs = as + TILE_BYTES;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) af[a] = *swz(as, wm * 64 + a * 8 + fr, kk + fk);
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = *swz(bs, wn * 32 + b * 8 + fr, kk + fk);
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(bars + STAGES + s));  // this warp is done with the stage
  }
  // partial tile out: part[(split * npairs + pair)][BM][BN]
  double* out = part + (static_cast<long long>(blockIdx.y) * npairs + blockIdx.x) * (BM * BN);
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = wm * 64 + a * 8 + fr;
      const int c = wn * 32 + b * 8 + fk * 2;
      *reinterpret_cast<double2*>(out + r * BN + c) = make_double2(acc[a][b][0], acc[a][b][1]);
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// rows x cols row-major FP64 matrix with row stride ld, boxes of 128 rows x 16 columns
bool make_map(CUtensorMap* map, const double* A, long long rows, long long cols, long long ld) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  const cuuint32_t box[2] = {dgt::BK, dgt::BM};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// false: not launched (no driver entry point, unaligned operands, or GNW_DGEMM_TMA=0) -- the
// caller falls back to the cp.async kernel
bool capacitance_dgemm_tma(const double* J, long long ldj, const double* Ht, long long ldh, int m, long long N,
                           const DgemmPlan& plan, const int2* dpairs, double* part, cudaStream_t s) {
  static const bool off = [] {
    const char* e = std::getenv("GNW_DGEMM_TMA");
    return e != nullptr && std::atoi(e) == 0;
  }();
  if (off) return false;
  if ((reinterpret_cast<uintptr_t>(J) & 15) || (reinterpret_cast<uintptr_t>(Ht) & 15) || (ldj & 1) || (ldh & 1) ||
      N > 0x7fffffffLL)
    return false;
  CUtensorMap mapA, mapB;
  if (!make_map(&mapA, J, m, N, ldj) || !make_map(&mapB, Ht, m, N, ldh)) return false;
  smem_optin(reinterpret_cast<const void*>(k_dgemm_tma), dgt::SMEM);
  const dim3 grid(plan.npairs, plan.splits);
  GNW_LAUNCH(launch_k(k_dgemm_tma, grid, dgt::THREADS, dgt::SMEM, s, mapA, mapB, N, plan.kchunk, dpairs, plan.npairs, part));
  note_launch("dgemm_tma");
  return true;
}

}  // namespace gnw
