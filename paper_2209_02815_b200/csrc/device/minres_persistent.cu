// minres_persistent.cu -- the MINRES loop (minres.cpp:70-148) as ONE persistent cooperative
// kernel, for problems whose whole working set is L2-resident (BASELINE C1: 64^2 mesh, m = 32).
//
// At that size every kernel of the graph loop is latency-bound: an iteration is ~20 dependent
// launches of ~2 us each (C1: 0.044 ms for 14.5 MB).  Here a few dozen CTAs (one per ~192 edge
// rows; C1: 65) stay resident for the whole solve and the phases of an iteration are separated
// by grid barriers (one global arrival counter, release/acquire) instead of kernel boundaries:
// eight barriers per iteration at C1 (two one-pass levels above a 519-row dense tail).
// The arithmetic is the lean schedule's (q = J^T t' feeds the next operator,
// z2 = B (v2 - q / beta), one refinement step on t' = C^-1 t):
//
//   [saddle]   y = A zhat (first iteration; afterwards fused with the previous update phase)
//   B          delta; v_next = y + c1 v_cur + c2 v_prev; z1 = q_diag_inv v1; partial t = H^T v2
//   C          t (fixed-order sum of the CTA partials), t' = C^-1 t refined; q = J^T t';
//              y' = v2 - q / beta                                   (every CTA solves the m x m part)
//   D          V-cycle of y': one-pass lane-ELL levels (lell.cuh), dense collapsed tail; the last
//              level's rows also store z2 and accumulate <z, v>, <z, z>
//   F + A      Givens rotation (minres_scalars.cuh, every CTA on its own copy of the state);
//              w, u, x, r recurrences and ||r||^2; the NEXT iteration's operator y = A zhat_next
//   tail       ||r|| / ||b||, history, convergence / exhaustion / maxit (update_tail)
//
// Every CTA reduces the same partials in the same order, so all CTAs hold the same scalars and
// take the same control-flow decisions; CTA 0 writes the state and the histories back.  The
// kernel returns when the recurred residual meets the tolerance (the host then verifies the true
// residual exactly as for the graph loop, minres.cpp:108-120), on exhaustion, maxit or an error.
// Reductions are summed in a different order than the graph loop's kernels, so results agree with
// it to rounding (same bars as the other schedules: iterations +-1, solution <= 1e-8).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "lell.cuh"
#include "minres_persistent.cuh"
#include "minres_scalars.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {

constexpr int kPT = 256;          // threads per CTA (each owns at most one edge row and one cell row)
constexpr int kPW = kPT / 32;     // warps per CTA
constexpr int kMaxM = 64;         // rows of J handled with C, C^-1 in shared memory
constexpr int kSlots = 8;         // partial-sum slots per CTA

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// grid barrier: a monotone arrival counter (zeroed by the host before the launch), polled by
// one thread per CTA.  (Measured against a last-arriver-publishes-a-flag variant: the flag adds
// a third L2 round trip per barrier, C1 iteration 0.034 -> 0.038 ms.)
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
    const unsigned target = epoch * gridDim.x;
    while (ld_acquire(bar) < target) {
    }
  }
  __syncthreads();
}

// sum over the CTAs' partials of slot k (written as part[cta * kSlots + k]) in a fixed order:
// lane l adds CTAs l, l + 32, ... then the xor tree -- the same bits on every CTA
__device__ __forceinline__ double total_of(const double* part, int k) {
  double a = 0.0;
  for (int c = threadIdx.x & 31; c < static_cast<int>(gridDim.x); c += 32) a += __ldcg(&part[c * kSlots + k]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

// the same for NS consecutive slots k0 .. k0 + NS - 1 in one pass (one L2 round trip)
template <int NS>
__device__ __forceinline__ void totals_of(const double* part, int k0, double (&out)[NS]) {
#pragma unroll
  for (int k = 0; k < NS; ++k) out[k] = 0.0;
  for (int c = threadIdx.x & 31; c < static_cast<int>(gridDim.x); c += 32)
#pragma unroll
    for (int k = 0; k < NS; ++k) out[k] += __ldcg(&part[c * kSlots + k0 + k]);
#pragma unroll
  for (int k = 0; k < NS; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) out[k] += __shfl_xor_sync(0xffffffffu, out[k], o);
}

// block sum of NV values; result in every thread (red: NV * kPW doubles)
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red) {
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) red[warp * NV + k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
    for (int w = 0; w < kPW; ++w) s += red[w * NV + k];
    v[k] = s;
  }
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}

__device__ __forceinline__ double* ring_slot(double* const (&p)[3], int mod, long long j, int off) {
  return p[static_cast<int>((j + off) % mod)];
}

// lane-ELL level pass over the virtual warps of this CTA: out[i] = sum_k A(i, k) f(col_k)
// (+ the second operator), G lanes per row -- the sums of k_vcl_restrict / k_vcl_up
template <int G, class F, class Store>
__device__ __forceinline__ void lell_rows(const DLell& A, F f, Store store) {
  const int rpw = 32 / G, lane = threadIdx.x & 31;
  const int nslices = (A.n_rows + rpw - 1) / rpw;
  for (int vw = blockIdx.x * kPW + (threadIdx.x >> 5); vw < nslices; vw += gridDim.x * kPW) {
    const unsigned* __restrict__ p = A.words + static_cast<unsigned>(vw) * static_cast<unsigned>(A.width * 32) + lane;
    double acc = 0.0;
    for (int k = 0; k < A.width; k += 4) {
      LellBatch b;
      b.load(p, k, A.width);
      acc = b.add(A, acc, f);
    }
    const double s = gsum<G>(acc);
    const int i = vw * rpw + lane / G;
    if (i < A.n_rows && lane % G == 0) store(i, s);
  }
}
template <int G, class F1, class F2, class Store>
__device__ __forceinline__ void lell_rows2(const DLell& S, const DLell& T, F1 f1, F2 f2, Store store) {
  const int rpw = 32 / G, lane = threadIdx.x & 31;
  const int nslices = (S.n_rows + rpw - 1) / rpw;
  for (int vw = blockIdx.x * kPW + (threadIdx.x >> 5); vw < nslices; vw += gridDim.x * kPW) {
    const unsigned* __restrict__ ps = S.words + static_cast<unsigned>(vw) * static_cast<unsigned>(S.width * 32) + lane;
    const unsigned* __restrict__ pt = T.words + static_cast<unsigned>(vw) * static_cast<unsigned>(T.width * 32) + lane;
    double a = 0.0, b = 0.0;
    const int W = S.width > T.width ? S.width : T.width;
    for (int k = 0; k < W; k += 4) {
      LellBatch sb, tb;
      sb.load(ps, k, S.width);
      tb.load(pt, k, T.width);
      a = sb.add(S, a, f1);
      b = tb.add(T, b, f2);
    }
    const double sa = gsum<G>(a), sb2 = gsum<G>(b);
    const int i = vw * rpw + lane / G;
    if (i < S.n_rows && lane % G == 0) store(i, sa + sb2);
  }
}

#define GNW_P_LANES(G, CALL)        \
  switch (G) {                      \
    case 1: { constexpr int GG = 1; CALL; } break;   \
    case 2: { constexpr int GG = 2; CALL; } break;   \
    case 4: { constexpr int GG = 4; CALL; } break;   \
    case 8: { constexpr int GG = 8; CALL; } break;   \
    case 16: { constexpr int GG = 16; CALL; } break; \
    default: { constexpr int GG = 32; CALL; } break; \
  }

// one row of a SELL-32 matrix (at most W entries) decoded into registers: the operator rows a
// thread owns stay there for the whole solve
template <int W>
struct RowCache {
  int c[W];
  double v[W];
  __device__ __forceinline__ void load(const DSell& A, long long row, bool ok) {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      c[k] = -1;
      v[k] = 0.0;
    }
    if (!ok) return;
    const long long base = (row >> 5) * 32LL * A.width + (row & 31);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      if (k >= A.width) break;
      const int q = __ldg(A.cols + base + 32 * k);
      if (A.signed_cols) {
        c[k] = q >= -1 ? q : -q - 2;
        v[k] = q >= -1 ? 1.0 : -1.0;
      } else {
        c[k] = q;
        v[k] = A.codes ? __ldg(A.table + __ldg(A.codes + base + 32 * k)) : __ldg(A.vals + base + 32 * k);
      }
    }
  }
  // the gathers of one application, issued together
  __device__ __forceinline__ void gather(const double* __restrict__ x, long long off, double (&g)[W]) const {
#pragma unroll
    for (int k = 0; k < W; ++k) g[k] = c[k] >= 0 ? x[off + c[k]] : 0.0;
  }
  // sum_k v_k (g_k * sc) in entry order (sell_finish, scaled)
  __device__ __forceinline__ double dot(const double (&g)[W], double sc) const {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (c[k] >= 0) s = s + v[k] * (g[k] * sc);
    return s;
  }
};

__global__ void __launch_bounds__(kPT, 1) k_minres_persistent(PersistArgs a) {
  extern __shared__ double dyn[];  // C^-1, C (stride m + 1), then the CTA's slices of J and Ht
  __shared__ MinresState ls;
  __shared__ double red[5 * kPW];
  __shared__ double tsm[kMaxM], t2sm[kMaxM], rsm[kMaxM];
  __shared__ double v2sm[kPT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = gridDim.x, cta = blockIdx.x;
  const int m = a.m;
  const long long K = a.K, N = a.N;
  // contiguous ownership: thread t of CTA c owns edge e_lo + t and cell c_lo + t (at most one each)
  const long long e_lo = K * cta / nb, e_hi = K * (cta + 1) / nb;
  const long long c_lo = N * cta / nb, c_hi = N * (cta + 1) / nb;
  const int nc = static_cast<int>(c_hi - c_lo);
  const long long e0 = e_lo + tid, c0 = c_lo + tid;
  const bool has_e = e0 < e_hi, has_c = c0 < c_hi;
  const int mp = m + 1;           // row stride m + 1: thread i reads row i without bank conflicts
  double* csm = dyn;              // C^-1
  double* cfm = csm + m * mp;     // C
  double* jsm = cfm + m * mp;     // J(i, c_lo + t)  at [i * nc + t]
  double* hsm = jsm + m * nc;     // Ht(i, c_lo + t) at [i * nc + t]
  for (int k = tid; k < m * m; k += kPT) {
    csm[(k / m) * mp + k % m] = a.Cinv[k];
    cfm[(k / m) * mp + k % m] = a.Cfull[k];
  }
  for (int k = tid; k < m * nc; k += kPT) {
    const int i = k / nc, t = k % nc;
    jsm[k] = a.J[static_cast<long long>(i) * a.ldj + c_lo + t];
    hsm[k] = a.Ht[static_cast<long long>(i) * a.ldh + c_lo + t];
  }
  // the operator rows this thread owns, decoded once
  RowCache<5> rq;
  RowCache<2> rt;
  RowCache<3> rd;
  rq.load(a.op.Qs, e0, has_e);
  rt.load(a.op.Dts, e0, has_e);
  rd.load(a.op.Ds, c0, has_c);
  const double qinv_e = has_e ? a.qinv[e0] : 0.0;
  if (tid == 0) ls = *a.st;
  __syncthreads();
  unsigned epoch = 0;
  const double nib = *a.neg_inv_beta;
  // optional phase profile (a.prof: 8 bins of nanoseconds, CTA 0): B, C, restrict, dense, up, F + A, tail
  unsigned long long tprev = 0;
  const bool prof = a.prof != nullptr && cta == 0 && tid == 0;
  auto lap = [&](int bin) {
    if (!prof) return;
    const unsigned long long t = gtime();
    a.prof[bin] += t - tprev;
    tprev = t;
  };
  double* part = a.part;

  // The operator y = A zhat on the own rows, zhat = z * ig, in two halves: the gathers (issued as
  // soon as z is complete) and the sums (once ig is known); delta partial -> slot 0.
  double gq[5], gt[2], gd[3], z_e = 0.0, z_c = 0.0, dq_c = 0.0;
  auto saddle_gather = [&](const double* __restrict__ z) {
    rq.gather(z, 0, gq);
    rt.gather(z, K, gt);
    rd.gather(z, 0, gd);
    z_e = has_e ? z[e0] : 0.0;
    z_c = has_c ? z[K + c0] : 0.0;
    dq_c = has_c ? a.dq[c0] : 0.0;
  };
  auto saddle_finish = [&](double ig, double* __restrict__ y) {
    double d[1] = {0.0};
    if (has_e) {
      const double sq = rq.dot(gq, ig), sd = rt.dot(gt, ig);
      double o = 0.0;
      o = o + 1.0 * sq;
      o = o + 1.0 * sd;
      y[e0] = o;
      d[0] = d[0] + o * (z_e * ig);
    }
    if (has_c) {
      const double sd = rd.dot(gd, ig);
      double o = 0.0;
      o = o + 1.0 * sd;
      o = o + nib * (dq_c * ig);  // J^T (J zhat2) = q * ig (Woodbury identity, lean schedule)
      y[K + c0] = o;
      d[0] = d[0] + o * (z_c * ig);
    }
    block_sum<1>(d, red);
    if (tid == 0) part[cta * kSlots + 5] = d[0];  // delta partial
  };

  int iters = 0;
  if (ls.status == kRunning) {
    saddle_gather(ring_slot(a.Z, 2, ls.j, 0));
    saddle_finish(ls.inv_gamma, a.az);
    grid_sync(a.bar, epoch);
  }
  if (prof) tprev = gtime();
  bool first_pass = true;
  double delta_next = 0.0;
  while (ls.status == kRunning && iters < a.max_iters) {
    const long long j = ls.j;
    const double* __restrict__ vp = ring_slot(a.V, 3, j, 0);
    const double* __restrict__ vc = ring_slot(a.V, 3, j, 1);
    double* __restrict__ vn = ring_slot(a.V, 3, j, 2);
    const double* __restrict__ zc = ring_slot(a.Z, 2, j, 0);
    double* __restrict__ zn = ring_slot(a.Z, 2, j, 1);
    // ---------------------------------------------------------------- B
    // the own rows of A zhat, v_cur, v_prev are loaded while the delta partials are summed
    const double az_e = has_e ? a.az[e0] : 0.0, vc_e = has_e ? vc[e0] : 0.0, vp_e = has_e ? vp[e0] : 0.0;
    const double az_c = has_c ? a.az[K + c0] : 0.0, vc_c = has_c ? vc[K + c0] : 0.0, vp_c = has_c ? vp[K + c0] : 0.0;
    {
      const double delta = first_pass ? total_of(part, 5) : delta_next;
      first_pass = false;
      if (tid == 0) {
        ls.delta = delta;
        ls.coef_v1 = -delta / ls.gamma_cur;
        ls.coef_v2 = -ls.gamma_cur / ls.gamma_prev;
      }
      __syncthreads();
    }
    const double c1 = ls.coef_v1, c2 = ls.coef_v2;
    double dots[3] = {0.0, 0.0, 0.0};  // <z, v>, <z, z>, <v, v>
    if (has_e) {
      double v = az_e + c1 * vc_e;
      v = v + c2 * vp_e;
      vn[e0] = v;
      const double z = qinv_e * v;
      zn[e0] = z;
      dots[0] = z * v;
      dots[1] = z * z;
      dots[2] = v * v;
    }
    double v2_own = 0.0;
    if (has_c) {
      double v = az_c + c1 * vc_c;
      v = v + c2 * vp_c;
      vn[K + c0] = v;
      v2_own = v;
      dots[2] = dots[2] + v * v;
    }
    v2sm[tid] = v2_own;
    __syncthreads();
    // partial t_i = sum over the own cells of Ht(i, c) v2(c): a warp per row i, from shared memory
    for (int i = warp; i < m; i += kPW) {
      double s = 0.0;
      for (int t = lane; t < nc; t += 32) s = s + hsm[i * nc + t] * v2sm[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) a.tpart[static_cast<long long>(cta) * m + i] = s;
    }
    grid_sync(a.bar, epoch);
    lap(0);
    // ---------------------------------------------------------------- C
    for (int i = warp; i < m; i += kPW) {  // t_i: the CTAs' partials in a fixed order (lanes, then the xor tree)
      double s = 0.0;
      for (int c = lane; c < nb; c += 32) s += __ldcg(&a.tpart[static_cast<long long>(c) * m + i]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) tsm[i] = s;
    }
    __syncthreads();
    if (tid < m) {  // t' = C^-1 t
      double s = 0.0;
      for (int k = 0; k < m; ++k) s = s + csm[tid * mp + k] * tsm[k];
      t2sm[tid] = s;
    }
    __syncthreads();
    if (tid < m) {  // one refinement step: t' += C^-1 (t - C t')
      double s = 0.0;
      for (int k = 0; k < m; ++k) s = s + cfm[tid * mp + k] * t2sm[k];
      rsm[tid] = tsm[tid] - s;
    }
    __syncthreads();
    if (tid < m) {
      double s = 0.0;
      for (int k = 0; k < m; ++k) s = s + csm[tid * mp + k] * rsm[k];
      t2sm[tid] = t2sm[tid] + s;
    }
    __syncthreads();
    if (has_c) {  // q = J^T t' (ascending rows), y' = v2 - q / beta
      double q = 0.0;
      for (int i = 0; i < m; ++i) q = q + jsm[i * nc + tid] * t2sm[i];
      a.dq[c0] = q;
      a.bq[c0] = v2_own + nib * q;
    }
    grid_sync(a.bar, epoch);
    lap(1);
    // ---------------------------------------------------------------- D: V-cycle of bq
    double dz[2] = {0.0, 0.0};  // <z2, v2>, <z2, z2> of the rows this CTA finishes
    auto store_top = [&](int i, double s) {
      zn[K + i] = s;
      const double v = vn[K + i];
      dz[0] = dz[0] + s * v;
      dz[1] = dz[1] + s * s;
    };
    auto dense_tail = [&](const double* __restrict__ rin, bool top, double* __restrict__ eout) {
      for (int i = cta * kPW + warp; i < a.nM; i += nb * kPW) {
        const double* __restrict__ row = a.M + static_cast<long long>(i) * a.nM;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int k = lane;
        for (; k + 480 < a.nM; k += 512) {  // 16 matrix loads in flight per lane
          double mm[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) mm[u] = __ldg(&row[k + 32 * u]);
#pragma unroll
          for (int u = 0; u < 16; u += 4) {
            s0 = s0 + mm[u] * rin[k + 32 * u];
            s1 = s1 + mm[u + 1] * rin[k + 32 * (u + 1)];
            s2 = s2 + mm[u + 2] * rin[k + 32 * (u + 2)];
            s3 = s3 + mm[u + 3] * rin[k + 32 * (u + 3)];
          }
        }
        for (; k + 96 < a.nM; k += 128) {
          const double m0 = __ldg(&row[k]), m1 = __ldg(&row[k + 32]), m2 = __ldg(&row[k + 64]), m3 = __ldg(&row[k + 96]);
          s0 = s0 + m0 * rin[k];
          s1 = s1 + m1 * rin[k + 32];
          s2 = s2 + m2 * rin[k + 64];
          s3 = s3 + m3 * rin[k + 96];
        }
        for (; k < a.nM; k += 32) s0 = s0 + __ldg(&row[k]) * rin[k];
        double s = (s0 + s1) + (s2 + s3);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
          if (top)
            store_top(i, s);
          else
            eout[i] = s;
        }
      }
    };
    if (a.nlev == 0) {
      dense_tail(a.bq, true, nullptr);
    } else {
      for (int l = 0; l < a.nlev; ++l) {  // r_{l+1} = T_l^T r_l
        const double* __restrict__ rl = l == 0 ? a.bq : a.vr[l];
        double* __restrict__ rc = a.vr[l + 1];
        GNW_P_LANES(a.gTt[l], (lell_rows<GG>(a.Tt[l], [&](int c) { return rl[c]; }, [&](int i, double s) { rc[i] = s; })));
        grid_sync(a.bar, epoch);
      }
      lap(2);
      dense_tail(a.vr[a.nlev], false, a.ve[a.nlev]);
      grid_sync(a.bar, epoch);
      lap(3);
      for (int l = a.nlev - 1; l >= 0; --l) {  // e_l = S_l r_l + T_l e_{l+1}
        const double* __restrict__ rl = l == 0 ? a.bq : a.vr[l];
        const double* __restrict__ ec = a.ve[l + 1];
        if (l == 0) {
          GNW_P_LANES(a.gS[0], (lell_rows2<GG>(a.S[0], a.T[0], [&](int c) { return rl[c]; }, [&](int c) { return ec[c]; },
                                               store_top)));
        } else {
          double* __restrict__ el = a.ve[l];
          GNW_P_LANES(a.gS[l], (lell_rows2<GG>(a.S[l], a.T[l], [&](int c) { return rl[c]; }, [&](int c) { return ec[c]; },
                                               [&](int i, double s) { el[i] = s; })));
          grid_sync(a.bar, epoch);
        }
      }
    }
    {  // dot partials: slots 1..3 = <z, v>, <z, z>, <v, v> (edge part from B + the cell rows finished here)
      double d5[3] = {dots[0] + dz[0], dots[1] + dz[1], dots[2]};
      block_sum<3>(d5, red);
      if (tid == 0) {
        part[cta * kSlots + 1] = d5[0];
        part[cta * kSlots + 2] = d5[1];
        part[cta * kSlots + 3] = d5[2];
      }
    }
    grid_sync(a.bar, epoch);
    lap(4);
    // ---------------------------------------------------------------- F (+ A of the next iteration)
    // z_next is complete: the next operator's gathers and the update's loads (all written before
    // this iteration's barriers) are issued before the dot totals are read
    saddle_gather(zn);
    const double* __restrict__ wp = ring_slot(a.W, 3, j, 0);
    const double* __restrict__ wc = ring_slot(a.W, 3, j, 1);
    double* __restrict__ wn = ring_slot(a.W, 3, j, 2);
    const double* __restrict__ up = ring_slot(a.U, 3, j, 0);
    const double* __restrict__ uc = ring_slot(a.U, 3, j, 1);
    double* __restrict__ un = ring_slot(a.U, 3, j, 2);
    double in_e[7], in_c[7];  // z_cur, w_prev, w_cur, u_prev, u_cur, x, r of the own edge / cell
#pragma unroll
    for (int k = 0; k < 7; ++k) in_e[k] = in_c[k] = 0.0;
    if (has_e) {
      in_e[0] = zc[e0], in_e[1] = wp[e0], in_e[2] = wc[e0], in_e[3] = up[e0], in_e[4] = uc[e0], in_e[5] = a.x[e0],
      in_e[6] = a.r[e0];
    }
    if (has_c) {
      const long long i = K + c0;
      in_c[0] = zc[i], in_c[1] = wp[i], in_c[2] = wc[i], in_c[3] = up[i], in_c[4] = uc[i], in_c[5] = a.x[i], in_c[6] = a.r[i];
    }
    {
      double t3[3];
      totals_of<3>(part, 1, t3);  // <z, v>, <z, z>, <v, v>
      if (tid == 0) givens_step(t3[0], t3[1], t3[2], &ls);
      __syncthreads();
    }
    if (ls.status != kRunning) break;  // kErrNotPD / kErrStagnated, the same on every CTA
    {
      const double ig = ls.inv_gamma, na3 = -ls.alpha3, na2 = -ls.alpha2, ia = ls.inv_alpha1;
      const double tau = ls.tau, ntau = -tau;
      double rr[1] = {0.0};
      auto upd = [&](long long i, const double (&in)[7], double azv) {  // minres.cpp:93-106
        const double zh = in[0] * ig;
        double w = zh + na3 * in[1];
        w = w + na2 * in[2];
        w = w * ia;
        double uu = azv + na3 * in[3];
        uu = uu + na2 * in[4];
        uu = uu * ia;
        wn[i] = w;
        un[i] = uu;
        a.x[i] = in[5] + tau * w;
        const double ro = in[6] + ntau * uu;
        a.r[i] = ro;
        rr[0] = rr[0] + ro * ro;
      };
      if (has_e) upd(e0, in_e, az_e);
      if (has_c) upd(K + c0, in_c, az_c);
      block_sum<1>(rr, red);
      if (tid == 0) part[cta * kSlots + 4] = rr[0];
    }
    // the own rows of az were read in phase B (registers): the next operator may overwrite them
    saddle_finish(1.0 / ls.gamma_next, a.az);  // iteration j + 1 reads z_next scaled by 1 / gamma_next
    grid_sync(a.bar, epoch);
    lap(5);
    {
      double t2[2];
      totals_of<2>(part, 4, t2);  // ||r||^2 and the next iteration's delta, one pass
      delta_next = t2[1];
      if (tid == 0) update_tail(t2[0], &ls, a.hist_e, a.hist_p, cta == 0 ? a.hist_cap : 0);
      __syncthreads();
    }
    lap(6);
    ++iters;
  }
  if (cta == 0 && tid == 0) *a.st = ls;
}

}  // namespace

int persistent_max_m() { return kMaxM; }

bool launch_minres_persistent(PersistArgs a, int sm_count, cudaStream_t s) {
  static bool ok = [] {
    int dev = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    return coop != 0;
  }();
  if (!ok || a.m < 1 || a.m > kMaxM) return false;
  if (a.op.Qs.width < 1 || a.op.Qs.width > 5 || a.op.Dts.width < 1 || a.op.Dts.width > 2 || a.op.Ds.width < 1 ||
      a.op.Ds.width > 3)
    return false;  // the register row caches hold triangle-mesh rows (5 + 2 and 3 entries)
  // As few CTAs as the one-row-per-thread ownership allows (~192 of the 256 threads own an edge):
  // a grid barrier costs less with fewer arrivals (C1: 128 CTAs 0.034 ms per iteration, 64 CTAs
  // 0.032), and the level phases still have a warp per row slice.
  static const int env_ctas = [] {  // env GNW_PERSIST_CTAS: the CTA count (experiments)
    const char* e = std::getenv("GNW_PERSIST_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  long long want = std::max<long long>((a.K + 191) / 192, (a.N + 191) / 192);
  if (env_ctas > 0) want = env_ctas;
  const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(sm_count, want)));
  const long long e_max = (a.K + grid - 1) / grid + 1, c_max = (a.N + grid - 1) / grid + 1;
  if (e_max > kPT || c_max > kPT) return false;
  const size_t smem = (static_cast<size_t>(2) * a.m * (a.m + 1) + static_cast<size_t>(2) * a.m * c_max) * sizeof(double);
  constexpr int kSmemCap = 200 * 1024;
  if (smem > kSmemCap) return false;
  // the opt-in is recorded once per (kernel, device): always ask for the cap, not this launch's size
  smem_optin(reinterpret_cast<const void*>(k_minres_persistent), kSmemCap);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_minres_persistent, kPT, smem) != cudaSuccess || per_sm < 1)
    return false;
  if (cudaMemsetAsync(a.bar, 0, 64 * sizeof(unsigned), s) != cudaSuccess) return false;
  void* args[] = {&a};
  // a cooperative launch fails (rather than deadlocks) when the grid cannot be co-resident, e.g.
  // with another process on the GPU: the caller then runs the graph loop
  if (cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_minres_persistent), dim3(grid), dim3(kPT), args, smem,
                                  s) != cudaSuccess) {
    cudaGetLastError();  // clear the launch error
    return false;
  }
  note_launch("minres_persistent");
  return true;
}

}  // namespace gnw
