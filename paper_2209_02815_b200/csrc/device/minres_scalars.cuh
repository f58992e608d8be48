// minres_scalars.cuh -- the scalar epilogues of the MINRES iteration shared by the kernels that
// end a phase with a grid reduction (kernels.cu k_finish_prec, vcycle_fused.cu's fused last
// level): gamma_next and the Givens rotation of minres.cpp:79-101.
#pragma once

#include "common.cuh"

namespace gnw {

// minres.cpp:79-101: gamma_next and the Givens rotation from <z,v>, <z,z>, <v,v>
__device__ __forceinline__ void givens_step(double gsq, double zz, double vv, MinresState* st) {
  if (gsq < -1e-12 * (sqrt(zz) * sqrt(vv) + 1.0)) {
    st->status = kErrNotPD;
    return;
  }
  const double gamma_next = sqrt(fmax(gsq, 0.0));
  const double delta = st->delta, gc = st->gamma_cur;
  const double alpha0 = st->c_cur * delta - st->c_prev * st->s_cur * gc;
  const double alpha1 = sqrt(alpha0 * alpha0 + gamma_next * gamma_next);
  const double alpha2 = st->s_cur * delta + st->c_prev * st->c_cur * gc;
  const double alpha3 = st->s_prev * gc;
  if (alpha1 == 0.0) {
    st->status = kErrStagnated;
    return;
  }
  st->gamma_next = gamma_next;
  st->c_next = alpha0 / alpha1;
  st->s_next = gamma_next / alpha1;
  st->alpha2 = alpha2;
  st->alpha3 = alpha3;
  st->inv_alpha1 = 1.0 / alpha1;
  st->tau = st->c_next * st->eta;
  st->eta = -st->s_next * st->eta;
}


// k_finish_prec's tail: add the combine kernel's partials (edge blocks: all three; cell
// blocks: <v,v>) to the cell totals, then gamma_next and the Givens rotation.
__device__ __forceinline__ void finish_scalars(const double (&tot)[3], const double* __restrict__ dots_edge, int n_edge_blocks,
                               int loop, MinresState* st, double* red) {
  double e3[3] = {0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < n_edge_blocks; b += blockDim.x)
    for (int k = 0; k < 3; ++k) e3[k] += __ldcg(&dots_edge[b * 3 + k]);
  block_reduce<3>(e3, red);
  if (threadIdx.x != 0) return;
  const double gsq = e3[0] + tot[0], zz = e3[1] + tot[1], vv = e3[2] + tot[2];
  if (!loop) {
    st->scratch[0] = gsq;
    st->scratch[1] = zz;
    st->scratch[2] = vv;
    return;
  }
  givens_step(gsq, zz, vv, st);
}

// minres.cpp:93-148 after the vector updates: history, convergence / exhaustion, rotation, j++
__device__ __forceinline__ void update_tail(double rr, MinresState* st, double* hist_e, double* hist_p, long long hist_cap) {
  const long long j = st->j;
  const double rel = sqrt(rr) / st->bnorm;
  st->iterations = j;
  st->rel = rel;
  if (j < hist_cap) {
    hist_e[j] = rel;
    hist_p[j] = fabs(st->eta) / st->gamma1;
  }
  if (rel <= st->tol) {
    st->status = kVerify;
  } else if (st->gamma_next <= st->exhausted_tol) {
    st->status = kExhausted;
  } else {
    st->gamma_prev = st->gamma_cur;
    st->gamma_cur = st->gamma_next;
    st->c_prev = st->c_cur;
    st->c_cur = st->c_next;
    st->s_prev = st->s_cur;
    st->s_cur = st->s_next;
    st->inv_gamma = 1.0 / st->gamma_cur;
    st->j = j + 1;
    if (j + 1 > st->maxit) st->status = kMaxit;
  }
}

}  // namespace gnw
