// minres_persistent.cuh -- arguments of the persistent cooperative MINRES kernel
// (minres_persistent.cu): the whole loop of minres.cpp:70-148 in one launch, for L2-resident
// problems (BASELINE C1).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace gnw {

constexpr int kPersistMaxLevels = 8;

struct PersistArgs {
  OperatorArgs op;  // SELL copies of Q, D^T, D
  long long K = 0, N = 0;
  int m = 0;
  const double* qinv = nullptr;
  const double* Ht = nullptr;
  long long ldh = 0;
  const double* J = nullptr;
  long long ldj = 0;
  const double* Cinv = nullptr;
  const double* Cfull = nullptr;
  const double* neg_inv_beta = nullptr;
  // MINRES vectors (rings indexed by the iteration counter)
  double* V[3] = {};
  double* W[3] = {};
  double* U[3] = {};
  double* Z[3] = {};  // two slots
  double *az = nullptr, *x = nullptr, *r = nullptr, *bq = nullptr, *dq = nullptr;
  MinresState* st = nullptr;
  double *hist_e = nullptr, *hist_p = nullptr;
  long long hist_cap = 0;
  // V-cycle: nlev one-pass lane-ELL levels above the dense tail M (nM x nM)
  int nlev = 0;
  DLell Tt[kPersistMaxLevels], S[kPersistMaxLevels], T[kPersistMaxLevels];
  int gTt[kPersistMaxLevels] = {}, gS[kPersistMaxLevels] = {};
  double* vr[kPersistMaxLevels + 1] = {};
  double* ve[kPersistMaxLevels + 1] = {};
  const double* M = nullptr;
  int nM = 0;
  // scratch: 8 partial-sum slots per CTA, m partials of t per CTA, the barrier counter
  double* part = nullptr;
  double* tpart = nullptr;
  unsigned* bar = nullptr;
  int max_iters = 0;
  unsigned long long* prof = nullptr;  // optional: 8 phase bins (ns) accumulated by CTA 0
};

// largest m the kernel handles (C and C^-1 live in shared memory)
int persistent_max_m();
// false: not launched (no cooperative launch, m out of range)
bool launch_minres_persistent(PersistArgs a, int sm_count, cudaStream_t s);

}  // namespace gnw
