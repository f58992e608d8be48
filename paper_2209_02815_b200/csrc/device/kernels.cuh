// kernels.cuh -- launch interfaces of the gnw device kernels (sm_100a, FP64).
// Reference citations are to /root/reference/proj.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace gnw {

// One level of the device AMG hierarchy (amg.hpp:25-29).  R = P^T stored
// explicitly so restriction is a gather (rows of R sorted by fine index, which
// reproduces spmv_transpose's scatter order, sparse.cpp:85-95).
struct DLevel {
  DCsr A, P, R;
  double* wd = nullptr;  // omega * inv_diag (rounded exactly as amg.cpp:98)
  int n = 0;             // rows of A
  // lanes per row of the single-RHS kernels (vcycle_wide.cu): 1 = thread-per-row in the
  // reference order (kernels.cu), 2..32 = a G-lane group per row
  int gA = 1, gP = 1, gR = 1;
  // SELL-32 copies for the thread-per-row kernels (same order, coalesced; width 0: CSR)
  DSell As, Ps, Rs;
  // default-mode one-pass-per-direction operators (vcycle_fused.cu, host::fused_cycle_ops):
  // r_c = Tt r, e = S r + T e_c; fused = 0: not built for this level
  DCsr S, T, Tt;
  int gS = 1, gTt = 1, fused = 0;
  // lane-ELL copies with coded values read by the single-RHS kernels (words == nullptr: CSR)
  DLell Sl, Tl, Ttl;
};

// one pass per level each way (vcycle_fused.cu): rc = Tt r; out = S r + T ec
void vcf_restrict(const DLevel& L, VSel r, double* rc, const MinresState* st, cudaStream_t s);
void vcf_up(const DLevel& L, VSel r, const double* ec, double* out, const MinresState* st, cudaStream_t s);
void mvcf_restrict(const DLevel& L, const double* r, double* rc, int b, cudaStream_t s);
// with ht != nullptr the result may go straight to Ht rows (returns true when it did)
bool mvcf_up(const DLevel& L, const double* r, const double* ec, double* out, int b, double* ht, long long ldh,
             cudaStream_t s);

// G-lanes-per-row kernels (vcycle_wide.cu), G = DLevel::gA / gR / gP
void vcg_down(const DLevel& L, VSel r, double* resid, const MinresState* st, cudaStream_t s);
void vcg_restrict(const DLevel& L, const double* resid, double* rc, cudaStream_t s);
void vcg_up1(const DLevel& L, VSel r, const double* ec, double* x, const MinresState* st, cudaStream_t s);
void vcg_up2(const DLevel& L, VSel r, const double* x, double* out, const MinresState* st, cudaStream_t s);
// lanes per row for a matrix with `nnz` entries over `rows` rows (env GNW_VC_T tunes it)
int vc_group_lanes(long long nnz, long long rows);

// narrow-level batched kernels, 2 columns per thread (vcycle_batch.cu); even b only
void mvc2_down(const DLevel& L, const double* r, int ldr, double* resid, int b, cudaStream_t s);
void mvc2_restrict(const DLevel& L, const double* resid, double* rc, int b, cudaStream_t s);
void mvc2_up1(const DLevel& L, const double* r, int ldr, const double* ec, double* x, int b, cudaStream_t s);
void mvc2_up2(const DLevel& L, const double* r, int ldr, const double* x, double* out, int ldo, int b,
              cudaStream_t s);
// level-0 up2 storing straight into rows of Ht (ht = &Ht[r0 * ldh], column i = fine row);
// false when the shape does not fit (V = 2, 32 lanes per row, n % 8 == 0) -- nothing launched
bool mvc2_up2_rows(const DLevel& L, const double* r, int ldr, const double* x, double* ht, long long ldh, int b,
                   cudaStream_t s);

// ------------------------------------------------------------------ V-cycle
// Single right-hand side (amg.cpp:90-111); `r` may be a ring slot (level 0).
void vc_down(const DLevel& L, VSel r, double* resid, const MinresState* st, cudaStream_t s);
void vc_restrict(const DLevel& L, const double* resid, double* rc, cudaStream_t s);
void vc_up1(const DLevel& L, VSel r, const double* ec, double* x, const MinresState* st, cudaStream_t s);
void vc_up2(const DLevel& L, VSel r, const double* x, double* out, const MinresState* st, cudaStream_t s);
// coarsest level: x = A_c^-1 r (explicit inverse, warp per row)
void coarse_inverse(const double* Ainv, int n, VSel r, double* x, const MinresState* st, int nrhs,
                    cudaStream_t s);
// coarsest level, reference cholesky_solve replayed (linalg.cpp:107-123), one thread per rhs
void coarse_cholesky(const double* L, int n, VSel r, double* x, const MinresState* st, int nrhs,
                     int ld, cudaStream_t s);

// Multi right-hand side (b columns interleaved: X[row * ld + q]); per column
// bit-identical to the single-RHS kernels.
void mvc_down(const DLevel& L, const double* r, int ldr, double* resid, int b, cudaStream_t s);
void mvc_restrict(const DLevel& L, const double* resid, double* rc, int b, cudaStream_t s);
void mvc_up1(const DLevel& L, const double* r, int ldr, const double* ec, double* x, int b, cudaStream_t s);
void mvc_up2(const DLevel& L, const double* r, int ldr, const double* x, double* out, int ldo, int b,
             cudaStream_t s);
void mcoarse_inverse(const double* Ainv, int n, const double* r, double* x, int b, cudaStream_t s);
// batched dense apply in sequential order (the batched V-cycle's collapsed tail)
void dense_seq_batch(const double* M, int n, const double* X, double* Y, int b, cudaStream_t s);
void identity_rows(double* I, int n, cudaStream_t s);
void transpose_square(const double* A, double* T, int n, cudaStream_t s);


// rows [r0, r0+b) of a row-major (rows x cols) matrix -> cols x b interleaved
void transpose_rows_to_batch(const double* A, long long cols, long long ld, int r0, int b, double* X,
                             cudaStream_t s);
// cols x b interleaved -> rows [r0, r0+b) of a row-major (rows x cols) matrix
void transpose_batch_to_rows(const double* X, long long cols, long long ld, int r0, int b, double* A,
                             cudaStream_t s);

// ---------------------------------------------------------------- operator
struct OperatorArgs {
  DCsr Q, D, Dt;       // Dt = D^T (rows = edges, columns = cells ascending)
  DSell Qs, Ds, Dts;   // SELL-32 copies read by k_saddle (width 0: CSR loops)
  const double* J = nullptr;  // m x N row-major (nullptr: no low-rank term)
  int m = 0;
  long long K = 0, N = 0;
  long long ldj = 0;  // row stride of J (>= N; padded to spread DRAM channels)
  const double* neg_inv_beta = nullptr;  // device scalar -1/beta (graph-stable across beta)
  // Woodbury-fused loop: J^T u = (J^T t') / gamma with q = J^T t'
  // produced by the previous preconditioner pass; J is then not read by the operator.
  const double* q = nullptr;
};

// u = A[:, ] x2 * scale partial GEMV over rows of a row-major (m x N) matrix,
// scale = st->inv_gamma when scaled != 0 (zhat = z / gamma), else 1.
struct RowGemv {
  int chunk = 0, nchunks = 0, ngroups = 0;
};
RowGemv row_gemv_plan(long long N, int m, int reserve = 0);
// number of blocks of the elementwise combine kernel (dots partials)
int combine_blocks(long long K, long long N);
// out[0..2] = the n triples of parts summed in a fixed order (one CTA)
void sum_triples(const double* parts, int n, double* out, cudaStream_t s);
void row_gemv(const double* A, int m, long long N, long long ld, VSel x, long long x_off, int scaled,
              const MinresState* st, double* partial, unsigned* counter, double* out,
              const RowGemv& plan, cudaStream_t s);

// y = A x (saddle operator, inversion.cpp:47-69) with x = z * scale; u = J x2
// precomputed.  When `loop`, the last block stores delta = <y, x> and the
// v-combination coefficients into st (minres.cpp:74-77).
void saddle_operator(const OperatorArgs& op, VSel x, int scaled, const double* u, VSel y,
                     MinresState* st, int loop, double* partial, unsigned* counter, cudaStream_t s);

// --------------------------------------------------------- preconditioner
struct PrecArgs {
  const double* qinv = nullptr;
  const double* Ht = nullptr;   // m x N row-major (H^T; h_hat(c, i) = Ht[i * N + c])
  const double* Cinv = nullptr; // m x m (explicit capacitance inverse)
  const double* Lc = nullptr;   // m x m lower Cholesky factor of C (exact mode)
  int m = 0;
  long long K = 0, N = 0;
  long long ldh = 0, ldj = 0;  // row strides of Ht and J
  const double* neg_inv_beta = nullptr;
  int exact = 0;
  // ill-conditioned C (set_jacobian's estimate from diag(L)): C^-1 t by the two triangular
  // solves with L instead of the explicit inverse, whose error grows like eps kappa(C)
  int cap_tri = 0;
  // fused loop: the finish pass also forms q = J^T t' (J read in the same sweep as H)
  const double* J = nullptr;
  double* q = nullptr;
  // fused/lean loops: t2 = C^-1 t refined once against the full C (cres: m scratch)
  const double* Cfull = nullptr;
  double* cres = nullptr;
};

// v_next = Az + c1 v_cur + c2 v_prev (combine, minres.cpp:76-77) or, when
// !loop, v_next = y (plain preconditioner input); z1 = qinv * v1; partial
// dots; t = Ht v2 (row GEMV) reduced by the last block into t_out.
// the element part of combine_precondition (v_next, z_next edge part, dots) alone
void combine_elem(const PrecArgs& pa, VSel az, VSel vcur, VSel vprev, VSel vnext, VSel znext, int loop,
                  MinresState* st, double* dots_part, cudaStream_t s);
void combine_precondition(const PrecArgs& pa, VSel az, VSel vcur, VSel vprev, VSel vnext, VSel znext,
                          int loop, MinresState* st, double* vcopy, double* dots_part,
                          double* t_part, unsigned* counter, double* t_out, const RowGemv& plan,
                          cudaStream_t s);
// q_c = sum_i A[i * ld + c] t[i] in ascending i for c < n (column sweep, lean loop's J^T t');
// with yout: also yout_c = y[yoff + c] + (*coef) q_c (the lean loop's V-cycle input v2 - q / beta)
void col_sweep(const double* A, long long ld, const double* t, int m, long long n, double* q, cudaStream_t s,
               VSel ys = VSel{}, long long yoff = 0, const MinresState* st = nullptr, const double* coef = nullptr,
               double* yout = nullptr);
// upper triangle of C := its lower triangle
void mirror_lower(double* C, int n, cudaStream_t s);
// t2 = C^-1 t (inverse apply) or the exact cholesky_solve (exact mode)
void capacitance_solve(const PrecArgs& pa, const double* t, double* t2, cudaStream_t s);
// z2 = s + (-1/beta) H t2; dots <z, v>, ||z||^2; last block: Givens update
// (minres.cpp:78-101) when loop, else totals to st->scratch.
int finish_blocks(const PrecArgs& pa);
void finish_precondition(const PrecArgs& pa, const double* svc, const double* t2, VSel vnext,
                         VSel znext, int loop, MinresState* st, const double* dots_edge,
                         int n_edge_blocks, double* part, unsigned* counter, cudaStream_t s);

// w/u/x/r recurrences (minres.cpp:93-106) + ||r||; last block: history,
// convergence/exhaustion checks, rotation, graph loop condition.
void minres_update(long long n, VSel z, VSel az, VSel wprev, VSel wcur, VSel wnext, VSel uprev,
                   VSel ucur, VSel unext, double* x, double* r, MinresState* st, double* hist_e,
                   double* hist_p, long long hist_cap, double* part, unsigned* counter,
                   unsigned long long cond_handle, int use_cond, cudaStream_t s);
// host-driven continuation after a failed verification: rotation + j++
void minres_rotate(MinresState* st, cudaStream_t s);

// r = b - y and ||r||^2 -> st->scratch[4] (and ||b||^2 -> scratch[5] when want_b)
void residual(long long n, const double* b, const double* y, double* r, MinresState* st, int want_b,
              double* part, unsigned* counter, cudaStream_t s);
// dot products for the generic entry points: out[0] = <a, b>
void dot(long long n, const double* a, const double* b, double* out, double* part, unsigned* counter,
         cudaStream_t s);

// rhs = [-D^T (m - m_ref); J^T (g - g_obs) / beta]  (inversion.cpp:126-146)
// rhs = [-D^T (mdl - mref); J^T (g - gobs) / beta]  (assemble_gn_rhs, inversion.cpp:126-146)
void assemble_rhs(const OperatorArgs& op, double beta, const double* mdl, const double* mref, const double* g,
                  const double* gobs, double* rhs, cudaStream_t s);

// ------------------------------------------------------------- dense / DMMA
// C = I + (J Ht^T) / beta, lower triangle (or full) by split-K FP64 DMMA.
struct DgemmPlan {
  int tile = 0, ntiles = 0, npairs = 0, splits = 0;
  long long kchunk = 0;
  int full = 0;
};
DgemmPlan dgemm_plan(int m, long long N, int full, int sm_count);
void capacitance_dgemm(const double* J, long long ldj, const double* Ht, long long ldh, int m, long long N,
                       double beta, const DgemmPlan& plan, double* part, double* C, cudaStream_t s);
// the split-K partial tiles by the TMA-staged kernel (dgemm_tma.cu); false when it cannot run
bool capacitance_dgemm_tma(const double* J, long long ldj, const double* Ht, long long ldh, int m, long long N,
                           const DgemmPlan& plan, const int2* dpairs, double* part, cudaStream_t s);
// dense_cholesky (linalg.cpp:88-105), operation order preserved; *fail = 1 on a
// non-positive pivot.
void cholesky(const double* C, double* L, int n, int* fail, cudaStream_t s);
// the same factorisation, blocked right-looking with per-element sequential
// updates (dense.cu): bit-identical to the reference, O(m) critical path.  W: m x m work
void cholesky_blocked(const double* C, double* W, double* L, int n, int* fail, cudaStream_t s);
// Y = L^-1 by 32-row blocks (dense.cu)
void trinv_blocked(const double* L, double* Y, int n, cudaStream_t s);
// symmetrize C in place (cholesky_with_retry, inversion.cpp:24-33)
void symmetrize(double* C, int n, cudaStream_t s);
// Cinv = L^-T L^-1
void cholesky_inverse(const double* L, double* Y, double* Cinv, int n, cudaStream_t s);

void fill_zero(double* p, long long n, cudaStream_t s);

// ---- partitioned (multi-GPU) solve (context_rowpart.cu) ----
// st->scratch[k0 + i] = sum over ranks r (in rank order) of parts[r * cnt + i]
void sum_scratch(const double* parts, int P, int cnt, MinresState* st, int k0, cudaStream_t s);
// the saddle kernel's loop epilogue (delta, v-combination coefficients) from scratch[0]
void delta_coef(MinresState* st, cudaStream_t s);
// the finish kernel's loop epilogue (gamma_next, Givens rotation; minres.cpp:79-101) from scratch[0..2]
void givens_from_scratch(MinresState* st, cudaStream_t s);
// the update kernel's epilogue (history, convergence, rotation) from scratch[6] = ||r||^2
void update_tail_from_scratch(MinresState* st, double* hist_e, double* hist_p, long long hist_cap, cudaStream_t s);
// out[i] = sum_{r < P} parts[r * n + i], r ascending (deterministic allreduce body)
void sum_partials(const double* parts, int P, long long n, double* out, cudaStream_t s);
// C = I + (sum_r parts[r]) / beta, parts m x m each (capacitance, inversion.cpp:37-43)
void capacitance_reduce(const double* parts, int P, int m, double beta, double* C, cudaStream_t s);

}  // namespace gnw
