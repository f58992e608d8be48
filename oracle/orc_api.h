/*
 * orc_api.h -- C API shared by the two CPU oracles (TEST INFRASTRUCTURE ONLY).
 *
 * Two libraries export exactly these symbols:
 *   oracle/_ref/libertinv_ref.so   the UNMODIFIED reference sources under
 *                                  /root/reference/proj/src compiled by
 *                                  oracle/Makefile, wrapped by oracle/ref_capi.cpp
 *   oracle/build/liborc.so         oracle/gnw_oracle.c, a plain-C restatement of
 *                                  the same algorithms (file:line cited per function)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load either library, and only as the checker or the CPU
 * baseline.  The product (paper_2209_02815_b200/, libgnw.so) never links them.
 *
 * Status codes: 0 ok, 1 invalid argument (std::invalid_argument in the
 * reference), 2 numerical failure (std::runtime_error).  Message: orc_last_error().
 */
#ifndef ORC_API_H
#define ORC_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_amg_opts {
  uint64_t coarse_threshold;      /* AmgOptions::coarse_threshold   amg.hpp:12 */
  double strength;                /* AmgOptions::strength           amg.hpp:13 */
  double jacobi_damping;          /* amg.hpp:14 */
  double prolongation_damping;    /* amg.hpp:15 */
  uint64_t max_aggregate_size;    /* amg.hpp:19 */
  uint64_t max_levels;            /* amg.hpp:20 */
} orc_amg_opts;

typedef struct orc_problem orc_problem;

typedef struct orc_minres_report {
  uint64_t iterations;
  int32_t converged;
  double true_relative_residual;
  uint64_t n_hist;            /* entries written to the history arrays */
} orc_minres_report;

const char* orc_last_error(void);
const char* orc_flavor(void); /* "reference" or "restatement" */

/* Mixed problem from raw mesh arrays: finalize_mesh + make_mixed_spaces +
 * assemble_Q/D + 1/diag(Q) + amg_setup(assemble_lumped_schur(Q, D), opts)
 * (inversion.cpp:196-213). */
orc_problem* orc_create_mixed(const double* vertices, uint64_t n_vertices,
                              const int64_t* cells, uint64_t n_cells,
                              const orc_amg_opts* opts);
/* Plain AMG hierarchy over a caller CSR matrix (amg_setup amg.cpp:115-187). */
orc_problem* orc_create_amg_csr(uint64_t n, const int64_t* rowptr, const int64_t* cols,
                                const double* vals, const orc_amg_opts* opts);
void orc_destroy(orc_problem* p);

/* sizes[0]=K sizes[1]=N sizes[2]=n_vertices sizes[3]=n_cells sizes[4]=n_edges
 * sizes[5]=n_levels sizes[6]=n_boundary_edges sizes[7]=coarse n */
int orc_sizes(const orc_problem* p, uint64_t sizes[8]);

/* Mesh connectivity (mesh.cpp:85-154). Any pointer may be NULL. */
int orc_mesh(const orc_problem* p, int64_t* cells, int64_t* edges, int64_t* cell_edges,
             int32_t* cell_edge_signs, int64_t* boundary_edges, int32_t* boundary_tags);

/* CSR export. which: 0=Q 1=D 2=S_hat 3=A_level 4=P_level.  Call with NULL
 * arrays to query dims/nnz. */
int orc_csr(const orc_problem* p, int which, uint64_t level, uint64_t* n_rows,
            uint64_t* n_cols, uint64_t* nnz, int64_t* rowptr, int64_t* cols, double* vals);
int orc_level_inv_diag(const orc_problem* p, uint64_t level, double* out);
int orc_coarse_cholesky(const orc_problem* p, double* out); /* n_c x n_c row-major */
int orc_q_diag_inv(const orc_problem* p, double* out);

int orc_amg_apply(const orc_problem* p, const double* r, double* z);

/* build_woodbury_preconditioner (inversion.cpp:91-124); m == 0 selects the
 * plain Laplace preconditioner (inversion.cpp:251-256).  timings: t_H, t_C, t_chol. */
int orc_set_jacobian(orc_problem* p, const double* J, uint64_t m, double beta,
                     double timings[3]);
/* Alg. 4 (GnAlgorithm::kLaplaceMinres, inversion.cpp:251-256): the next
 * orc_set_jacobian keeps J in the operator but builds the plain Laplace
 * preconditioner (pc.J = nullptr). */
int orc_set_pc_laplace(orc_problem* p, int laplace);
int orc_get_H(const orc_problem* p, double* out);   /* N x m row-major */
int orc_get_L(const orc_problem* p, double* out);   /* m x m row-major */

int orc_apply_operator(const orc_problem* p, const double* x, double* y);
int orc_precondition(const orc_problem* p, const double* y, double* z);
int orc_assemble_rhs(const orc_problem* p, const double* m, const double* m_ref,
                     const double* g, const double* g_obs, double* rhs);
int orc_minres(const orc_problem* p, const double* b, const double* x0, double tol,
               uint64_t maxit, double* x, orc_minres_report* rep, double* hist_euclid,
               double* hist_pnorm, uint64_t hist_cap);

/* Bounded timing sample of one GN-step solve (reference library only; see
 * ref_capi.cpp): out = {s per H column, s per C row, s Cholesky, s per MINRES iteration,
 * s of minres's fixed start-up (r0 = b - A x0, first preconditioner application)}. */
int orc_sample_gnstep(orc_problem* p, const double* J, uint64_t m, double beta, uint64_t k_cols,
                      uint64_t k_rows, uint64_t k_iters, double out[5]);

/* ERT forward model on the mixed problem's mesh: evaluate_response_and_jacobian
 * (forward.cpp:100-172) with Mesh::electrode_nodes = nodes, configs (a, b, m, n, k)
 * (b = -1: pole at infinity).  J is n_cfg x N row-major. */
int orc_response_jacobian(orc_problem* p, const int64_t* nodes, uint64_t n_nodes, const int64_t* a,
                          const int64_t* b, const int64_t* m, const int64_t* n, const double* k, uint64_t n_cfg,
                          const double* model, double* J, double* g);
/* gauss_newton (inversion.cpp:187-292), reference library only (the restatement composes it
 * in orc.py from the functions above).  algorithm: 0 kWoodburyMinres, 1 kLaplaceMinres.
 * steps: n_steps x {misfit, minres_iters, converged, euclid rel. residual, pnorm rel. residual}. */
int orc_gauss_newton(orc_problem* p, const int64_t* nodes, uint64_t n_nodes, const int64_t* a, const int64_t* b,
                     const int64_t* m, const int64_t* n, const double* k, uint64_t n_cfg, const double* g_obs,
                     const double* m_ref, const double* m0, double beta, uint64_t max_outer_steps, double minres_tol,
                     uint64_t minres_maxit, int algorithm, double misfit_reduction_tol, double* m_out,
                     double* steps, uint64_t steps_cap, uint64_t* n_steps, double* final_misfit);
/* The reference's file formats (reference library only): mesh JSON (mesh.cpp:331-383),
 * survey CSV (survey.cpp:81-116), model JSON (kind 0) / observations CSV (kind 1)
 * (forward.cpp:174-219), result JSON (inversion.cpp:294-317; steps: 9 doubles each).
 * Readers: call with NULL arrays for the counts first. */
int orc_io_write_mesh(orc_problem* p, const int64_t* electrodes, uint64_t ne, const char* path);
int orc_io_read_mesh(const char* path, uint64_t* nv, uint64_t* nc, uint64_t* ne, double* vertices, int64_t* cells,
                     int64_t* electrodes);
int orc_io_write_survey(const int64_t* a, const int64_t* b, const int64_t* m, const int64_t* n, const double* k,
                        uint64_t count, const char* path);
int orc_io_read_survey(const char* path, uint64_t* count, int64_t* a, int64_t* b, int64_t* m, int64_t* n, double* k);
int orc_io_write_vector(int kind, const double* v, uint64_t count, const char* path);
int orc_io_read_vector(int kind, const char* path, uint64_t* count, double* v);
int orc_io_write_result(const double* m, uint64_t N, const double* steps, uint64_t n_steps, double final_misfit,
                        uint64_t K, uint64_t M, const char* path);
/* geometric_factor (survey.cpp:22-46); b == NULL: pole at infinity. */
int orc_geometric_factor(const double a[3], const double* b, const double m[3], const double n[3], int dim,
                         double* k);

/* Dense Cholesky (linalg.cpp:88-105): returns 2 on a non-positive pivot. */
int orc_dense_cholesky(uint64_t n, const double* C, double* L);

#ifdef __cplusplus
}
#endif

#endif
