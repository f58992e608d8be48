/*
 * gnw.h -- C-ABI of the B200-native Woodbury-MINRES Gauss-Newton step solver
 * (arXiv 2209.02815; reference: /root/reference/proj, "ertinv").
 *
 * This is the drop-in boundary.  Plain pointers and
 * sizes only; no torch or CUDA types.  Every entry point names the reference
 * interface it replaces.  All floating point is FP64.
 *
 *   gnw_assemble         <- make_mixed_spaces + assemble_Q/assemble_D + 1/diag(Q)
 *                           + amg_setup(assemble_lumped_schur(Q, D), opts)
 *                           (proj/src/inversion.cpp:196-213; fem_mixed.hpp:28-38;
 *                           amg.hpp:44; finalize_mesh mesh.hpp:53-55)
 *   gnw_set_jacobian     <- build_woodbury_preconditioner(q_diag_inv, amg, J, beta,
 *                           timings*) (inversion.hpp:47-50, inversion.cpp:91-124) and
 *                           SaddleOperator{&Q, &D, &J, beta} (inversion.cpp:258);
 *                           m == 0 selects the plain Laplace preconditioner
 *                           (inversion.cpp:251-256, Alg. 4)
 *   gnw_apply_operator   <- SaddleOperator::apply (inversion.hpp:25, inversion.cpp:47-69)
 *   gnw_precondition     <- WoodburyPreconditioner::apply (inversion.hpp:38,
 *                           inversion.cpp:71-89)
 *   gnw_amg_apply        <- amg_apply (amg.hpp:47, amg.cpp:189-194)
 *   gnw_assemble_rhs     <- assemble_gn_rhs (inversion.hpp:53-55, inversion.cpp:126-146)
 *   gnw_minres_solve     <- minres(apply_A, apply_Pinv, b, x0, tol, maxit)
 *                           (minres.hpp:29-33, minres.cpp:20-155) with A/P bound to the
 *                           context's operator and preconditioner
 *   gnw_dense_cholesky   <- dense_cholesky (linalg.hpp:44, linalg.cpp:88-105), on device
 *
 * Error convention (reference: std::invalid_argument / std::runtime_error,
 * SURVEY.md 8(b)): every call returns GNW_OK or a status; gnw_last_error()
 * returns the thread-local message, whose text matches the reference's
 * exception text (e.g. "minres: breakdown (stagnated rotation)").
 *
 * Pointer mode: by default vector arguments are HOST pointers (copied in/out
 * on the context's stream).  gnw_set_pointer_mode(ctx, GNW_DEVICE_POINTERS)
 * makes them device pointers on the context's device (no copies).
 */
#ifndef GNW_H
#define GNW_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gnw_status {
  GNW_OK = 0,
  GNW_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  GNW_NUMERICAL = 2,        /* std::runtime_error in the reference */
  GNW_DEVICE = 3            /* CUDA / NCCL failure (no reference analogue) */
} gnw_status;

enum { GNW_HOST_POINTERS = 0, GNW_DEVICE_POINTERS = 1 };

/* Coarsest-level solve of the V-cycle.  GNW_COARSE_INVERSE (default) applies
 * the explicit inverse of the coarsest Galerkin matrix (one GEMV); the
 * GNW_COARSE_CHOLESKY mode replays the reference's cholesky_solve
 * (linalg.cpp:107-123) operation-for-operation so a V-cycle is bit-identical
 * to amg_apply (used by the parity tests). */
enum { GNW_COARSE_INVERSE = 0, GNW_COARSE_CHOLESKY = 1 };

/* Preconditioner of the next gnw_set_jacobian (GnConfig::algorithm,
 * inversion.hpp:64): Alg. 3 Laplace-Woodbury (default) or Alg. 4 Laplace-only,
 * where J stays in the operator and the Schur block is the bare V-cycle
 * (inversion.cpp:251-256). */
enum { GNW_PC_WOODBURY = 0, GNW_PC_LAPLACE = 1 };

typedef struct gnw_ctx gnw_ctx;

/* AmgOptions, proj/include/ertinv/amg.hpp:11-23 (exact_solve is not supported:
 * it needs a sparse LU and is an oracle-only mode of the reference). */
typedef struct gnw_amg_options {
  uint64_t coarse_threshold;   /* default 64 */
  double strength;             /* default 0.08 */
  double jacobi_damping;       /* default 2/3 */
  double prolongation_damping; /* default 2/3 */
  uint64_t max_aggregate_size; /* default 3 */
  uint64_t max_levels;         /* default 25 */
} gnw_amg_options;

/* A CSR matrix view (SparseMatrix, sparse.hpp:14-25, with int64 indices). */
typedef struct gnw_csr {
  uint64_t n_rows;
  uint64_t n_cols;
  const int64_t* rowptr; /* n_rows + 1, rowptr[0] = 0 */
  const int64_t* cols;
  const double* vals;
} gnw_csr;

/* Raw triangulation, the inputs of finalize_mesh (mesh.hpp:53-55). */
typedef struct gnw_mesh {
  uint64_t n_vertices;
  const double* vertices; /* 2 * n_vertices, (x, z) */
  uint64_t n_cells;
  const int64_t* cells;   /* 3 * n_cells vertex ids */
} gnw_mesh;

/* WoodburyBuildTimings, inversion.hpp:41-45 (seconds, CUDA-event timed). */
typedef struct gnw_timings {
  double t_H;
  double t_C;
  double t_chol;
} gnw_timings;

/* MinresReport, minres.hpp:13-22.  The histories are written to caller arrays
 * (capacity hist_cap); n_hist is the full length (iterations + 1). */
typedef struct gnw_report {
  uint64_t iterations;
  int32_t converged;
  double true_relative_residual;
  uint64_t n_hist;
  double* relative_residuals;       /* may be NULL */
  double* pnorm_relative_residuals; /* may be NULL */
  uint64_t hist_cap;
} gnw_report;

/* Sizes of an assembled context (gnw_get_info). */
typedef struct gnw_info {
  uint64_t K;            /* flux dofs = edges */
  uint64_t N;            /* cell dofs */
  uint64_t n_vertices;
  uint64_t n_edges;
  uint64_t n_boundary_edges;
  uint64_t n_levels;
  uint64_t coarse_n;
  uint64_t m;            /* rows of J (0: Laplace-only) */
  double beta;
  uint64_t device_bytes; /* device memory held by the context */
  int64_t collapse_level; /* first V-cycle level replaced by its dense collapsed map (-1: none) */
} gnw_info;

const char* gnw_last_error(void);
const char* gnw_version(void);

gnw_status gnw_create(int n_devices, const int* devices, gnw_ctx** out);
void gnw_destroy(gnw_ctx* ctx);
gnw_status gnw_set_pointer_mode(gnw_ctx* ctx, int mode);
gnw_status gnw_set_coarse_mode(gnw_ctx* ctx, int mode);
gnw_status gnw_set_preconditioner(gnw_ctx* ctx, int kind);
/* MINRES loop schedule.  GNW_LOOP_REFERENCE evaluates A zhat exactly as
 * SaddleOperator::apply does (J zhat2, then J^T u: two sweeps over J).
 * GNW_LOOP_FUSED uses the Woodbury identity J P22^-1 v2 = C^-1 H^T v2 = t':
 * the preconditioner's sweep over H also forms q = J^T t', and the next operator
 * takes J^T u = q / gamma, so J is swept once per iteration instead of twice.
 * Same operator in exact arithmetic; rounding differs.  If a true-residual
 * check (minres.cpp:108-120) fails in fused mode, the solve restarts from the current
 * x on the reference schedule (gnw_stats.loop_restarts counts these).  Partitioned
 * contexts and the Laplace-only preconditioner always run the reference schedule.
 * GNW_LOOP_LEAN goes one step further: since H = B J^T and the V-cycle B is linear,
 * z2 = B v2 - H t' / beta = B (v2 - J^T t' / beta); the preconditioner forms q = J^T t' by
 * one sweep over J and runs its one V-cycle on v2 - q / beta, so H is swept once per
 * iteration (H^T v2) and J once (q): two dense sweeps instead of four, with the V-cycle
 * after the sweeps instead of beside them.
 * Both keep C t' = t backward stable with one refinement step on the explicit C^-1.
 * GNW_LOOP_AUTO (default): for solves with tol >= 1e-8, lean when a sweep over J moves more
 * bytes than two V-cycles (else fused); the reference schedule below 1e-8. */
enum { GNW_LOOP_REFERENCE = 0, GNW_LOOP_FUSED = 1, GNW_LOOP_AUTO = 2, GNW_LOOP_LEAN = 3, GNW_LOOP_PERSISTENT = 4 };
/* GNW_LOOP_PERSISTENT: the lean schedule's arithmetic with the whole loop in ONE persistent
 * cooperative kernel (grid barriers instead of kernel boundaries), for problems whose working
 * set is L2-resident (BASELINE C1).  Falls back to GNW_LOOP_LEAN when the problem is not
 * eligible (m > 64, working set above ~96 MB, exact coarse mode, partitioned).  GNW_LOOP_AUTO
 * picks it by itself for eligible problems at tol >= 1e-8 (env GNW_PERSISTENT=0: never). */
gnw_status gnw_set_loop_mode(gnw_ctx* ctx, int mode);

gnw_status gnw_assemble(gnw_ctx* ctx, const gnw_mesh* mesh, const gnw_amg_options* opts);
/* AMG hierarchy alone over an SPD CSR matrix (amg_setup(s_hat, opts)); after
 * this only gnw_amg_apply is valid. */
gnw_status gnw_assemble_amg_csr(gnw_ctx* ctx, uint64_t n, const int64_t* rowptr,
                                const int64_t* cols, const double* vals,
                                const gnw_amg_options* opts);
/* The mixed problem from the caller's assembled Q (K x K) and D (N x K) -- the operands of
 * SaddleOperator{&Q, &D, &J, beta} (inversion.hpp:18-26) -- instead of a mesh; with opts, also
 * amg_setup(assemble_lumped_schur(Q, D), *opts) (inversion.cpp:196-213); opts = NULL builds no
 * hierarchy (gnw_set_amg_hierarchy supplies the caller's). */
gnw_status gnw_assemble_saddle_csr(gnw_ctx* ctx, const gnw_csr* Q, const gnw_csr* D, const gnw_amg_options* opts);
/* The caller's AmgHierarchy (amg.hpp:25-42): per level A and P (P of the coarsest level is
 * empty) and 1/diag(A); the coarsest dense Cholesky factor (nc x nc, row-major).  The Jacobian
 * must be set again afterwards. */
gnw_status gnw_set_amg_hierarchy(gnw_ctx* ctx, uint64_t n_levels, const gnw_csr* A, const gnw_csr* P,
                                 const double* const* inv_diag, const double* coarse_chol, uint64_t nc,
                                 const gnw_amg_options* opts);
/* The flux block diag(Q)^-1 of the preconditioner (WoodburyPreconditioner::q_diag_inv,
 * inversion.hpp:31) given by the caller: K values, host memory. */
gnw_status gnw_set_flux_scaling(gnw_ctx* ctx, const double* q_diag_inv);
gnw_status gnw_get_info(const gnw_ctx* ctx, gnw_info* info);

gnw_status gnw_set_jacobian(gnw_ctx* ctx, const double* J, uint64_t m, uint64_t n_cells,
                            double beta, gnw_timings* timings);
/* Pipelining aid for consecutive GN steps (no reference analogue: the reference
 * holds J in host memory).  Host-pointer mode only.  Starts the host->device copy
 * of the NEXT step's J (m x n_cells row-major, ideally pinned) on a copy stream, so
 * it overlaps the current solve; the next gnw_set_jacobian with the same pointer and
 * shape takes the staged bytes instead of copying.  J must stay unchanged until then. */
gnw_status gnw_prefetch_jacobian(gnw_ctx* ctx, const double* J, uint64_t m, uint64_t n_cells);

gnw_status gnw_apply_operator(gnw_ctx* ctx, const double* x, double* y);
gnw_status gnw_precondition(gnw_ctx* ctx, const double* y, double* z);
gnw_status gnw_amg_apply(gnw_ctx* ctx, const double* r, double* z);
/* H columns S_hat^-1 J^T on device, exported N x m row-major like h_hat. */
gnw_status gnw_get_woodbury(gnw_ctx* ctx, double* H, double* L);
gnw_status gnw_assemble_rhs(gnw_ctx* ctx, const double* m, const double* m_ref,
                            const double* g, const double* g_obs, double* rhs);
gnw_status gnw_minres_solve(gnw_ctx* ctx, const double* b, const double* x0, double* x,
                            double tol, uint64_t maxit, gnw_report* report);
/* The reference's GN-step solve in one call (gauss_newton, inversion.cpp:259-265):
 *   b = assemble_gn_rhs(m, m_ref, g, g_obs, J, D, beta); x0 = 0; minres(op, pc, b, x0, tol, maxit).
 * Same results as gnw_assemble_rhs + gnw_minres_solve with a zero x0, bit for bit; the
 * right-hand side stays on the device and the zero start is not transferred.  x: K + N.
 * gnw_minres_solve itself accepts x0 == NULL for the zero start.  Single-GPU contexts. */
gnw_status gnw_gn_step_solve(gnw_ctx* ctx, const double* m, const double* m_ref, const double* g,
                             const double* g_obs, double* x, double tol, uint64_t maxit,
                             gnw_report* report);
/* The full residual histories of the last gnw_minres_solve (MinresReport::relative_residuals
 * and ::pnorm_relative_residuals, minres.hpp:15-16), for callers whose report capacity was
 * smaller than n_hist: copies min(cap, n_hist) entries; *n_hist = the full length. */
gnw_status gnw_minres_history(const gnw_ctx* ctx, double* relative_residuals,
                              double* pnorm_relative_residuals, uint64_t cap, uint64_t* n_hist);

/* Structure export for bit-exact parity checks (host arrays).  which: 0=Q 1=D
 * 2=S_hat 3=A_level 4=P_level; NULL arrays query sizes only. */
gnw_status gnw_export_csr(const gnw_ctx* ctx, int which, uint64_t level, uint64_t* n_rows,
                          uint64_t* n_cols, uint64_t* nnz, int64_t* rowptr, int64_t* cols,
                          double* vals);
gnw_status gnw_export_mesh(const gnw_ctx* ctx, int64_t* cells, int64_t* edges,
                           int64_t* cell_edges, int32_t* cell_edge_signs,
                           int64_t* boundary_edges, int32_t* boundary_tags);

/* dense_cholesky on device (linalg.cpp:88-105), operation order preserved. */
gnw_status gnw_dense_cholesky(gnw_ctx* ctx, uint64_t n, const double* C, double* L);

/* ---------------------------------------------------------------- ERT (C4/C5)
 * ElectrodeConfig (survey.hpp:15-21): current electrodes a, b (b = -1: pole at
 * infinity), receiver dipole m, n, geometric factor k.  Electrode indices refer
 * to the node list given to gnw_set_electrodes (Mesh::electrode_nodes). */
typedef struct gnw_ert_config {
  int64_t a, b, m, n;
  double k;
} gnw_ert_config;

typedef struct gnw_ert_stats {
  double t_assemble;  /* host: P1 stiffness values (assemble_forward, forward.cpp:58-80) */
  double t_amg;       /* preconditioner setup: device geometric MG (structured unit-square
                         meshes) or host amg_setup of the stiffness + upload */
  double t_solve;     /* device: batched PCG unit-pole solves (solve_unit_pole, forward.cpp:83-98) */
  double t_jacobian;  /* device: gradients, J rows and g (forward.cpp:122-167) */
  uint64_t pcg_iterations;
  uint64_t gmg_levels;  /* 0: SA-AMG preconditioner, else geometric MG levels */
} gnw_ert_stats;

/* Mesh::electrode_nodes for the assembled mesh; nodes must lie on z = 0. */
gnw_status gnw_set_electrodes(gnw_ctx* ctx, const int64_t* nodes, uint64_t n);
/* evaluate_response_and_jacobian (forward.hpp:40-42, forward.cpp:100-172): g (n_cfg)
 * and J (n_cfg x N row-major) at log-conductivity m (N).  `tol` is the relative
 * residual of the batched PCG pole solves (the reference factorises exactly). */
gnw_status gnw_response_jacobian(gnw_ctx* ctx, const double* m, const gnw_ert_config* cfgs, uint64_t n_cfg,
                                 double* J, double* g, double tol, gnw_ert_stats* stats);
/* gauss_newton (inversion.hpp:66-105, inversion.cpp:187-292) for the iterative algorithms:
 * each outer step evaluates g and J at m (gnw_response_jacobian; the electrodes come from
 * gnw_set_electrodes), builds the Woodbury (or Laplace) preconditioner, assembles the rhs
 * and solves with MINRES from x0 = 0, then m += x[K:].  GnAlgorithm::kDirect (sparse LU)
 * is out of scope. */
typedef struct gnw_gn_config {
  double beta;                  /* GnConfig::beta (> 0) */
  uint64_t max_outer_steps;     /* GnConfig::max_outer_steps */
  double minres_tol;            /* GnConfig::minres_tol */
  uint64_t minres_maxit;        /* 0 -> 2 (K + N) */
  int32_t algorithm;            /* GNW_PC_WOODBURY (kWoodburyMinres) or GNW_PC_LAPLACE (kLaplaceMinres) */
  double misfit_reduction_tol;  /* 0 disables the early exit */
  double forward_tol;           /* pole-solve PCG tolerance (0 -> 1e-14) */
} gnw_gn_config;

typedef struct gnw_gn_step {    /* GnStepReport (inversion.hpp:77-87) */
  double misfit;
  uint64_t minres_iters;
  int32_t converged;
  double euclid_relative_residual;
  double pnorm_relative_residual;
  double t_H, t_C, t_chol, t_norm;
  double t_forward;             /* evaluate_response_and_jacobian of the step (not in t_norm) */
} gnw_gn_step;

gnw_status gnw_gauss_newton(gnw_ctx* ctx, const double* m0, const double* m_ref, const gnw_ert_config* cfgs,
                            uint64_t n_cfg, const double* g_obs, const gnw_gn_config* config, double* m_out,
                            gnw_gn_step* steps, uint64_t steps_cap, uint64_t* n_steps, double* final_misfit);

/* geometric_factor (survey.hpp:33-37, survey.cpp:22-46); b == NULL: pole at infinity. */
gnw_status gnw_geometric_factor(const double a[3], const double* b, const double m[3], const double n[3], int dim,
                                double* k);

/* Device time of the last gnw_minres_solve / set_jacobian, and launch counts. */
typedef struct gnw_stats {
  double t_minres;        /* seconds, CUDA events around the MINRES loop */
  double t_rhs;
  uint64_t kernel_launches; /* kernels launched by the last solve (graph nodes x iterations) */
  uint64_t setup_kernel_launches;
  uint64_t loop_restarts;   /* fused-loop solves restarted on the reference schedule (lifetime) */
  uint64_t fused_iterations; /* of the last solve's iterations, run on the fused or lean schedule */
  uint64_t lean_iterations;  /* of those, on the lean schedule */
  uint64_t persistent_iterations; /* of those, inside the persistent kernel (GNW_LOOP_PERSISTENT) */
  uint64_t comm_calls;       /* partitioned: exchanges this rank issued in the last solve */
  double comm_bytes;         /* partitioned: bytes this rank sent in them */
} gnw_stats;
gnw_status gnw_get_stats(const gnw_ctx* ctx, gnw_stats* stats);

/* CUDA events on the context's stream (slots 0..15) for device-side timing. */
gnw_status gnw_event_record(gnw_ctx* ctx, int slot);
gnw_status gnw_event_elapsed(gnw_ctx* ctx, int slot_begin, int slot_end, double* seconds);

/* Kernel-level measurement for the roofline: launches one hot-path kernel in
 * isolation `reps` times on the context's stream (after one warm-up launch) and
 * returns its mean CUDA-event duration and its ALGORITHMIC traffic per launch
 * (bytes; flops for GNW_K_DGEMM), counted as SURVEY.md 8(d) does: every matrix
 * streamed once, FP64 values 8 B, int32 indices 4 B. */
enum {
  GNW_K_ROW_GEMV = 0,      /* u = J x2 (row GEMV over J) */
  GNW_K_SADDLE = 1,        /* saddle operator incl. J^T u */
  GNW_K_COMBINE_PREC = 2,  /* v-combine + qinv + H^T v2 */
  GNW_K_FINISH_PREC = 3,   /* z2 = s - H t / beta + dots + Givens */
  GNW_K_VCYCLE = 4,        /* one single-RHS V-cycle (all its kernels) */
  GNW_K_UPDATE = 5,        /* w/u/x/r recurrences */
  GNW_K_DGEMM = 6,         /* capacitance DGEMM (DMMA), flops */
  GNW_K_ITERATION = 7,     /* one full MINRES iteration of the last solve (t_minres / iterations; bytes of
                              the schedule it ran: GNW_LOOP_FUSED iterations skip one sweep over J) */
  GNW_K_BODY = 8,          /* the loop body captured once and replayed without loop control;
                              env GNW_EXP_SKIP (bit mask) leaves parts out, for attribution only */
  GNW_K_SADDLE_FUSED = 9,  /* saddle operator taking J^T u = q from the preconditioner sweep (fused) */
  GNW_K_FINISH_FUSED = 10, /* finish_prec that also forms q = J^T t' (fused: sweeps H and J) */
  GNW_K_COL_SWEEP = 11,    /* q = J^T t' and y' = v2 - q / beta (lean schedule) */
  GNW_K_FINISH_LEAN = 12   /* finish_prec with z2 = the V-cycle's output (lean: elementwise, no sweep) */
};
gnw_status gnw_profile_kernel(gnw_ctx* ctx, int kernel, int reps, double* seconds_per_launch,
                              double* algorithmic_per_launch);

/* ---------------------------------------------------------------------------
 * Cell-partitioned multi-GPU solve (C3/C5).  One rank per GPU.
 * Every rank assembles the same mesh and holds all sparse operators, the AMG
 * hierarchy and the MINRES vectors; J and H are split by cell columns, rank r
 * owning cells [c_lo, c_hi) (gnw_get_partition, known after gnw_assemble).
 * gnw_set_jacobian then takes the m x (c_hi - c_lo) column slice J[:, c_lo:c_hi]
 * (row stride c_hi - c_lo); all other vectors are full length and identical on
 * every rank.  gnw_assemble, gnw_set_jacobian, gnw_assemble_rhs,
 * gnw_apply_operator, gnw_precondition and gnw_minres_solve are collective: every
 * rank calls them in the same order.  Results are bitwise identical on all ranks.
 * The reference has no multi-GPU path; its single-process calls are the P = 1 case.
 * ------------------------------------------------------------------------- */
/* 128-byte NCCL unique id: created on one rank, broadcast by the caller. */
gnw_status gnw_nccl_unique_id(unsigned char id[128]);
/* One rank of a P-GPU group over NCCL (NVLink / NVSwitch), this process's device. */
gnw_status gnw_create_partitioned(int device, int rank, int world, const unsigned char id[128], gnw_ctx** out);
/* `world` ranks in THIS process on one device (out[0..world)), each driven by its
 * own host thread; exchanges are host barriers plus device copies.  Same results as
 * `world` GPUs over NCCL; used to test the partitioned path on one GPU. */
gnw_status gnw_create_local_group(int device, int world, gnw_ctx** out);
gnw_status gnw_get_partition(const gnw_ctx* ctx, int* rank, int* world, int64_t* c_lo, int64_t* c_hi);
/* The partition rule (host only): lo[0..world], rank r owns cells [lo[r], lo[r+1]);
 * boundaries are multiples of 64 cells. */
gnw_status gnw_partition_cells(uint64_t n_cells, int world, int64_t* lo);
/* The row partition of the saddle system [[Q, D^T], [D, 0]] (host/partition.hpp) as rank `rank`
 * of `world` would hold it, computed on the host from an assembled context (no GPU needed):
 * sizes = {own edges, own cells, ghosts, send entries}; local_to_global (own + ghosts; edge e
 * -> e, cell c -> K + c), recv_off / send_off (world + 1), send_idx.  NULL arrays: sizes only. */
gnw_status gnw_partition_saddle(const gnw_ctx* ctx, int world, int rank, uint64_t sizes[4],
                                int64_t* local_to_global, int64_t* recv_off, int64_t* send_off,
                                int32_t* send_idx);
/* That rank's local operators: which 0 = Q, 1 = D, 2 = D^T (cell columns stored minus the own
 * edge count, as the kernels address them).  NULL arrays: sizes only. */
gnw_status gnw_partition_csr(const gnw_ctx* ctx, int world, int rank, int which, uint64_t* n_rows,
                             uint64_t* nnz, int64_t* rowptr, int32_t* cols, double* vals);

#ifdef __cplusplus
}
#endif

#endif /* GNW_H */
