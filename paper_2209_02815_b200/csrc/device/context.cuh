// context.cuh -- the device-resident solver context behind the gnw C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../host/ert.hpp"
#include "../host/setup.hpp"
#include "amg_device.cuh"
#include "sparse_device.cuh"
#include "minres_persistent.cuh"
#include "comm.cuh"
#include "ert_gmg.cuh"
#include "ert_kernels.cuh"
#include "kernels.cuh"
#include "part_amg.cuh"

namespace gnw {

struct MinresResult {
  std::vector<double> hist_e, hist_p;
  uint64_t iterations = 0;
  bool converged = false;
  double true_rel = 0.0;
};

// GnConfig / GnStepReport / GnReport (inversion.hpp:66-95)
struct GnConfig {
  double beta = 0.1;
  uint64_t max_outer_steps = 2;
  double minres_tol = 1e-7;
  uint64_t minres_maxit = 0;  // 0 -> 2 (K + N)
  int laplace = 0;            // GnAlgorithm::kLaplaceMinres instead of kWoodburyMinres
  double misfit_reduction_tol = 0.0;
  double forward_tol = 1e-14;  // batched PCG of the pole solves (the reference factorises exactly)
};
struct GnStepReport {
  double misfit = 0.0;
  uint64_t minres_iters = 0;
  bool converged = true;
  double euclid_relative_residual = 0.0, pnorm_relative_residual = 0.0;
  double t_H = 0.0, t_C = 0.0, t_chol = 0.0, t_norm = 0.0;
  double t_forward = 0.0;  // evaluate_response_and_jacobian (outside t_norm, as the reference)
};
struct GnResult {
  std::vector<GnStepReport> steps;
  double final_misfit = 0.0;
};

struct ErtTimings {
  double t_assemble = 0.0, t_amg = 0.0, t_solve = 0.0, t_jacobian = 0.0;
  uint64_t pcg_iterations = 0;
  uint64_t gmg_levels = 0;  // 0: SA-AMG preconditioner (host setup), else geometric MG levels
};

class Context {
 public:
  explicit Context(int device);  // device < 0: host-only context (setup and export only)
  ~Context();

  bool has_device() const { return device_ >= 0; }
  int vc_collapse_level() const { return damg_.collapse_level(); }
  int ptr_mode = 0;
  int coarse_mode = 0;
  int pc_laplace = 0;  // GnAlgorithm::kLaplaceMinres (inversion.cpp:251-256)
  // Woodbury-fused MINRES loop: J^T u from the preconditioner sweep
  // loop modes (gnw.h GNW_LOOP_*): 0 reference, 1 fused, 2 auto, 3 lean.  auto runs
  // auto_sched_ when the solve's tol >= kAutoFusedTol, the reference schedule below.
  static constexpr double kAutoFusedTol = 1e-8;
  int auto_sched_ = 0;  // schedule auto picks: 0 by sweep vs V-cycle bytes, 1 fused, 2 lean (env GNW_AUTO_SCHED)
  double vcycle_bytes() const;
  // mode 4 (GNW_LOOP_PERSISTENT): lean arithmetic inside the persistent kernel when eligible
  void set_fused(int mode) {
    persist_mode_ = mode == 4 ? 2 : (mode == 2 ? 1 : 0);
    fused_ = mode == 4 ? 3 : mode;
  }
  int persist_mode_ = 1;  // 0 never, 1 auto (with GNW_LOOP_AUTO), 2 requested
  bool persistent_eligible() const;
  uint64_t last_persist_iters_ = 0;
  int fused() const { return fused_; }
  uint64_t loop_restarts = 0;  // fused-loop solves restarted on the reference schedule
  void set_coarse(int mode) {
    if (mode != coarse_mode) destroy_graph();  // the loop graph bakes the kernel choice
    coarse_mode = mode;
  }

  void assemble(const double* vertices, int64_t nv, const int64_t* cells, int64_t nc, const host::AmgOptions& o);
  void assemble_amg_csr(int64_t n, const int64_t* rowptr, const int64_t* cols, const double* vals,
                        const host::AmgOptions& o);
  void assemble_saddle_csr(int64_t K, int64_t N, const int64_t* qrp, const int64_t* qci, const double* qv,
                           const int64_t* drp, const int64_t* dci, const double* dv, const host::AmgOptions* o);
  void set_hierarchy(const host::AmgHierarchy& h);
  void set_qinv(const double* q);
  void set_jacobian(const double* J, int64_t m, int64_t n_cells, double beta, double timings[3]);
  // async H2D of the next step's J beside the current solve (host-pointer mode)
  void prefetch_jacobian(const double* J, int64_t m, int64_t n_cells);
  void apply_operator(const double* x, double* y);
  void precondition(const double* y, double* z);
  void amg_apply(const double* r, double* z);
  void assemble_rhs(const double* mdl, const double* mref, const double* g, const double* gobs, double* rhs);
  MinresResult minres(const double* b, const double* x0, double* x, double tol, uint64_t maxit);
  // assemble_gn_rhs + minres from the zero start in one call (inversion.cpp:259-265)
  MinresResult gn_step_solve(const double* mdl, const double* mref, const double* g, const double* gobs, double* x,
                             double tol, uint64_t maxit);
  void get_woodbury(double* H, double* L);
  void dense_cholesky(int64_t n, const double* C, double* L);
  void event_record(int slot);
  double event_elapsed(int a, int b);
  void profile_kernel(int kernel, int reps, double* seconds, double* algorithmic);
  uint64_t last_iterations = 0;
  double *ppart_ = nullptr, *ptpart_ = nullptr;  // persistent kernel: partial sums
  unsigned* pbar_ = nullptr;                     // and its grid-barrier counter
  int ppart_m_ = 0;
  uint64_t last_fused_iters_ = 0;  // of last_iterations, run on the fused or lean schedule
  uint64_t last_sched_iters_[3] = {0, 0, 0};  // of last_iterations, per schedule (reference, fused, lean)

  // Row-partitioned multi-GPU mode (context_rowpart.cu); set before assemble.
  // The rank owns cells [c_lo, c_hi) (whole mesh rows) and the edges first met in them; J and
  // H are its m x (c_hi - c_lo) column slices (set_jacobian takes that slice).  The public
  // entry points still take and return GLOBAL vectors (every rank passes the same input and
  // receives the full result); the solve itself runs on the owned rows with halo exchanges.
  void set_comm(std::shared_ptr<Comm> c);
  bool partitioned() const { return comm_ != nullptr; }
  const Comm* comm() const { return comm_.get(); }
  long long c_lo() const { return c_lo_; }
  long long c_hi() const { return c_hi_; }
  long long own_edges() const { return comm_ ? Kl_ : K_; }
  long long own_cells() const { return comm_ ? Nl_ : N_; }
  long long ghost_entries() const { return comm_ ? nloc_ - Kl_ - Nl_ : 0; }
  int part_levels() const { return pamg_ ? pamg_->partitioned_levels() : 0; }
  unsigned long long comm_calls() const { return comm_calls_; }
  double comm_bytes() const { return comm_bytes_; }

  // ERT forward model (forward.cpp:39-172) on the assembled mesh
  void set_electrodes(const int64_t* nodes, int64_t n);
  void response_jacobian(const double* mdl, const host::ErtConfig* cfgs, int64_t n_cfg, double* J_out, double* g_out,
                         double tol, ErtTimings* t);

  // gauss_newton (inversion.cpp:187-292), iterative algorithms, on the device: forward
  // response + J, Woodbury (or Laplace) preconditioner, rhs, MINRES, model update.
  GnResult gauss_newton(const double* m0, const double* m_ref, const host::ErtConfig* cfgs, int64_t n_cfg,
                        const double* g_obs, const GnConfig& cfg, double* m_out);

  // structure
  const host::Mesh& mesh() const { return mesh_; }
  const host::Csr& Q() const { return Q_; }
  const host::Csr& D() const { return D_; }
  const host::Csr& S() const { return S_; }
  const host::AmgHierarchy& amg() const { return amg_; }
  bool mixed() const { return mixed_; }
  bool assembled() const { return assembled_; }
  int64_t K() const { return K_; }
  int64_t N() const { return N_; }
  int64_t m() const { return m_; }
  double beta() const { return beta_; }
  size_t device_bytes() const {
    return mem_.bytes + (jmem_ ? jmem_->bytes : 0) + (stage_mem_ ? stage_mem_->bytes : 0) + damg_.bytes() + fwd_amg_.bytes() + fwd_gmg_.bytes() + (emem_ ? emem_->bytes : 0);
  }

  double t_minres = 0.0, t_rhs = 0.0;
  uint64_t launches = 0, setup_launches = 0;

 private:
  void require_device() const;
  void require_mixed() const;
  void upload_structure();
  void finish_assembly();
  void upload_hierarchy();
  void vcycle(VSel r0, double* out0, const MinresState* st, cudaStream_t s = nullptr);
  void operator_into(VSel x, int scaled, VSel y, MinresState* st, int loop, bool fused = false);
  // the current solve's loop schedule: 0 reference, 1 fused (3 dense sweeps), 2 lean (2 sweeps)
  int loop_sched() const;
  void precondition_into(VSel y, VSel yv2, VSel z, MinresState* st, int loop, VSel vcur, VSel vprev,
                         int sched = 0);
  bool fused_active() const { return loop_sched() != 0; }
  void build_graph();
  void launch_iteration(unsigned long long cond_handle, int use_cond);
  bool no_graph_ = false;  // env GNW_NO_GRAPH=1: host-driven loop (for ncu; kernels in conditional graphs are not listed)
  void destroy_graph();
  double* stage_in(const double* p, size_t n, double* dev);
  void stage_out(double* host, const double* dev, size_t n);
  void sync();

  int device_ = -1;
  cudaStream_t stream_ = nullptr;
  // The V-cycle runs on a second stream (a parallel graph branch) beside the
  // H^T v row GEMV it does not depend on; env GNW_FORK_VCYCLE=0 serialises it.
  cudaStream_t side_ = nullptr;
  cudaEvent_t fork_ev_[2] = {};
  bool fork_ = true;
  int sm_count_ = 148;
  DeviceMemory mem_;                      // structure + work vectors
  std::unique_ptr<DeviceMemory> jmem_;    // Jacobian-dependent buffers
  DeviceAmg damg_;                        // SA-AMG of S_hat on the device

  bool assembled_ = false, mixed_ = false;
  host::Mesh mesh_;
  host::Csr Q_, D_, S_;
  host::AmgHierarchy amg_;
  std::vector<DevFusedOps> fused_pre_;  // one-pass level operators formed (and kept) on the device by the setup
  bool device_setup_enabled(int64_t n_cells) const;
  int64_t K_ = 0, N_ = 0;

  // device structure
  OperatorArgs op_{};
  PrecArgs pa_{};
  double* svc_ = nullptr;  // V-cycle output (s)

  // Jacobian / Woodbury
  int64_t m_ = 0;
  double beta_ = 1.0;
  double *dJ_ = nullptr, *dHt_ = nullptr, *dC_ = nullptr, *dL_ = nullptr, *dCinv_ = nullptr, *dY_ = nullptr;
  double *u_ = nullptr, *t_ = nullptr, *t2_ = nullptr;
  double *gpart_ = nullptr, *tpart_ = nullptr;
  RowGemv plan_{};    // J x (nothing runs beside it)
  RowGemv plan_h_{};  // H^T y (leaves CTA slots for the forked V-cycle)
  int exp_skip_ = 0;     // profiling only (profile_kernel "body"): bit mask of iteration parts left out
  int rg_reserve_ = 2;  // env GNW_RG_RESERVE; of 4 resident k_row_gemv CTAs per SM (C2 sweep: 0: 0.895, 1: 0.862, 2: 0.847, 3: 0.950 ms/iteration)

  // MINRES vectors
  double *b_ = nullptr, *x_ = nullptr, *r_ = nullptr, *az_ = nullptr, *tmp_ = nullptr, *tmp2_ = nullptr;
  double* V_[3] = {};
  double* W_[3] = {};
  double* U_[3] = {};
  double* Z_[2] = {};
  double* Vk_[3] = {};  // V_[k] + K (cell part), V-cycle input ring
  double *opart_ = nullptr, *cpart_ = nullptr, *fpart_ = nullptr, *upart_ = nullptr, *rpart_ = nullptr;
  unsigned* counters_ = nullptr;  // 16 counters
  MinresState* st_ = nullptr;     // loop state
  MinresState* st_plain_ = nullptr;
  MinresState* h_st_ = nullptr;   // pinned host mirror
  double *hist_e_ = nullptr, *hist_p_ = nullptr;
  long long hist_cap_ = 0;
  double* io_a_ = nullptr;        // device staging for host-pointer mode
  double* io_b_ = nullptr;
  double* io_c_ = nullptr;
  double* io_d_ = nullptr;
  int* dflag_ = nullptr;

  cudaEvent_t events_[16] = {};
  cudaEvent_t jev_[4] = {};    // set_jacobian phase timers
  cudaEvent_t mev_[2] = {};    // minres timers
  cudaEvent_t rhs_ev_[2] = {};  // assemble_rhs timers
  cudaEvent_t tri_ev_[2] = {};  // fork / join of the dot-partials branch (k_sum_triples)
  double* ctot_ = nullptr;      // the combine kernel's dots, pre-summed
  int64_t jm_m_ = -1;          // shape of the persistent Jacobian buffers
  bool jm_owned_ = false;
  double* jown_ = nullptr;     // owned copy of J (host-pointer mode)
  cudaStream_t copy_ = nullptr;            // prefetch_jacobian's host->device stream
  cudaEvent_t stage_ev_[2] = {};           // [0] staged bytes landed, [1] staging buffer consumed
  std::unique_ptr<DeviceMemory> stage_mem_;
  double* jstage_ = nullptr;
  size_t stage_cap_ = 0;
  int64_t stage_key_m_ = -1;               // (m, row stride) the stage buffer was sized for
  long long stage_key_ld_ = -1;
  const double* staged_src_ = nullptr;     // host J of the pending stage (nullptr: none)
  int64_t staged_m_ = -1;
  int64_t staged_rows_ = 0;                // leading rows of J staged (< m when only part fits)
  long long staged_n_ = -1, staged_ld_ = -1;
  bool stage_deferred_ = false;            // requested, not yet issued (issue_stage)
  void issue_stage();
  double* dpart_ = nullptr;    // DGEMM split-K partials
  double* dnib_ = nullptr;     // device scalar -1/beta
  double* dq_ = nullptr;       // q = J^T t' (fused loop), N
  double* bq_ = nullptr;       // y' = v2 - q / beta, the lean loop's V-cycle input, N
  double* cres_ = nullptr;     // m scratch: capacitance refinement residual
  bool cinv_refine_ = true;    // fused/lean: refine t2 = C^-1 t once (env GNW_CINV_REFINE=0 disables)
  long long ldh_ = 0, ldj_ = 0;  // row strides of Ht / J on device
  long long pad_ = 64;           // row padding (doubles) of owned m x N matrices (env GNW_PAD)
  int fused_ = 2;
  bool j_borrowed_ = false;  // device-pointer J referenced, not copied (SaddleOperator holds a pointer)
  // loop graphs per schedule: [0] reference, [1] fused, [2] lean (built on first use)
  cudaGraph_t graph_[3] = {};
  cudaGraphExec_t graph_exec_[3] = {};
  uint64_t graph_nodes_[3] = {};
  bool fused_off_ = false;  // this solve restarted on the reference schedule (minres)
  int n_comb_blocks_ = 0;

  // partitioned mode (context_rowpart.cu)
  std::shared_ptr<Comm> comm_;
  std::vector<long long> part_lo_, part_e_;  // world + 1 cell / edge boundaries
  long long c_lo_ = 0, c_hi_ = 0, e_lo_ = 0, e_hi_ = 0;
  long long Kl_ = 0, Nl_ = 0, nloc_ = 0;     // own edges, own cells, local length with ghosts
  long long host_j_ = 0;                     // iteration index mirrored on the host (ring slots of the exchanges)
  long long kd() const { return comm_ ? Kl_ : K_; }  // edge / cell rows of the device vectors
  long long nd() const { return comm_ ? Nl_ : N_; }
  long long local_n() const { return nd(); }
  double* resolve(const VSel& v) const { return v.mod == 1 ? v.p[0] : v.p[(host_j_ + v.off) % v.mod]; }
  void setup_rowpart();
  void alloc_vectors(long long n_alloc, long long K, long long N);
  void reduce_m(const double* part, double* out, long long n, cudaStream_t s);  // fixed-order allreduce
  void reduce_scratch(MinresState* st, int k0, int cnt);  // st->scratch[k0, k0+cnt) summed over ranks
  void exchange_saddle(double* v);                         // ghost edges and cells of a saddle vector
  void global_to_local(const double* g, double* l, bool ghosts);
  void local_to_global(const double* l, double* g);
  const double* global_in(const double* p, size_t n, double* dev);
  void global_out(double* p, const double* dev, size_t n);
  void build_h_rowpart();
  DeviceMemory rpmem_;
  std::unique_ptr<DHalo> sh_;
  std::unique_ptr<PartAmg> pamg_;
  int *sad_l2g_ = nullptr, *cell_l2g_ = nullptr;
  long long n_cell_l2g_ = 0;
  double *gio_a_ = nullptr, *gio_b_ = nullptr, *gio_c_ = nullptr, *gio_d_ = nullptr, *sgath_ = nullptr;
  double *u_part_ = nullptr, *t_part_ = nullptr, *gath_ = nullptr, *Cpart_ = nullptr, *Cgath_ = nullptr;
  long long gath_cap_ = 0;
  unsigned long long comm_calls_ = 0;  // exchanges and bytes of the last minres (partitioned)
  double comm_bytes_ = 0.0;
  std::unique_ptr<DeviceMemory> hx_mem_;
  double *hx_ = nullptr, *hy_ = nullptr;
  int hx_b_ = 0;

  // ERT forward model state
  std::vector<int64_t> electrodes_;
  host::ForwardStructure fwd_;      // free-node map, stiffness pattern, per-entry contributions
  DeviceAmg fwd_amg_;               // SA-AMG of the P1 stiffness (rebuilt per model)
  ErtGmg fwd_gmg_;                  // geometric MG of the same operator (structured meshes)
  int fwd_gmg_n_ = -1;              // ErtGmg::structured_n of the mesh (-1: not checked yet)
  std::unique_ptr<DeviceMemory> emem_;  // mesh-only forward structure on the device (per mesh)
  DCsr ek_{};                           // stiffness pattern (values re-uploaded per model)
  int64_t *ecells_ = nullptr, *en2f_ = nullptr;
  double *egrad_ = nullptr, *earea_ = nullptr;
  std::unique_ptr<DeviceMemory> ews_;   // response_jacobian work buffers
  struct {
    double *X, *R, *Z, *P, *AP, *sc, *part, *m, *gx, *gz, *gpart, *J, *g;
    int *active, *col;
    int64_t* unit;
    ErtCfgDev* cfg;
  } ew_{};
  int ews_b_ = -1;
  int64_t ews_ncfg_ = -1;
  bool ews_own_ = false;
};

}  // namespace gnw
