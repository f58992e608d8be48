// ertinv_gnw.cpp -- the drop-in: the reference's SaddleOperator::apply,
// WoodburyPreconditioner::apply and build_woodbury_preconditioner (proj/src/inversion.cpp:47-124,
// declared in proj/include/ertinv/inversion.hpp:18-50) on the B200 through libgnw's C-ABI
// (include/gnw.h), plus a device-loop minres overload (include/ertinv_gnw.hpp).
//
// Compiled inside an ertinv tree (the reference's headers on the include path) in place of
// those three definitions of inversion.cpp (tests/cpp/dropin/Makefile
// links the reference's unchanged test_inversion.cpp against it).  The structs keep the
// reference's layout, so the device state is cached per object identity:
//   * SaddleOperator: a context per (Q, D) holding the saddle structure and the operator's J;
//   * WoodburyPreconditioner: a context per built preconditioner (keyed by its factor
//     storage, which moves with the struct) holding the caller's AmgHierarchy, q_diag_inv and
//     H, C on the device; a hand-assembled preconditioner (fields assigned, J = nullptr: the
//     Laplace preconditioner of inversion.cpp:251-256) gets one per (amg, q_diag_inv).
// Exceptions keep the reference's types and texts (gnw_last_error carries them).
#include <algorithm>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "ertinv_gnw.hpp"
#include "gnw.h"

namespace ertinv {
namespace {

std::recursive_mutex g_mu;

void check(gnw_status s) {
  if (s == GNW_OK) return;
  const std::string m = gnw_last_error();
  if (s == GNW_INVALID_ARGUMENT) throw std::invalid_argument(m);
  throw std::runtime_error(m);
}

// Object identity is not enough to key a cached context: a destroyed object's address (and
// its buffers') can be reused by a new one.  A fingerprint adds the shapes, the buffer
// addresses and 16 sampled values.
struct Fp {
  std::size_t a = 0, b = 0, c = 0;
  const void* p = nullptr;
  double v[16] = {};
  bool operator==(const Fp& o) const {
    if (a != o.a || b != o.b || c != o.c || p != o.p) return false;
    for (int k = 0; k < 16; ++k)
      if (!(v[k] == o.v[k]) && !(v[k] != v[k] && o.v[k] != o.v[k])) return false;
    return true;
  }
};
Fp sample(Fp f, const double* x, std::size_t n) {
  f.p = x;
  for (int k = 0; k < 16 && n; ++k) f.v[k] = x[(n - 1) * static_cast<std::size_t>(k) / 15];
  return f;
}
Fp fp(const SparseMatrix& A) { return sample(Fp{A.n_rows, A.n_cols, A.nnz()}, A.values.data(), A.nnz()); }
Fp fp(const Vector& x) { return sample(Fp{x.size(), 0, 0}, x.data(), x.size()); }
Fp fp(const DenseMatrix& M) { return sample(Fp{M.n_rows, M.n_cols, 1}, M.values.data(), M.values.size()); }
Fp fp(const AmgHierarchy& h) {
  Fp f = sample(Fp{h.levels.size(), h.size(), h.levels.empty() ? 0 : h.levels[0].matrix.nnz()},
                h.coarse_cholesky.values.data(), h.coarse_cholesky.values.size());
  return f;
}

// Every drop-in context evaluates in the reference's order (GNW_COARSE_CHOLESKY): the
// V-cycle bit for bit as amg_apply (amg.cpp:90-111), the coarse and capacitance solves as
// cholesky_solve_in_place.  The Woodbury correction subtracts two nearly equal vectors when
// J S^-1 J^T / beta is large (ERT sensitivities), so a caller's own tolerances -- tuned on the
// reference -- are kept only if the rounding follows the reference's as closely as possible.
struct Ctx {
  gnw_ctx* h = nullptr;
  Ctx() {
    int dev = 0;
    check(gnw_create(1, &dev, &h));
    check(gnw_set_coarse_mode(h, GNW_COARSE_CHOLESKY));
  }
  ~Ctx() {
    if (h) gnw_destroy(h);
  }
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
};

static_assert(sizeof(std::size_t) == sizeof(int64_t), "SparseMatrix indices are viewed as int64");
gnw_csr view(const SparseMatrix& A) {
  return gnw_csr{A.n_rows, A.n_cols, reinterpret_cast<const int64_t*>(A.row_offsets.data()),
                 reinterpret_cast<const int64_t*>(A.column_indices.data()), A.values.data()};
}

gnw_amg_options options_of(const AmgOptions& o) {
  return gnw_amg_options{o.coarse_threshold, o.strength, o.jacobi_damping, o.prolongation_damping,
                         o.max_aggregate_size, o.max_levels};
}

void upload_hierarchy(gnw_ctx* c, const AmgHierarchy& amg) {
  const std::size_t L = amg.levels.size();
  std::vector<gnw_csr> A(L), P(L);
  std::vector<const double*> inv(L);
  for (std::size_t l = 0; l < L; ++l) {
    A[l] = view(amg.levels[l].matrix);
    P[l] = view(amg.levels[l].prolongation);
    inv[l] = amg.levels[l].inv_diag.data();
  }
  const gnw_amg_options o = options_of(amg.options);
  check(gnw_set_amg_hierarchy(c, L, A.data(), P.data(), inv.data(), amg.coarse_cholesky.values.data(),
                              amg.coarse_cholesky.n_rows, &o));
}

// A context that only preconditions: the caller's hierarchy and q_diag_inv; the saddle
// structure it is assembled with (Q = I, D = 0) is never applied.
std::unique_ptr<Ctx> pc_context(const AmgHierarchy& amg, const Vector& qinv) {
  auto c = std::make_unique<Ctx>();
  const std::size_t K = qinv.size(), N = amg.size();
  std::vector<int64_t> qrp(K + 1), qci(K), drp(N + 1, 0);
  std::vector<double> qv(K, 1.0);
  for (std::size_t i = 0; i <= K; ++i) qrp[i] = static_cast<int64_t>(i);
  for (std::size_t i = 0; i < K; ++i) qci[i] = static_cast<int64_t>(i);
  const gnw_csr Q{K, K, qrp.data(), qci.data(), qv.data()};
  const gnw_csr D{N, K, drp.data(), nullptr, nullptr};
  check(gnw_assemble_saddle_csr(c->h, &Q, &D, nullptr));
  upload_hierarchy(c->h, amg);
  check(gnw_set_flux_scaling(c->h, qinv.data()));
  return c;
}

// The Jacobian a context holds: (object, storage, rows, beta, preconditioner kind)
struct JKey {
  const DenseMatrix* J = nullptr;
  const double* data = nullptr;
  std::size_t m = SIZE_MAX;
  double beta = 0.0;
  int pc = -1;
  Fp f;
  bool operator==(const JKey& o) const {
    return J == o.J && data == o.data && m == o.m && beta == o.beta && pc == o.pc && f == o.f;
  }
};
void set_j(gnw_ctx* c, JKey& have, const DenseMatrix* J, double beta, int pc, std::size_t N) {
  JKey want{J, J ? J->values.data() : nullptr, J ? J->n_rows : 0, beta, pc, J ? fp(*J) : Fp{}};
  if (want == have) return;
  check(gnw_set_preconditioner(c, pc));
  check(gnw_set_jacobian(c, want.m ? J->values.data() : nullptr, want.m, N, beta, nullptr));
  have = want;
}

struct OpEntry {
  const SparseMatrix *Q, *D;
  Fp fq, fd;
  std::unique_ptr<Ctx> c;
  JKey j;
  bool matches(const SaddleOperator& op) const { return Q == op.Q && D == op.D && fq == fp(*op.Q) && fd == fp(*op.D); }
};
struct PcEntry {
  const AmgHierarchy* amg;
  const Vector* qinv;
  const void* key;  // the preconditioner's factor storage (nullptr: a Laplace preconditioner)
  Fp fa, fq, fk;
  std::unique_ptr<Ctx> c;
  JKey j;
  bool matches(const WoodburyPreconditioner& pc, const void* k) const {
    return amg == pc.amg && qinv == pc.q_diag_inv && key == k && fa == fp(*pc.amg) && fq == fp(*pc.q_diag_inv) &&
           (k == nullptr || fk == fp(pc.capacitance_chol));
  }
};
struct SolveEntry {
  const SparseMatrix *Q, *D;
  const AmgHierarchy* amg;
  const Vector* qinv;
  Fp fq, fd, fa, fv;
  std::unique_ptr<Ctx> c;
  JKey j;
  bool matches(const SaddleOperator& op, const WoodburyPreconditioner& pc) const {
    return Q == op.Q && D == op.D && amg == pc.amg && qinv == pc.q_diag_inv && fq == fp(*op.Q) && fd == fp(*op.D) &&
           fa == fp(*pc.amg) && fv == fp(*pc.q_diag_inv);
  }
};
std::vector<OpEntry> g_ops;
std::vector<PcEntry> g_pcs;
std::vector<SolveEntry> g_solves;
constexpr std::size_t kCache = 8;  // oldest contexts are dropped beyond this many per kind

template <class V>
void trim(V& v) {
  while (v.size() > kCache) v.erase(v.begin());
}

gnw_ctx* operator_context(const SaddleOperator& op) {
  for (auto it = g_ops.rbegin(); it != g_ops.rend(); ++it)  // newest first
    if (it->matches(op)) {
      set_j(it->c->h, it->j, op.J, op.beta, GNW_PC_LAPLACE, op.D->n_rows);
      return it->c->h;
    }
  OpEntry e{op.Q, op.D, fp(*op.Q), fp(*op.D), std::make_unique<Ctx>(), {}};
  const gnw_csr Q = view(*op.Q), D = view(*op.D);
  check(gnw_assemble_saddle_csr(e.c->h, &Q, &D, nullptr));
  set_j(e.c->h, e.j, op.J, op.beta, GNW_PC_LAPLACE, op.D->n_rows);
  g_ops.push_back(std::move(e));
  trim(g_ops);
  return g_ops.back().c->h;
}

gnw_ctx* preconditioner_context(const WoodburyPreconditioner& pc) {
  const bool wood = pc.J != nullptr && pc.J->n_rows > 0;
  const void* key = wood ? static_cast<const void*>(pc.capacitance_chol.values.data()) : nullptr;
  for (auto it = g_pcs.rbegin(); it != g_pcs.rend(); ++it)  // newest first
    if (it->matches(pc, key)) {
      set_j(it->c->h, it->j, wood ? pc.J : nullptr, pc.beta, GNW_PC_WOODBURY, pc.amg->size());
      return it->c->h;
    }
  PcEntry e{pc.amg, pc.q_diag_inv, key, fp(*pc.amg), fp(*pc.q_diag_inv), wood ? fp(pc.capacitance_chol) : Fp{},
            pc_context(*pc.amg, *pc.q_diag_inv), {}};
  set_j(e.c->h, e.j, wood ? pc.J : nullptr, pc.beta, GNW_PC_WOODBURY, pc.amg->size());
  g_pcs.push_back(std::move(e));
  trim(g_pcs);
  return g_pcs.back().c->h;
}

}  // namespace

// inversion.cpp:47-69
Vector SaddleOperator::apply(std::span<const double> x) const {
  const std::size_t K = Q->n_rows, N = D->n_rows;
  if (x.size() != K + N) throw std::invalid_argument("SaddleOperator: dimension mismatch");
  std::lock_guard<std::recursive_mutex> lock(g_mu);
  gnw_ctx* c = operator_context(*this);
  Vector out(K + N, 0.0);
  check(gnw_apply_operator(c, x.data(), out.data()));
  return out;
}

// inversion.cpp:71-89
Vector WoodburyPreconditioner::apply(std::span<const double> y) const {
  const std::size_t K = q_diag_inv->size(), N = amg->size();
  if (y.size() != K + N) throw std::invalid_argument("WoodburyPreconditioner: dimension mismatch");
  std::lock_guard<std::recursive_mutex> lock(g_mu);
  gnw_ctx* c = preconditioner_context(*this);
  Vector out(K + N, 0.0);
  check(gnw_precondition(c, y.data(), out.data()));
  return out;
}

// inversion.cpp:91-124: H = S_hat^-1 J^T by batched V-cycles, C = I + J H / beta by the
// DMMA GEMM and its Cholesky factor, on the device; h_hat and capacitance_chol are exported
// into the returned struct (the reference's fields), the device copies stay cached with it.
WoodburyPreconditioner build_woodbury_preconditioner(const Vector& q_diag_inv, const AmgHierarchy& amg,
                                                     const DenseMatrix& J, double beta,
                                                     WoodburyBuildTimings* timings) {
  if (!(beta > 0.0)) throw std::invalid_argument("build_woodbury_preconditioner: beta <= 0");
  const std::size_t N = amg.size(), M = J.n_rows;
  if (J.n_cols != N) throw std::invalid_argument("build_woodbury_preconditioner: J shape mismatch");
  WoodburyPreconditioner pc;
  pc.q_diag_inv = &q_diag_inv;
  pc.amg = &amg;
  pc.J = &J;
  pc.beta = beta;
  pc.h_hat = DenseMatrix(N, M);
  pc.capacitance_chol = DenseMatrix(M, M);
  if (timings) *timings = WoodburyBuildTimings{};
  if (M == 0) return pc;
  std::lock_guard<std::recursive_mutex> lock(g_mu);
  const void* key = pc.capacitance_chol.values.data();
  g_pcs.erase(std::remove_if(g_pcs.begin(), g_pcs.end(), [&](const PcEntry& x) { return x.key == key; }), g_pcs.end());
  PcEntry e{&amg, &q_diag_inv, key, fp(amg), fp(q_diag_inv), Fp{}, pc_context(amg, q_diag_inv), {}};
  check(gnw_set_preconditioner(e.c->h, GNW_PC_WOODBURY));
  gnw_timings t{};
  check(gnw_set_jacobian(e.c->h, J.values.data(), M, N, beta, &t));
  e.j = JKey{&J, J.values.data(), M, beta, GNW_PC_WOODBURY, fp(J)};
  check(gnw_get_woodbury(e.c->h, pc.h_hat.values.data(), pc.capacitance_chol.values.data()));
  for (std::size_t i = 0; i < M; ++i)  // the lower factor (dense_cholesky leaves the upper part 0)
    for (std::size_t k = i + 1; k < M; ++k) pc.capacitance_chol(i, k) = 0.0;
  if (timings) *timings = WoodburyBuildTimings{t.t_H, t.t_C, t.t_chol};
  e.fk = fp(pc.capacitance_chol);
  g_pcs.push_back(std::move(e));
  trim(g_pcs);
  return pc;
}

// minres(op.apply, pc.apply, b, x0, tol, maxit) (minres.cpp:20-155) with the loop on the device.
std::pair<Vector, MinresReport> minres(const SaddleOperator& op, const WoodburyPreconditioner& pc,
                                       std::span<const double> b, std::span<const double> x0, double tol,
                                       std::size_t maxit) {
  const bool wood = pc.J != nullptr && pc.J->n_rows > 0;
  if ((wood && (op.J != pc.J || op.beta != pc.beta)) || pc.amg->size() != op.D->n_rows ||
      pc.q_diag_inv->size() != op.Q->n_rows) {  // not one GN-step system: the host loop
    return minres([&op](std::span<const double> v) { return op.apply(v); },
                  [&pc](std::span<const double> v) { return pc.apply(v); }, b, x0, tol, maxit);
  }
  const std::size_t n = op.size();
  if (b.size() != n || x0.size() != n) throw std::invalid_argument("minres: dimension mismatch");
  std::lock_guard<std::recursive_mutex> lock(g_mu);
  SolveEntry* s = nullptr;
  for (auto it = g_solves.rbegin(); it != g_solves.rend() && !s; ++it)
    if (it->matches(op, pc)) s = &*it;
  if (!s) {
    SolveEntry e{op.Q, op.D, pc.amg, pc.q_diag_inv, fp(*op.Q), fp(*op.D), fp(*pc.amg), fp(*pc.q_diag_inv),
                 std::make_unique<Ctx>(), {}};
    const gnw_csr Q = view(*op.Q), D = view(*op.D);
    check(gnw_assemble_saddle_csr(e.c->h, &Q, &D, nullptr));
    upload_hierarchy(e.c->h, *pc.amg);
    check(gnw_set_flux_scaling(e.c->h, pc.q_diag_inv->data()));
    g_solves.push_back(std::move(e));
    trim(g_solves);
    s = &g_solves.back();
  }
  if (wood)
    set_j(s->c->h, s->j, pc.J, pc.beta, GNW_PC_WOODBURY, op.D->n_rows);
  else
    set_j(s->c->h, s->j, op.J, op.beta, GNW_PC_LAPLACE, op.D->n_rows);
  Vector x(n, 0.0);
  std::vector<double> he(std::min<std::size_t>(maxit, 4095) + 1), hp(he.size());
  gnw_report r{};
  r.relative_residuals = he.data();
  r.pnorm_relative_residuals = hp.data();
  r.hist_cap = he.size();
  check(gnw_minres_solve(s->c->h, b.data(), x0.data(), x.data(), tol, maxit, &r));
  if (r.n_hist > he.size()) {
    he.resize(r.n_hist);
    hp.resize(r.n_hist);
    check(gnw_minres_history(s->c->h, he.data(), hp.data(), he.size(), nullptr));
  }
  MinresReport rep;
  rep.iterations = r.iterations;
  rep.converged = r.converged != 0;
  rep.true_relative_residual = r.true_relative_residual;
  rep.relative_residuals.assign(he.begin(), he.begin() + static_cast<std::ptrdiff_t>(r.n_hist));
  rep.pnorm_relative_residuals.assign(hp.begin(), hp.begin() + static_cast<std::ptrdiff_t>(r.n_hist));
  return {std::move(x), std::move(rep)};
}

void gnw_release_contexts() {
  std::lock_guard<std::recursive_mutex> lock(g_mu);
  g_ops.clear();
  g_pcs.clear();
  g_solves.clear();
}

}  // namespace ertinv
