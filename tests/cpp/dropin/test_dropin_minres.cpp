// test_dropin_minres.cpp -- TEST INFRASTRUCTURE: the drop-in's device-loop minres overload
// (include/ertinv_gnw.hpp) against the reference's generic host-loop minres over the same
// operator and preconditioner objects (the call gauss_newton makes, inversion.cpp:261-265),
// on the reference's own small instance construction (test_inversion.cpp:341-382).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <algorithm>
#include <cstdio>
#include <random>

#include "ertinv_gnw.hpp"
#include "test_helpers.hpp"

using namespace ertinv;

namespace {
DenseMatrix random_j(std::size_t M, std::size_t N, std::mt19937& rng) {
  std::normal_distribution<double> g(0.0, 1.0);
  DenseMatrix J(M, N);
  for (double& v : J.values) v = g(rng);
  return J;
}
}  // namespace

TEST_CASE("device minres overload reproduces the generic minres on the same objects") {
  const Mesh mesh = test_helpers::make_unit_square_mesh(12);
  const MixedSpaces spaces = make_mixed_spaces(mesh);
  const SparseMatrix Q = assemble_Q(spaces), D = assemble_D(spaces);
  const std::size_t K = spaces.n_flux_dofs, N = D.n_rows;
  Vector q_inv = diagonal(Q);
  for (double& v : q_inv) v = 1.0 / v;
  const AmgHierarchy amg = amg_setup(assemble_lumped_schur(Q, D));
  std::mt19937 rng(7);
  const DenseMatrix J = random_j(9, N, rng);
  const double beta = 1e-2;
  const SaddleOperator op{&Q, &D, &J, beta};
  const WoodburyPreconditioner pc_w = build_woodbury_preconditioner(q_inv, amg, J, beta);
  WoodburyPreconditioner pc_l;  // the Laplace preconditioner, fields assigned (inversion.cpp:251-256)
  pc_l.q_diag_inv = &q_inv;
  pc_l.amg = &amg;
  pc_l.J = nullptr;
  pc_l.beta = beta;
  const Vector b = test_helpers::random_vector(K + N, rng);
  const Vector x0(K + N, 0.0);
  for (const WoodburyPreconditioner* pc : std::vector<const WoodburyPreconditioner*>{&pc_w, &pc_l}) {
    auto [xh, rh] = minres([&op](std::span<const double> v) { return op.apply(v); },
                           [pc](std::span<const double> v) { return pc->apply(v); }, b, x0, 1e-8, 2 * (K + N));
    auto [xd, rd] = minres(op, *pc, b, x0, 1e-8, 2 * (K + N));
    std::printf("host loop %zu iterations, device loop %zu\n", rh.iterations, rd.iterations);
    REQUIRE(rh.converged);
    REQUIRE(rd.converged);
    // the Euclidean stopping residual oscillates near tol on the Laplace-preconditioned run, so
    // the two loops (device reductions vs the host's sequential dots) may stop a few apart
    const std::size_t slack = std::max<std::size_t>(2, rh.iterations / 20);
    CHECK(rd.iterations <= rh.iterations + slack);
    CHECK(rh.iterations <= rd.iterations + slack);
    CHECK(rd.relative_residuals.size() == rd.iterations + 1);
    CHECK(test_helpers::rel_diff(xd, xh) <= 1e-6);
    CHECK(rd.true_relative_residual <= 1e-7);
  }
  // the Woodbury preconditioner needs fewer iterations (the paper's point; test_inversion.cpp:381)
  auto [xw, rw] = minres(op, pc_w, b, x0, 1e-8, 2 * (K + N));
  auto [xl, rl] = minres(op, pc_l, b, x0, 1e-8, 2 * (K + N));
  CHECK(rl.iterations > rw.iterations);
}

TEST_CASE("device minres keeps the reference's errors") {
  const Mesh mesh = test_helpers::make_unit_square_mesh(4);
  const MixedSpaces spaces = make_mixed_spaces(mesh);
  const SparseMatrix Q = assemble_Q(spaces), D = assemble_D(spaces);
  Vector q_inv = diagonal(Q);
  for (double& v : q_inv) v = 1.0 / v;
  const AmgHierarchy amg = amg_setup(assemble_lumped_schur(Q, D));
  const SaddleOperator op{&Q, &D, nullptr, 1.0};
  WoodburyPreconditioner pc;
  pc.q_diag_inv = &q_inv;
  pc.amg = &amg;
  const Vector b(op.size(), 1.0), short_x0(op.size() - 1, 0.0), x0(op.size(), 0.0);
  CHECK_THROWS_AS(minres(op, pc, b, short_x0, 1e-8, 100), std::invalid_argument);
  CHECK_THROWS_AS(minres(op, pc, b, x0, 0.0, 100), std::invalid_argument);
  CHECK_THROWS_AS(op.apply(short_x0), std::invalid_argument);
  CHECK_THROWS_AS(build_woodbury_preconditioner(q_inv, amg, DenseMatrix(2, 3), 1.0), std::invalid_argument);
  CHECK_THROWS_AS(build_woodbury_preconditioner(q_inv, amg, DenseMatrix(2, D.n_rows), 0.0), std::invalid_argument);
}
