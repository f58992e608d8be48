// gn_step_example.cpp -- a reference-style C++ caller of the drop-in (include/gnw.hpp).
// Mirrors proj/tests/test_inversion.cpp:341-382 ("MINRES with Woodbury and Laplace
// preconditioners agree and Woodbury needs fewer iterations") on unit_square(5), M=7,
// beta=0.25, but through the B200 C-ABI.  Exit code 0 on success.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "gnw.hpp"

static void unit_square(std::size_t n, std::vector<double>& v, std::vector<std::int64_t>& c) {
  for (std::size_t j = 0; j <= n; ++j)
    for (std::size_t i = 0; i <= n; ++i) {
      v.push_back(static_cast<double>(i) / static_cast<double>(n));
      v.push_back(static_cast<double>(j) / static_cast<double>(n));
    }
  auto id = [n](std::size_t i, std::size_t j) { return static_cast<std::int64_t>(j * (n + 1) + i); };
  for (std::size_t j = 0; j < n; ++j)
    for (std::size_t i = 0; i < n; ++i) {
      c.insert(c.end(), {id(i, j), id(i + 1, j), id(i + 1, j + 1)});
      c.insert(c.end(), {id(i, j), id(i + 1, j + 1), id(i, j + 1)});
    }
}

int main() {
  std::vector<double> v;
  std::vector<std::int64_t> cells;
  unit_square(5, v, cells);
  gnw::GnStepSolver s(v, cells);
  const std::size_t K = s.n_flux_dofs(), N = s.n_cell_dofs(), M = 7;
  if (K != 85 || N != 50) {
    std::fprintf(stderr, "unexpected sizes K=%zu N=%zu\n", K, N);
    return 1;
  }
  std::mt19937 rng(17);
  std::normal_distribution<double> normal(0.0, 1.0);
  std::vector<double> J(M * N), m(N), m_ref(N, 0.0), g(M), g_obs(M, 0.0);
  for (double& x : J) x = normal(rng);
  for (double& x : m) x = normal(rng);
  for (double& x : g) x = normal(rng);
  const double beta = 0.25;
  const std::vector<double> x0(K + N, 0.0);

  gnw::WoodburyBuildTimings t;
  s.build_woodbury_preconditioner(J.data(), M, beta, &t);
  const std::vector<double> b = s.assemble_gn_rhs(m, m_ref, g, g_obs);
  gnw::MinresReport rw, rl;
  const std::vector<double> xw = s.minres(b, x0, 1e-10, 2 * (K + N), &rw);
  s.laplace_preconditioner(J.data(), M, beta);
  const std::vector<double> xl = s.minres(b, x0, 1e-10, 2 * (K + N), &rl);
  double d = 0.0, nrm = 0.0;
  for (std::size_t i = 0; i < xw.size(); ++i) {
    d += (xw[i] - xl[i]) * (xw[i] - xl[i]);
    nrm += xw[i] * xw[i];
  }
  const double rel = std::sqrt(d / nrm);
  std::printf("woodbury %zu iterations, laplace %zu iterations, rel diff %.3e, t_H %.3e s\n", rw.iterations,
              rl.iterations, rel, t.t_H);
  bool ok = rw.converged && rl.converged && rl.iterations > rw.iterations && rel <= 1e-5;
  // error path keeps the reference's exception type and text
  try {
    s.build_woodbury_preconditioner(J.data(), M, 0.0);
    ok = false;
  } catch (const std::invalid_argument& e) {
    ok = ok && std::string(e.what()).find("beta <= 0") != std::string::npos;
  }
  return ok ? 0 : 1;
}
