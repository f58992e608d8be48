// factorization_standin.cpp -- TEST INFRASTRUCTURE.  Eigen3 (the reference's
// SparseLU backend, proj/CMakeLists.txt:11, proj/src/factorization.cpp:5-6) is
// absent from this image, so the reference's `Factorization` class
// (proj/include/ertinv/factorization.hpp:12-30) is provided here by a banded
// LU without pivoting.  It is exact for the SPD P1 stiffness of the ERT forward
// path (vertices j-major => half-bandwidth ~ n+2) and is NOT used on the
// Woodbury-MINRES path at all.  Linked only into oracle/_ref/libertinv_ref.so.
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "ertinv/factorization.hpp"

namespace ertinv {

struct Factorization::Impl {
  std::size_t n = 0, bw = 0;       // half bandwidth
  std::vector<double> band;        // row i holds columns [i-bw, i+bw]
  double& at(std::size_t i, std::size_t j) { return band[i * (2 * bw + 1) + (j + bw - i)]; }
  double at(std::size_t i, std::size_t j) const { return band[i * (2 * bw + 1) + (j + bw - i)]; }
};

Factorization::Factorization(const SparseMatrix& A) : impl_(std::make_unique<Impl>()) {
  if (A.n_rows != A.n_cols) throw std::invalid_argument("sparse_factorize: matrix not square");
  n_ = A.n_rows;
  Impl& f = *impl_;
  f.n = n_;
  std::size_t bw = 0;
  for (std::size_t i = 0; i < n_; ++i)
    for (std::size_t k = A.row_offsets[i]; k < A.row_offsets[i + 1]; ++k) {
      const std::size_t j = A.column_indices[k];
      bw = std::max(bw, j > i ? j - i : i - j);
    }
  f.bw = bw;
  f.band.assign(n_ * (2 * bw + 1), 0.0);
  for (std::size_t i = 0; i < n_; ++i)
    for (std::size_t k = A.row_offsets[i]; k < A.row_offsets[i + 1]; ++k)
      f.at(i, A.column_indices[k]) += A.values[k];
  // Doolittle LU restricted to the band (no pivoting; SPD inputs only).
  for (std::size_t k = 0; k < n_; ++k) {
    const double piv = f.at(k, k);
    if (!(std::abs(piv) > 0.0)) throw std::runtime_error("sparse_factorize: numerically singular pivot");
    const std::size_t iend = std::min(n_, k + bw + 1);
    for (std::size_t i = k + 1; i < iend; ++i) {
      const double l = f.at(i, k) / piv;
      if (l == 0.0) continue;
      f.at(i, k) = l;
      for (std::size_t j = k + 1; j < iend; ++j) f.at(i, j) -= l * f.at(k, j);
    }
  }
}

Factorization::~Factorization() = default;
Factorization::Factorization(Factorization&&) noexcept = default;
Factorization& Factorization::operator=(Factorization&&) noexcept = default;

Vector Factorization::solve(std::span<const double> b) const {
  if (b.size() != n_) throw std::invalid_argument("Factorization::solve: dimension mismatch");
  const Impl& f = *impl_;
  Vector x(b.begin(), b.end());
  for (std::size_t i = 0; i < n_; ++i) {
    const std::size_t j0 = i > f.bw ? i - f.bw : 0;
    double s = x[i];
    for (std::size_t j = j0; j < i; ++j) s -= f.at(i, j) * x[j];
    x[i] = s;
  }
  for (std::size_t ii = n_; ii-- > 0;) {
    const std::size_t j1 = std::min(n_, ii + f.bw + 1);
    double s = x[ii];
    for (std::size_t j = ii + 1; j < j1; ++j) s -= f.at(ii, j) * x[j];
    x[ii] = s / f.at(ii, ii);
  }
  return x;
}

Factorization sparse_factorize(const SparseMatrix& A) { return Factorization(A); }

}  // namespace ertinv
