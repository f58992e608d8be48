// spectral_stub.cpp -- TEST INFRASTRUCTURE.  proj/src/spectral.cpp needs Eigen (absent from this
// image); the drop-in test binary links these throwing definitions of
// proj/include/ertinv/spectral.hpp instead.  Only the eigenvalue test cases of
// test_inversion.cpp (Pearson inclusion, Murphy-Golub-Wathen spectrum) reach them, and the
// drop-in test excludes those cases (-tce=...).
#include <stdexcept>

#include "ertinv/spectral.hpp"

namespace ertinv {

DenseMatrix dense_saddle_matrix(const SparseMatrix&, const SparseMatrix&, const DenseMatrix&, double) {
  throw std::runtime_error("spectral: Eigen is not available in this build");
}

DenseMatrix dense_ideal_preconditioner(const SparseMatrix&, const SparseMatrix&, const DenseMatrix&, double) {
  throw std::runtime_error("spectral: Eigen is not available in this build");
}

std::vector<double> preconditioned_eigenvalues(const DenseMatrix&, const DenseMatrix&) {
  throw std::runtime_error("spectral: Eigen is not available in this build");
}

}  // namespace ertinv
