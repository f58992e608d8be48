// ert_gmg.cuh -- geometric multigrid preconditioner of the ERT pole solves on the structured
// unit-square mesh (ert_gmg.cu).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "../host/ert.hpp"
#include "amg_device.cuh"

namespace gnw {

class ErtGmg {
 public:
  // n (squares per side) when `mesh` is make_unit_square_mesh(n) with the FAR boundary
  // grounded as assemble_forward numbers it and n can be coarsened at least once; else 0
  static int structured_n(const host::Mesh& mesh, const host::ForwardStructure& fwd);
  // levels n, n/2, ... (to <= 16) for sigma = exp(m) (m on the device), b columns
  void build(int n, const double* m_dev, int b, int* dflag, cudaStream_t s);
  // z = V(2,2)-cycle applied to r (free nodes x b, interleaved)
  void vcycle(const double* r, double* z, cudaStream_t s);
  int levels() const { return static_cast<int>(lv_.size()); }
  size_t bytes() const { return mem_ ? mem_->bytes : 0; }

 private:
  struct Level {
    int n = 0;
    long long nfree = 0;
    double *sigma = nullptr, *st = nullptr;  // cells (2 n^2), 5-point stencil per free node
    double *X = nullptr, *T = nullptr, *R = nullptr, *B = nullptr;  // b columns each
  };
  void cycle(size_t l, const double* B, double* out, cudaStream_t s);
  std::unique_ptr<DeviceMemory> mem_;
  std::vector<Level> lv_;
  int n_ = 0, b_ = 0;
  double *Adense_ = nullptr, *W_ = nullptr, *L_ = nullptr, *Ainv_ = nullptr, *Y_ = nullptr;
};

}  // namespace gnw
