// ert.hpp -- host side of the ERT forward model (C4/C5): survey geometry and the
// P1 stiffness of -div(exp(m) grad u) with the FAR boundary grounded
// (proj/src/forward.cpp:39-98, proj/src/survey.cpp:22-46).
#pragma once

#include <cstdint>
#include <vector>

#include "setup.hpp"

namespace gnw::host {

constexpr int64_t kPoleAtInfinity = -1;  // survey.hpp:10

/// ElectrodeConfig, survey.hpp:15-21: current a (and b, or infinity), receivers m, n.
struct ErtConfig {
  int64_t a = 0, b = kPoleAtInfinity, m = 0, n = 0;
  double k = 0.0;
};

/// geometric_factor, survey.cpp:22-46 (b == nullptr: electrode at infinity).
double geometric_factor(const double a[3], const double* b, const double m[3], const double n[3], int dim);

/// Mesh-only part of assemble_forward (forward.cpp:39-81): grounded nodes, free
/// numbering, the stiffness sparsity and, per stored entry, the cell contributions in
/// the reference's triplet order; plus the cell areas and barycentric gradients
/// (cell_geometry, forward.cpp:17-36).
struct ForwardStructure {
  int64_t n_free = 0;
  std::vector<int64_t> node_to_free;  // -1 on grounded nodes
  std::vector<int64_t> free_to_node;
  Csr pattern;                        // free x free, values unused
  std::vector<int64_t> contrib_start; // per stored entry
  std::vector<int64_t> contrib_cell;
  std::vector<int32_t> contrib_ij;    // 3 * li + lj
  std::vector<double> area;           // per cell
  std::vector<double> grad;           // per cell: grad_i (x, z), i = 0..2 -> 6 values
};

ForwardStructure forward_structure(const Mesh& mesh);
/// Stiffness values sigma = exp(m): entry = sum of sigma_c * area_c * (grad_i . grad_j).
Csr forward_stiffness(const ForwardStructure& f, const double* m);

}  // namespace gnw::host
