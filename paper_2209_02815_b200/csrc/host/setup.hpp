// setup.hpp -- host-side (CPU, once per inversion) setup of the Woodbury-MINRES
// path: mesh connectivity, RT0 x P0 assembly and the smoothed-aggregation AMG
// hierarchy.  These run the reference's algorithms with its exact floating-point
// evaluation order, so every index array and every value is bit-identical to
// the reference (SURVEY.md section 7 "hard part 1": the greedy aggregation is
// sequential and defines the preconditioner).  The independent loops (per-row
// sparse products, per-edge assembly) are OpenMP-parallel; each row is still
// computed in the reference's order, so the results do not depend on threads.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace gnw::host {

/// Compressed rows; columns strictly increasing per row (sparse.hpp:14-25).
struct Csr {
  int64_t n_rows = 0;
  int64_t n_cols = 0;
  std::vector<int64_t> rowptr;  // n_rows + 1
  std::vector<int32_t> cols;
  std::vector<double> vals;
  int64_t nnz() const { return static_cast<int64_t>(vals.size()); }
};

/// finalize_mesh output (mesh.hpp:17-33); boundary tag 0 = SURFACE, 1 = FAR.
struct Mesh {
  int64_t nv = 0, nc = 0, ne = 0;
  std::vector<double> vertices;      // 2 per vertex
  std::vector<int64_t> cells;        // 3 per cell, counterclockwise
  std::vector<int64_t> edges;        // 2 per edge, low -> high
  std::vector<int64_t> cell_edges;   // 3 per cell
  std::vector<int32_t> cell_signs;   // 3 per cell
  std::vector<int64_t> boundary_edges;
  std::vector<int32_t> boundary_tags;
};

struct AmgOptions {  // amg.hpp:11-23
  int64_t coarse_threshold = 64;
  double strength = 0.08;
  double jacobi_damping = 2.0 / 3.0;
  double prolongation_damping = 2.0 / 3.0;
  int64_t max_aggregate_size = 3;
  int64_t max_levels = 25;
};

struct AmgLevel {  // amg.hpp:25-29
  Csr A;
  Csr P;  // empty on the coarsest level
  std::vector<double> inv_diag;
};

struct AmgHierarchy {  // amg.hpp:34-42
  std::vector<AmgLevel> levels;
  std::vector<double> coarse_chol;  // lower factor, nc x nc row-major
  int64_t nc = 0;
  AmgOptions options;
};

Mesh finalize_mesh(const double* vertices, int64_t nv, const int64_t* cells, int64_t nc);
Csr assemble_Q(const Mesh& mesh);
Csr assemble_D(const Mesh& mesh);
Csr transpose(const Csr& A);
Csr spgemm(const Csr& A, const Csr& B);
/// Optional device implementation of spgemm for the calling thread (same result bit for bit;
/// set by a device context around its setup, nullptr = host).  Used for products with at
/// least `min_products` scalar products.
using SpgemmHook = Csr (*)(const Csr& A, const Csr& B, void* user);
void set_spgemm_hook(SpgemmHook fn, void* user, int64_t min_products);
Csr scale_rows(const Csr& A, const std::vector<double>& s);
std::vector<double> diagonal(const Csr& A);
double symmetry_error(const Csr& A);
Csr lumped_schur(const Csr& Q, const Csr& D);
/// Sorted-triplet construction with duplicate summation (sparse.cpp:19-51).
Csr from_triplets(int64_t n_rows, int64_t n_cols, std::vector<int64_t> rows,
                  std::vector<int64_t> cols, std::vector<double> vals);
AmgHierarchy amg_setup(const Csr& S, const AmgOptions& opt, bool check_symmetry = true);
/// The pieces of amg_setup the device-resident setup (device/sparse_device.cuh) shares:
/// the sequential greedy aggregation (amg.cpp:13-68) and 1 / diag(A) (amg.cpp:81-88).
std::vector<int64_t> aggregate(const Csr& A, const AmgOptions& o, int64_t& n_agg);
std::vector<double> inverse_diagonal(const Csr& A);
/// One level of the default-mode V-cycle (amg.cpp:90-111) as two sparse operators.  With
/// Wd = omega diag(A)^-1 the level computes x1 = Wd r + P e_c, e = x1 + Wd (r - A x1) and passes
/// r_c = P^T (r - A Wd r) down; for symmetric A that is
///     r_c = T^T r,    e = S r + T e_c,    T = (I - Wd A) P,    S = 2 Wd - Wd A Wd,
/// i.e. ONE pass per level on the way down and one on the way up instead of two each (the
/// same linear map; rounding differs from the level-by-level order, which the exact mode keeps).
struct FusedCycleOps {
  Csr S, T, Tt;  // Tt = transpose(T): the restriction, exactly T's entries
};
FusedCycleOps fused_cycle_ops(const Csr& A, const Csr& P, const std::vector<double>& wd);
/// dense_cholesky (linalg.cpp:88-105); throws std::runtime_error on failure.
std::vector<double> dense_cholesky(int64_t n, const std::vector<double>& C);
/// Explicit inverse L^-T L^-1 of an SPD matrix from its lower factor.
std::vector<double> cholesky_inverse(int64_t n, const std::vector<double>& L);

}  // namespace gnw::host
