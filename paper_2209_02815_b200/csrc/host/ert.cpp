// ert.cpp -- host side of the ERT forward model (see ert.hpp).
#include "ert.hpp"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace gnw::host {

namespace {
double dist3(const double* p, const double* q) {
  return std::sqrt((p[0] - q[0]) * (p[0] - q[0]) + (p[1] - q[1]) * (p[1] - q[1]) + (p[2] - q[2]) * (p[2] - q[2]));
}
double signed_area(const double* a, const double* b, const double* c) {  // mesh.cpp:16-19
  return 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]));
}
}  // namespace

// survey.cpp:22-46
double geometric_factor(const double a[3], const double* b, const double m[3], const double n[3], int dim) {
  if (dim != 2 && dim != 3) throw std::invalid_argument("geometric_factor: dim must be 2 or 3");
  const double am = dist3(a, m), an = dist3(a, n);
  if (am == 0.0 || an == 0.0 || dist3(m, n) == 0.0 ||
      (b && (dist3(b, m) == 0.0 || dist3(b, n) == 0.0 || dist3(a, b) == 0.0)))
    throw std::invalid_argument("geometric_factor: coincident electrodes");
  double denom;
  if (dim == 2) {
    denom = -std::log(am) + std::log(an);
    if (b) denom += std::log(dist3(b, m)) - std::log(dist3(b, n));
    if (std::abs(denom) < 1e-14) throw std::runtime_error("geometric_factor: degenerate configuration (zero log ratio)");
    return M_PI / denom;
  }
  denom = 1.0 / am - 1.0 / an;
  if (b) denom += -1.0 / dist3(b, m) + 1.0 / dist3(b, n);
  if (std::abs(denom) < 1e-14) throw std::runtime_error("geometric_factor: degenerate configuration (zero denominator)");
  return 2.0 * M_PI / denom;
}

ForwardStructure forward_structure(const Mesh& mesh) {
  ForwardStructure f;
  const int64_t nv = mesh.nv, nc = mesh.nc;
  // grounded nodes: every vertex of a FAR boundary edge (forward.cpp:44-56)
  f.node_to_free.assign(nv, 0);
  for (size_t b = 0; b < mesh.boundary_edges.size(); ++b)
    if (mesh.boundary_tags[b] == 1) {
      const int64_t e = mesh.boundary_edges[b];
      f.node_to_free[mesh.edges[2 * e]] = -1;
      f.node_to_free[mesh.edges[2 * e + 1]] = -1;
    }
  for (int64_t v = 0; v < nv; ++v)
    if (f.node_to_free[v] == 0) {
      f.node_to_free[v] = static_cast<int64_t>(f.free_to_node.size());
      f.free_to_node.push_back(v);
    }
  f.n_free = static_cast<int64_t>(f.free_to_node.size());
  // cell geometry (cell_geometry, forward.cpp:17-36)
  f.area.resize(nc);
  f.grad.resize(6 * nc);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nc; ++c) {
    const int64_t* t = &mesh.cells[3 * c];
    const double* p0 = &mesh.vertices[2 * t[0]];
    const double* p1 = &mesh.vertices[2 * t[1]];
    const double* p2 = &mesh.vertices[2 * t[2]];
    const double area = signed_area(p0, p1, p2);
    const double inv2a = 1.0 / (2.0 * area);
    f.area[c] = area;
    double* g = &f.grad[6 * c];
    g[0] = -(p2[1] - p1[1]) * inv2a;
    g[1] = (p2[0] - p1[0]) * inv2a;
    g[2] = -(p0[1] - p2[1]) * inv2a;
    g[3] = (p0[0] - p2[0]) * inv2a;
    g[4] = -(p1[1] - p0[1]) * inv2a;
    g[5] = (p1[0] - p0[0]) * inv2a;
  }
  // triplets (fi, fj, cell, li, lj) in the reference's generation order (forward.cpp:58-78)
  struct T {
    int64_t r, c, cell;
    int32_t ij;
  };
  std::vector<T> trip;
  trip.reserve(9 * nc);
  for (int64_t c = 0; c < nc; ++c) {
    const int64_t* t = &mesh.cells[3 * c];
    for (int i = 0; i < 3; ++i) {
      const int64_t fi = f.node_to_free[t[i]];
      if (fi < 0) continue;
      for (int j = 0; j < 3; ++j) {
        const int64_t fj = f.node_to_free[t[j]];
        if (fj < 0) continue;
        trip.push_back({fi, fj, c, 3 * i + j});
      }
    }
  }
  std::stable_sort(trip.begin(), trip.end(), [](const T& x, const T& y) { return x.r != y.r ? x.r < y.r : x.c < y.c; });
  Csr& P = f.pattern;
  P.n_rows = P.n_cols = f.n_free;
  P.rowptr.assign(f.n_free + 1, 0);
  for (size_t k = 0; k < trip.size();) {
    const int64_t r = trip[k].r, col = trip[k].c;
    f.contrib_start.push_back(static_cast<int64_t>(f.contrib_cell.size()));
    while (k < trip.size() && trip[k].r == r && trip[k].c == col) {
      f.contrib_cell.push_back(trip[k].cell);
      f.contrib_ij.push_back(trip[k].ij);
      ++k;
    }
    P.cols.push_back(static_cast<int32_t>(col));
    P.vals.push_back(0.0);
    P.rowptr[r + 1] = P.nnz();
  }
  f.contrib_start.push_back(static_cast<int64_t>(f.contrib_cell.size()));
  for (int64_t r = 0; r < f.n_free; ++r) P.rowptr[r + 1] = std::max(P.rowptr[r + 1], P.rowptr[r]);
  return f;
}

// k_ij = sigma * area * (grad_i . grad_j), summed per entry in triplet order (forward.cpp:68-76)
Csr forward_stiffness(const ForwardStructure& f, const double* m) {
  Csr K = f.pattern;
  const int64_t nnz = K.nnz();
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < nnz; ++e) {
    double v = 0.0;
    for (int64_t q = f.contrib_start[e]; q < f.contrib_start[e + 1]; ++q) {
      const int64_t c = f.contrib_cell[q];
      const int i = f.contrib_ij[q] / 3, j = f.contrib_ij[q] % 3;
      const double* g = &f.grad[6 * c];
      const double sigma = std::exp(m[c]);
      const double kij = sigma * f.area[c] * (g[2 * i] * g[2 * j] + g[2 * i + 1] * g[2 * j + 1]);
      v += kij;
    }
    K.vals[e] = v;
  }
  return K;
}

}  // namespace gnw::host
