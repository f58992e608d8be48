// setup.cpp -- host setup of the Woodbury-MINRES path, bit-identical to the
// reference (see setup.hpp).  Reference citations are to /root/reference/proj.
#include "setup.hpp"

#include <omp.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cstdint>
#include <cmath>
#include <numeric>
#include <utility>

namespace gnw::host {

namespace {

double signed_area(const double* a, const double* b, const double* c) {  // mesh.cpp:16-19
  return 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]));
}

// Small (col, value) lists: insertion sort by column, then the reference's
// duplicate summation `v = 0.0; v += t` (sparse.cpp:33-41).  All call sites
// produce at most two duplicates, and IEEE addition is commutative, so the
// order among duplicates cannot change a bit.
template <class Pair>
int emit_sorted(Pair* e, int n, int32_t* cols, double* vals) {
  for (int a = 1; a < n; ++a)
    for (int b = a; b > 0 && e[b - 1].first > e[b].first; --b) std::swap(e[b - 1], e[b]);
  int out = 0;
  for (int k = 0; k < n;) {
    const auto c = e[k].first;
    double v = 0.0;
    while (k < n && e[k].first == c) v += e[k++].second;
    cols[out] = static_cast<int32_t>(c);
    vals[out] = v;
    ++out;
  }
  return out;
}

double coeff(const Csr& A, int64_t i, int64_t j) {  // SparseMatrix::coeff, sparse.cpp:11-17
  const int32_t* b = A.cols.data() + A.rowptr[i];
  const int32_t* e = A.cols.data() + A.rowptr[i + 1];
  const int32_t* it = std::lower_bound(b, e, static_cast<int32_t>(j));
  if (it == e || *it != j) return 0.0;
  return A.vals[static_cast<size_t>(it - A.cols.data())];
}

}  // namespace

Mesh finalize_mesh(const double* vertices, int64_t nv, const int64_t* cells, int64_t nc) {
  Mesh m;
  m.nv = nv;
  m.nc = nc;
  m.vertices.assign(vertices, vertices + 2 * nv);
  m.cells.assign(cells, cells + 3 * nc);
  double scale = 0.0;
  for (int64_t i = 0; i < nv; ++i)
    scale = std::max({scale, std::abs(m.vertices[2 * i]), std::abs(m.vertices[2 * i + 1])});
  // orientation, mesh.cpp:97-106
  for (int64_t c = 0; c < nc; ++c) {
    int64_t* t = &m.cells[3 * c];
    for (int k = 0; k < 3; ++k)
      if (t[k] < 0 || t[k] >= nv) throw std::invalid_argument("finalize_mesh: vertex index out of range");
    double area = signed_area(&m.vertices[2 * t[0]], &m.vertices[2 * t[1]], &m.vertices[2 * t[2]]);
    if (area < 0.0) {
      std::swap(t[1], t[2]);
      area = -area;
    }
    if (!(area > 0.0)) throw std::invalid_argument("finalize_mesh: degenerate cell");
  }
  // Edge numbering by first encounter in (cell, local edge) order, mesh.cpp:116-137.
  // Occurrences are bucketed by their low vertex (stable in occurrence order);
  // the first bucket entry with the same high vertex is the first encounter.
  const int64_t nocc = 3 * nc;
  std::vector<int64_t> start(nv + 1, 0);
  for (int64_t o = 0; o < nocc; ++o) {
    const int64_t c = o / 3, loc = o % 3;
    const int64_t u = m.cells[3 * c + loc], v = m.cells[3 * c + (loc + 1) % 3];
    start[std::min(u, v) + 1]++;
  }
  for (int64_t i = 0; i < nv; ++i) start[i + 1] += start[i];
  std::vector<int64_t> fill(start.begin(), start.end() - 1);
  std::vector<int64_t> b_hi(nocc), b_occ(nocc);
  for (int64_t o = 0; o < nocc; ++o) {
    const int64_t c = o / 3, loc = o % 3;
    const int64_t u = m.cells[3 * c + loc], v = m.cells[3 * c + (loc + 1) % 3];
    const int64_t pos = fill[std::min(u, v)]++;
    b_hi[pos] = std::max(u, v);
    b_occ[pos] = o;
  }
  std::vector<int64_t> entry_edge(nocc, -1);
  m.cell_edges.resize(nocc);
  m.cell_signs.resize(nocc);
  std::vector<int> incidence, sign_sum;
  incidence.reserve(nocc / 2 + 16);
  sign_sum.reserve(nocc / 2 + 16);
  m.edges.reserve(nocc);
  for (int64_t o = 0; o < nocc; ++o) {
    const int64_t c = o / 3, loc = o % 3;
    const int64_t u = m.cells[3 * c + loc], v = m.cells[3 * c + (loc + 1) % 3];
    const int64_t lo = std::min(u, v), hi = std::max(u, v);
    int64_t first = -1;
    for (int64_t k = start[lo]; k < start[lo + 1]; ++k)
      if (b_hi[k] == hi) {
        first = k;
        break;
      }
    int64_t e;
    if (b_occ[first] == o) {
      e = m.ne++;
      entry_edge[first] = e;
      m.edges.push_back(lo);
      m.edges.push_back(hi);
      incidence.push_back(0);
      sign_sum.push_back(0);
    } else {
      e = entry_edge[first];
    }
    const int sign = (u < v) ? +1 : -1;  // mesh.cpp:131
    m.cell_edges[o] = e;
    m.cell_signs[o] = sign;
    incidence[e] += 1;
    sign_sum[e] += sign;
  }
  // boundary tags, mesh.cpp:139-152
  const double surface_tol = 1e-9 * (scale > 0.0 ? scale : 1.0);
  for (int64_t e = 0; e < m.ne; ++e) {
    if (incidence[e] == 1) {
      const int64_t a = m.edges[2 * e], b = m.edges[2 * e + 1];
      const bool on_surface = std::abs(m.vertices[2 * a + 1]) <= surface_tol &&
                              std::abs(m.vertices[2 * b + 1]) <= surface_tol;
      m.boundary_edges.push_back(e);
      m.boundary_tags.push_back(on_surface ? 0 : 1);
    } else if (incidence[e] == 2) {
      if (sign_sum[e] != 0)
        throw std::invalid_argument("finalize_mesh: interior edge with non-opposing orientations");
    } else {
      throw std::invalid_argument("finalize_mesh: edge shared by more than two cells");
    }
  }
  return m;
}

// assemble_Q, fem_mixed.cpp:29-68 (Gamma_N empty => dof = edge).  Built row by
// row from the <= 2 cells adjacent to each edge; each entry value is computed
// exactly as the reference's per-cell triplet.
Csr assemble_Q(const Mesh& m) {
  const int64_t ne = m.ne, nc = m.nc;
  std::vector<int64_t> adj_start(ne + 1, 0);
  for (int64_t o = 0; o < 3 * nc; ++o) adj_start[m.cell_edges[o] + 1]++;
  for (int64_t e = 0; e < ne; ++e) adj_start[e + 1] += adj_start[e];
  std::vector<int64_t> adj(3 * nc), pos(adj_start.begin(), adj_start.end() - 1);
  for (int64_t o = 0; o < 3 * nc; ++o) adj[pos[m.cell_edges[o]]++] = o;  // occurrence ids, ascending

  Csr Q;
  Q.n_rows = Q.n_cols = ne;
  Q.rowptr.assign(ne + 1, 0);
  std::vector<int32_t> tmp_cols(6 * ne);
  std::vector<double> tmp_vals(6 * ne);
  std::vector<int32_t> len(ne);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < ne; ++e) {
    std::pair<int64_t, double> ent[6];
    int n = 0;
    for (int64_t a = adj_start[e]; a < adj_start[e + 1]; ++a) {
      const int64_t o = adj[a], c = o / 3;
      const int li = static_cast<int>(o % 3);
      const int64_t* t = &m.cells[3 * c];
      const double* pts[3] = {&m.vertices[2 * t[0]], &m.vertices[2 * t[1]], &m.vertices[2 * t[2]]};
      const double area = signed_area(pts[0], pts[1], pts[2]);
      const double mids[3][2] = {{0.5 * (pts[0][0] + pts[1][0]), 0.5 * (pts[0][1] + pts[1][1])},
                                 {0.5 * (pts[1][0] + pts[2][0]), 0.5 * (pts[1][1] + pts[2][1])},
                                 {0.5 * (pts[2][0] + pts[0][0]), 0.5 * (pts[2][1] + pts[0][1])}};
      const double* opp_i = pts[(li + 2) % 3];
      const double si = m.cell_signs[3 * c + li];
      for (int lj = 0; lj < 3; ++lj) {
        const double* opp_j = pts[(lj + 2) % 3];
        const double sj = m.cell_signs[3 * c + lj];
        double integral = 0.0;
        for (const auto& q : mids)
          integral += (q[0] - opp_i[0]) * (q[0] - opp_j[0]) + (q[1] - opp_i[1]) * (q[1] - opp_j[1]);
        integral *= area / 3.0;
        ent[n++] = {m.cell_edges[3 * c + lj], si * sj * integral / (4.0 * area * area)};
      }
    }
    len[e] = emit_sorted(ent, n, &tmp_cols[6 * e], &tmp_vals[6 * e]);
  }
  for (int64_t e = 0; e < ne; ++e) Q.rowptr[e + 1] = Q.rowptr[e] + len[e];
  Q.cols.resize(Q.rowptr[ne]);
  Q.vals.resize(Q.rowptr[ne]);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < ne; ++e) {
    std::copy_n(&tmp_cols[6 * e], len[e], &Q.cols[Q.rowptr[e]]);
    std::copy_n(&tmp_vals[6 * e], len[e], &Q.vals[Q.rowptr[e]]);
  }
  return Q;
}

// assemble_D, fem_mixed.cpp:70-82: row c holds the three edge signs.
Csr assemble_D(const Mesh& m) {
  Csr D;
  D.n_rows = m.nc;
  D.n_cols = m.ne;
  D.rowptr.assign(m.nc + 1, 0);
  D.cols.resize(3 * m.nc);
  D.vals.resize(3 * m.nc);
  std::vector<int32_t> len(m.nc);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < m.nc; ++c) {
    std::pair<int64_t, double> ent[3];
    for (int k = 0; k < 3; ++k)
      ent[k] = {m.cell_edges[3 * c + k], static_cast<double>(m.cell_signs[3 * c + k])};
    len[c] = emit_sorted(ent, 3, &D.cols[3 * c], &D.vals[3 * c]);
  }
  for (int64_t c = 0; c < m.nc; ++c) D.rowptr[c + 1] = D.rowptr[c] + len[c];
  if (D.rowptr[m.nc] != 3 * m.nc) throw std::invalid_argument("assemble_D: repeated edge in a cell");
  return D;
}

// transpose, sparse.cpp:97-116 (rows of A visited in order -> sorted columns)
Csr transpose(const Csr& A) {
  Csr T;
  T.n_rows = A.n_cols;
  T.n_cols = A.n_rows;
  T.rowptr.assign(A.n_cols + 1, 0);
  for (int32_t c : A.cols) ++T.rowptr[c + 1];
  for (int64_t r = 0; r < T.n_rows; ++r) T.rowptr[r + 1] += T.rowptr[r];
  T.cols.resize(A.nnz());
  T.vals.resize(A.nnz());
  std::vector<int64_t> fill(T.rowptr.begin(), T.rowptr.end() - 1);
  for (int64_t i = 0; i < A.n_rows; ++i)
    for (int64_t k = A.rowptr[i]; k < A.rowptr[i + 1]; ++k) {
      const int64_t p = fill[A.cols[k]]++;
      T.cols[p] = static_cast<int32_t>(i);
      T.vals[p] = A.vals[k];
    }
  return T;
}

// sparse_matmul, sparse.cpp:118-154.  Row-parallel; each row accumulates in the
// reference's (A entry, B entry) order and emits sorted columns.
namespace {
thread_local SpgemmHook t_spgemm_hook = nullptr;
thread_local void* t_spgemm_user = nullptr;
thread_local int64_t t_spgemm_min = 0;
}  // namespace

void set_spgemm_hook(SpgemmHook fn, void* user, int64_t min_products) {
  t_spgemm_hook = fn;
  t_spgemm_user = user;
  t_spgemm_min = min_products;
}

Csr spgemm(const Csr& A, const Csr& B) {
  if (A.n_cols != B.n_rows) throw std::invalid_argument("sparse_matmul: dimension mismatch");
  if (t_spgemm_hook != nullptr) {
    int64_t products = 0;
    for (int64_t k = 0; k < A.nnz(); ++k) products += B.rowptr[A.cols[k] + 1] - B.rowptr[A.cols[k]];
    if (products >= t_spgemm_min) return t_spgemm_hook(A, B, t_spgemm_user);
  }
  Csr C;
  C.n_rows = A.n_rows;
  C.n_cols = B.n_cols;
  C.rowptr.assign(A.n_rows + 1, 0);
  const int nthreads = omp_get_max_threads();
  const int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(A.n_rows, 4 * nthreads));
  std::vector<std::vector<int32_t>> ccols(nchunks);
  std::vector<std::vector<double>> cvals(nchunks);
  std::vector<int64_t> rowlen(A.n_rows, 0);
#pragma omp parallel
  {
    std::vector<double> accum(B.n_cols, 0.0);
    std::vector<int64_t> mark(B.n_cols, -1);
    std::vector<int32_t> marked;
#pragma omp for schedule(dynamic, 1)
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int64_t r0 = A.n_rows * ch / nchunks, r1 = A.n_rows * (ch + 1) / nchunks;
      auto& oc = ccols[ch];
      auto& ov = cvals[ch];
      for (int64_t i = r0; i < r1; ++i) {
        marked.clear();
        for (int64_t ka = A.rowptr[i]; ka < A.rowptr[i + 1]; ++ka) {
          const int64_t j = A.cols[ka];
          const double aij = A.vals[ka];
          for (int64_t kb = B.rowptr[j]; kb < B.rowptr[j + 1]; ++kb) {
            const int32_t c = B.cols[kb];
            if (mark[c] != i) {
              mark[c] = i;
              accum[c] = 0.0;
              marked.push_back(c);
            }
            accum[c] += aij * B.vals[kb];
          }
        }
        std::sort(marked.begin(), marked.end());
        for (int32_t c : marked) {
          oc.push_back(c);
          ov.push_back(accum[c]);
        }
        rowlen[i] = static_cast<int64_t>(marked.size());
      }
    }
  }
  for (int64_t i = 0; i < A.n_rows; ++i) C.rowptr[i + 1] = C.rowptr[i] + rowlen[i];
  C.cols.resize(C.rowptr[A.n_rows]);
  C.vals.resize(C.rowptr[A.n_rows]);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t ch = 0; ch < nchunks; ++ch) {
    const int64_t r0 = A.n_rows * ch / nchunks;
    std::copy(ccols[ch].begin(), ccols[ch].end(), C.cols.begin() + C.rowptr[r0]);
    std::copy(cvals[ch].begin(), cvals[ch].end(), C.vals.begin() + C.rowptr[r0]);
  }
  return C;
}

FusedCycleOps fused_cycle_ops(const Csr& A, const Csr& P, const std::vector<double>& wd) {
  if (A.n_rows != A.n_cols || P.n_rows != A.n_rows || static_cast<int64_t>(wd.size()) != A.n_rows)
    throw std::invalid_argument("fused_cycle_ops: shape mismatch");
  FusedCycleOps f;
  // S = 2 Wd - Wd A Wd on A's pattern
  f.S = A;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < A.n_rows; ++i)
    for (int64_t k = A.rowptr[i]; k < A.rowptr[i + 1]; ++k) {
      const int64_t j = A.cols[k];
      const double v = -(wd[i] * A.vals[k] * wd[j]);
      f.S.vals[k] = (i == j) ? 2.0 * wd[i] + v : v;
    }
  // T = P - Wd (A P), rows merged by column
  const Csr AP = spgemm(A, P);
  f.T.n_rows = P.n_rows;
  f.T.n_cols = P.n_cols;
  f.T.rowptr.assign(P.n_rows + 1, 0);
  std::vector<int64_t> len(P.n_rows);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < P.n_rows; ++i) {  // |union of the two sorted column lists|
    int64_t a = P.rowptr[i], b = AP.rowptr[i], n = 0;
    while (a < P.rowptr[i + 1] || b < AP.rowptr[i + 1]) {
      const int32_t ca = a < P.rowptr[i + 1] ? P.cols[a] : INT32_MAX;
      const int32_t cb = b < AP.rowptr[i + 1] ? AP.cols[b] : INT32_MAX;
      if (ca <= cb) ++a;
      if (cb <= ca) ++b;
      ++n;
    }
    len[i] = n;
  }
  for (int64_t i = 0; i < P.n_rows; ++i) f.T.rowptr[i + 1] = f.T.rowptr[i] + len[i];
  f.T.cols.resize(f.T.rowptr[P.n_rows]);
  f.T.vals.resize(f.T.rowptr[P.n_rows]);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < P.n_rows; ++i) {
    int64_t a = P.rowptr[i], b = AP.rowptr[i], o = f.T.rowptr[i];
    while (a < P.rowptr[i + 1] || b < AP.rowptr[i + 1]) {
      const int32_t ca = a < P.rowptr[i + 1] ? P.cols[a] : INT32_MAX;
      const int32_t cb = b < AP.rowptr[i + 1] ? AP.cols[b] : INT32_MAX;
      double v = 0.0;
      if (ca <= cb) v = P.vals[a++];
      if (cb <= ca) v = v - wd[i] * AP.vals[b++];
      f.T.cols[o] = std::min(ca, cb);
      f.T.vals[o++] = v;
    }
  }
  f.Tt = transpose(f.T);
  return f;
}

Csr scale_rows(const Csr& A, const std::vector<double>& s) {  // sparse.cpp:156-163
  Csr B = A;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < A.n_rows; ++i)
    for (int64_t k = B.rowptr[i]; k < B.rowptr[i + 1]; ++k) B.vals[k] *= s[i];
  return B;
}

std::vector<double> diagonal(const Csr& A) {  // sparse.cpp:165-170
  const int64_t n = std::min(A.n_rows, A.n_cols);
  std::vector<double> d(n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) d[i] = coeff(A, i, i);
  return d;
}

double symmetry_error(const Csr& A) {  // sparse.cpp:172-179
  if (A.n_rows != A.n_cols) return INFINITY;
  double err = 0.0;
#pragma omp parallel for schedule(static) reduction(max : err)
  for (int64_t i = 0; i < A.n_rows; ++i)
    for (int64_t k = A.rowptr[i]; k < A.rowptr[i + 1]; ++k)
      err = std::max(err, std::abs(A.vals[k] - coeff(A, A.cols[k], i)));
  return err;
}

// assemble_lumped_schur, fem_mixed.cpp:84-94
Csr lumped_schur(const Csr& Q, const Csr& D) {
  if (Q.n_rows != Q.n_cols || D.n_cols != Q.n_rows)
    throw std::invalid_argument("assemble_lumped_schur: shape mismatch");
  std::vector<double> inv = diagonal(Q);
  for (double& v : inv) {
    if (!(v > 0.0)) throw std::runtime_error("assemble_lumped_schur: zero diagonal in Q (degenerate cell)");
    v = 1.0 / v;
  }
  return spgemm(D, scale_rows(transpose(D), inv));
}

Csr from_triplets(int64_t n_rows, int64_t n_cols, std::vector<int64_t> rows, std::vector<int64_t> cols,
                  std::vector<double> vals) {
  const size_t nt = vals.size();
  for (size_t k = 0; k < nt; ++k)
    if (rows[k] < 0 || rows[k] >= n_rows || cols[k] < 0 || cols[k] >= n_cols)
      throw std::invalid_argument("from_triplets: index out of range");
  std::vector<size_t> order(nt);
  std::iota(order.begin(), order.end(), size_t{0});
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return rows[a] != rows[b] ? rows[a] < rows[b] : cols[a] < cols[b];
  });
  Csr A;
  A.n_rows = n_rows;
  A.n_cols = n_cols;
  A.rowptr.assign(n_rows + 1, 0);
  for (size_t k = 0; k < nt;) {
    const int64_t r = rows[order[k]], c = cols[order[k]];
    double v = 0.0;
    while (k < nt && rows[order[k]] == r && cols[order[k]] == c) v += vals[order[k++]];
    A.cols.push_back(static_cast<int32_t>(c));
    A.vals.push_back(v);
    A.rowptr[r + 1] = A.nnz();
  }
  for (int64_t r = 0; r < n_rows; ++r) A.rowptr[r + 1] = std::max(A.rowptr[r + 1], A.rowptr[r]);
  return A;
}

std::vector<double> inverse_diagonal(const Csr& A) {  // amg.cpp:81-88
  std::vector<double> d = diagonal(A);
  for (double& v : d) {
    if (!(v > 0.0)) throw std::invalid_argument("amg_setup: non-positive diagonal entry");
    v = 1.0 / v;
  }
  return d;
}

// aggregate, amg.cpp:13-68 -- inherently sequential (greedy), kept as is.
std::vector<int64_t> aggregate(const Csr& A, const AmgOptions& o, int64_t& n_agg) {
  const int64_t n = A.n_rows;
  const double theta = o.strength;
  const std::vector<double> diag = diagonal(A);
  std::vector<int64_t> agg(n, -1);
  // strength flags, precomputed (row-local, same predicate as amg.cpp:22-26)
  std::vector<uint8_t> strong(A.nnz());
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = A.rowptr[i]; k < A.rowptr[i + 1]; ++k) {
      const int64_t j = A.cols[k];
      strong[k] = (j != i) && std::abs(A.vals[k]) > theta * std::sqrt(std::abs(diag[i] * diag[j]));
    }
  n_agg = 0;
  std::vector<std::pair<double, int64_t>> nbrs;
  for (int64_t i = 0; i < n; ++i) {  // pass 1
    if (agg[i] != -1) continue;
    nbrs.clear();
    bool free_nbhd = true;
    for (int64_t k = A.rowptr[i]; k < A.rowptr[i + 1]; ++k) {
      if (!strong[k]) continue;
      if (agg[A.cols[k]] != -1) {
        free_nbhd = false;
        break;
      }
      nbrs.emplace_back(-std::abs(A.vals[k]), A.cols[k]);
    }
    if (!free_nbhd || nbrs.empty()) continue;
    std::sort(nbrs.begin(), nbrs.end());
    const int64_t id = n_agg++;
    agg[i] = id;
    const size_t take = std::min<size_t>(nbrs.size(), static_cast<size_t>(o.max_aggregate_size - 1));
    for (size_t k = 0; k < take; ++k) agg[nbrs[k].second] = id;
  }
  for (int64_t i = 0; i < n; ++i) {  // pass 2
    if (agg[i] != -1) continue;
    double best = 0.0;
    int64_t best_agg = -1;
    for (int64_t k = A.rowptr[i]; k < A.rowptr[i + 1]; ++k) {
      const int64_t j = A.cols[k];
      if (strong[k] && agg[j] != -1 && std::abs(A.vals[k]) > best) {
        best = std::abs(A.vals[k]);
        best_agg = agg[j];
      }
    }
    if (best_agg != -1) agg[i] = best_agg;
  }
  for (int64_t i = 0; i < n; ++i)  // pass 3
    if (agg[i] == -1) agg[i] = n_agg++;
  return agg;
}

namespace {
// env GNW_SETUP_TIMING=1: per-phase wall times of the host setup on stderr
bool setup_timing() {
  static const bool on = [] {
    const char* e = std::getenv("GNW_SETUP_TIMING");
    return e != nullptr && std::atoi(e) != 0;
  }();
  return on;
}
struct PhaseTimer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void lap(const char* what, long long level = -1) {
    if (!setup_timing()) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gnw setup] %-24s level %2lld  %8.1f ms\n", what, level,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};
}  // namespace

// amg_setup, amg.cpp:115-187
AmgHierarchy amg_setup(const Csr& S, const AmgOptions& o, bool check_symmetry) {
  PhaseTimer pt;
  if (S.n_rows != S.n_cols) throw std::invalid_argument("amg_setup: matrix not square");
  double max_abs = 0.0;
  for (double v : S.vals) max_abs = std::max(max_abs, std::abs(v));
  // check_symmetry = false: S is a coarse level of a hierarchy being continued (the device
  // setup hands its small levels back), which amg.cpp:115-187 does not re-check
  if (check_symmetry && symmetry_error(S) > 1e-12 * std::max(max_abs, 1.0))
    throw std::invalid_argument("amg_setup: matrix not symmetric");
  AmgHierarchy h;
  h.options = o;
  Csr cur = S;
  while (static_cast<int64_t>(h.levels.size()) + 1 < o.max_levels && cur.n_rows > o.coarse_threshold) {
    int64_t n_agg = 0;
    const long long lev = static_cast<long long>(h.levels.size());
    pt.lap("(level start)", lev);
    const std::vector<int64_t> agg = aggregate(cur, o, n_agg);
    pt.lap("aggregate", lev);
    if (n_agg >= cur.n_rows) break;
    // tentative prolongator, amg.cpp:70-79 (one entry per row, no duplicates)
    std::vector<int64_t> count(n_agg, 0);
    for (int64_t a : agg) ++count[a];
    Csr T;
    T.n_rows = cur.n_rows;
    T.n_cols = n_agg;
    T.rowptr.resize(cur.n_rows + 1);
    T.cols.resize(cur.n_rows);
    T.vals.resize(cur.n_rows);
    for (int64_t i = 0; i <= cur.n_rows; ++i) T.rowptr[i] = i;
    for (int64_t i = 0; i < cur.n_rows; ++i) {
      T.cols[i] = static_cast<int32_t>(agg[i]);
      T.vals[i] = 1.0 / std::sqrt(static_cast<double>(count[agg[i]]));
    }
    std::vector<double> inv_diag = inverse_diagonal(cur);
    // filtered operator with weak couplings lumped into the diagonal, amg.cpp:141-166
    Csr F = cur;
    {
      const std::vector<double> diag = diagonal(cur);
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < cur.n_rows; ++i) {
        double lumped = 0.0;
        for (int64_t k = F.rowptr[i]; k < F.rowptr[i + 1]; ++k) {
          const int64_t j = F.cols[k];
          if (j == i) continue;
          if (std::abs(F.vals[k]) <= o.strength * std::sqrt(std::abs(diag[i] * diag[j]))) {
            lumped += F.vals[k];
            F.vals[k] = 0.0;
          }
        }
        for (int64_t k = F.rowptr[i]; k < F.rowptr[i + 1]; ++k)
          if (F.cols[k] == i) {
            F.vals[k] += lumped;
            break;
          }
      }
    }
    std::vector<double> scaled = inverse_diagonal(F);
    for (double& v : scaled) v *= o.prolongation_damping;
    pt.lap("tentative + filtered", lev);
    const Csr AT = spgemm(scale_rows(F, scaled), T);
    pt.lap("spgemm A_F T", lev);
    // P = T - AT through triplets (amg.cpp:168-177): per row, T's single entry
    // and AT's entries merged by column; duplicates (<= 2) summed from 0.0.
    Csr P;
    P.n_rows = T.n_rows;
    P.n_cols = T.n_cols;
    P.rowptr.assign(T.n_rows + 1, 0);
    {
      std::vector<int64_t> len(T.n_rows);
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < T.n_rows; ++i) {
        const int64_t tc = T.cols[i];
        bool hit = false;
        for (int64_t k = AT.rowptr[i]; k < AT.rowptr[i + 1]; ++k) hit |= (AT.cols[k] == tc);
        len[i] = (AT.rowptr[i + 1] - AT.rowptr[i]) + (hit ? 0 : 1);
      }
      for (int64_t i = 0; i < T.n_rows; ++i) P.rowptr[i + 1] = P.rowptr[i] + len[i];
      P.cols.resize(P.rowptr[T.n_rows]);
      P.vals.resize(P.rowptr[T.n_rows]);
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < T.n_rows; ++i) {
        const int32_t tc = T.cols[i];
        int64_t out = P.rowptr[i];
        bool done = false;
        for (int64_t k = AT.rowptr[i]; k < AT.rowptr[i + 1]; ++k) {
          const int32_t c = AT.cols[k];
          if (!done && tc < c) {
            P.cols[out] = tc;
            P.vals[out++] = 0.0 + T.vals[i];
            done = true;
          }
          if (c == tc) {
            double v = 0.0;
            v += T.vals[i];  // IEEE addition commutes: order among the two duplicates is irrelevant
            v += -AT.vals[k];
            P.cols[out] = c;
            P.vals[out++] = v;
            done = true;
          } else {
            P.cols[out] = c;
            P.vals[out++] = 0.0 + -AT.vals[k];
          }
        }
        if (!done) {
          P.cols[out] = tc;
          P.vals[out++] = 0.0 + T.vals[i];
        }
      }
    }
    pt.lap("P merge", lev);
    Csr coarse = spgemm(transpose(P), spgemm(cur, P));  // Galerkin, amg.cpp:179
    pt.lap("galerkin P^T A P", lev);
    h.levels.push_back({std::move(cur), std::move(P), std::move(inv_diag)});
    cur = std::move(coarse);
  }
  std::vector<double> inv_last = inverse_diagonal(cur);
  const int64_t nc = cur.n_rows;
  std::vector<double> dense(nc * nc, 0.0);
  for (int64_t i = 0; i < nc; ++i)
    for (int64_t k = cur.rowptr[i]; k < cur.rowptr[i + 1]; ++k) dense[i * nc + cur.cols[k]] += cur.vals[k];
  h.levels.push_back({std::move(cur), Csr{}, std::move(inv_last)});
  h.coarse_chol = dense_cholesky(nc, dense);
  h.nc = nc;
  pt.lap("coarse cholesky", static_cast<long long>(h.levels.size()) - 1);
  return h;
}

std::vector<double> dense_cholesky(int64_t n, const std::vector<double>& C) {  // linalg.cpp:88-105
  std::vector<double> L(n * n, 0.0);
  for (int64_t j = 0; j < n; ++j) {
    double d = C[j * n + j];
    for (int64_t k = 0; k < j; ++k) d -= L[j * n + k] * L[j * n + k];
    if (!(d > 0.0)) throw std::runtime_error("dense_cholesky: matrix not positive definite");
    const double ljj = std::sqrt(d);
    L[j * n + j] = ljj;
    // one fork/join per column: only worth it for columns with millions of products (with the
    // host oversubscribed, n = 1293 took 8.4 s through 1293 parallel regions, 0.34 s serial)
#pragma omp parallel for schedule(static) if ((n - j) * j > (int64_t{1} << 22))
    for (int64_t i = j + 1; i < n; ++i) {
      double s = C[i * n + j];
      for (int64_t k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = s / ljj;
    }
  }
  return L;
}

std::vector<double> cholesky_inverse(int64_t n, const std::vector<double>& L) {
  // Y = L^-1 column by column (forward substitution), then A^-1 = Y^T Y.
  std::vector<double> Y(n * n, 0.0);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = j; i < n; ++i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int64_t k = j; k < i; ++k) s -= L[i * n + k] * Y[k * n + j];
      Y[i * n + j] = s / L[i * n + i];
    }
  }
  std::vector<double> inv(n * n, 0.0);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j <= i; ++j) {
      double s = 0.0;
      for (int64_t k = i; k < n; ++k) s += Y[k * n + i] * Y[k * n + j];
      inv[i * n + j] = s;
      inv[j * n + i] = s;
    }
  return inv;
}

}  // namespace gnw::host
