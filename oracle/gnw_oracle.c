/*
 * gnw_oracle.c -- TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's Woodbury-MINRES Gauss-Newton step path (arXiv 2209.02815,
 * /root/reference/proj).  It is the CPU checker for the CUDA product and the
 * "port" CPU baseline; it is never linked into the product (libgnw.so).
 *
 * Pinned: tests/test_oracle_pin.py checks every exported function bit-for-bit
 * against the unmodified reference compiled by oracle/Makefile
 * (oracle/_ref/libertinv_ref.so) and against the committed golden fixtures in
 * tests/golden/ (generated from the reference by tests/golden/make_golden.py).
 *
 * Arithmetic is written in the reference's evaluation order and built with
 * -ffp-contract=off so results are bit-identical to the reference's
 * -O3 x86-64 build (no FMA).  Each function cites the reference file:line it
 * restates.  API: orc_api.h.
 */
#define _POSIX_C_SOURCE 200809L
#include "orc_api.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ errors */
static _Thread_local char g_err[512];
static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
#define EINV 1
#define ENUM 2
#define TRY(x)                \
  do {                        \
    int rc__ = (x);           \
    if (rc__) return rc__;    \
  } while (0)

const char* orc_last_error(void) { return g_err; }
const char* orc_flavor(void) { return "restatement"; }

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) {
    fprintf(stderr, "gnw_oracle: out of memory (%zu bytes)\n", n);
    abort();
  }
  return p;
}
static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s ? s : 1);
  if (!p) {
    fprintf(stderr, "gnw_oracle: out of memory\n");
    abort();
  }
  return p;
}
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* --------------------------------------------------------------------- CSR */
/* SparseMatrix, sparse.hpp:14-25 */
typedef struct {
  size_t n_rows, n_cols, nnz;
  size_t* rowptr;
  size_t* cols;
  double* vals;
} csr;

static void csr_free(csr* A) {
  free(A->rowptr);
  free(A->cols);
  free(A->vals);
  memset(A, 0, sizeof *A);
}
static csr csr_copy(const csr* A) {
  csr B = *A;
  B.rowptr = xmalloc((A->n_rows + 1) * sizeof(size_t));
  B.cols = xmalloc(A->nnz * sizeof(size_t));
  B.vals = xmalloc(A->nnz * sizeof(double));
  memcpy(B.rowptr, A->rowptr, (A->n_rows + 1) * sizeof(size_t));
  memcpy(B.cols, A->cols, A->nnz * sizeof(size_t));
  memcpy(B.vals, A->vals, A->nnz * sizeof(double));
  return B;
}

typedef struct {
  size_t row, col;
  double value;
} triplet;

static int trip_cmp(const void* a, const void* b) {
  const triplet* x = a;
  const triplet* y = b;
  if (x->row != y->row) return x->row < y->row ? -1 : 1;
  if (x->col != y->col) return x->col < y->col ? -1 : 1;
  return 0;
}

/* from_triplets, sparse.cpp:19-51.  Sort by (row, col), sum duplicates in
 * sorted order starting from 0.0.  Every call site in this path produces at
 * most two triplets per (row, col), and IEEE addition is commutative, so the
 * (unstable) sort order among duplicates cannot change a bit. */
static int from_triplets(size_t n_rows, size_t n_cols, triplet* t, size_t nt, csr* out) {
  for (size_t k = 0; k < nt; ++k)
    if (t[k].row >= n_rows || t[k].col >= n_cols)
      return fail(EINV, "from_triplets: index out of range");
  qsort(t, nt, sizeof(triplet), trip_cmp);
  csr A = {n_rows, n_cols, 0, NULL, NULL, NULL};
  A.rowptr = xcalloc(n_rows + 1, sizeof(size_t));
  A.cols = xmalloc(nt * sizeof(size_t));
  A.vals = xmalloc(nt * sizeof(double));
  for (size_t k = 0; k < nt;) {
    const size_t r = t[k].row, c = t[k].col;
    double v = 0.0;
    while (k < nt && t[k].row == r && t[k].col == c) {
      v += t[k].value;
      ++k;
    }
    A.cols[A.nnz] = c;
    A.vals[A.nnz] = v;
    A.nnz++;
    A.rowptr[r + 1] = A.nnz;
  }
  for (size_t r = 0; r < n_rows; ++r)
    if (A.rowptr[r + 1] < A.rowptr[r]) A.rowptr[r + 1] = A.rowptr[r];
  *out = A;
  return 0;
}

/* SparseMatrix::coeff, sparse.cpp:11-17 (binary search) */
static double csr_coeff(const csr* A, size_t i, size_t j) {
  size_t lo = A->rowptr[i], hi = A->rowptr[i + 1];
  while (lo < hi) {
    size_t mid = lo + (hi - lo) / 2;
    if (A->cols[mid] < j)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo == A->rowptr[i + 1] || A->cols[lo] != j) return 0.0;
  return A->vals[lo];
}

/* diagonal, sparse.cpp:165-170 */
static double* csr_diagonal(const csr* A) {
  size_t n = A->n_rows < A->n_cols ? A->n_rows : A->n_cols;
  double* d = xmalloc(n * sizeof(double));
  for (size_t i = 0; i < n; ++i) d[i] = csr_coeff(A, i, i);
  return d;
}

/* spmv_add, sparse.cpp:73-83:  y[i] += alpha * sum_k a_ik x_k */
static void spmv_add(const csr* A, const double* x, double alpha, double* y) {
  for (size_t i = 0; i < A->n_rows; ++i) {
    double s = 0.0;
    for (size_t k = A->rowptr[i]; k < A->rowptr[i + 1]; ++k) s += A->vals[k] * x[A->cols[k]];
    y[i] += alpha * s;
  }
}

/* spmv_transpose, sparse.cpp:85-95 (scatter in row order, zero rows skipped) */
static void spmv_transpose(const csr* A, const double* x, double* y) {
  memset(y, 0, A->n_cols * sizeof(double));
  for (size_t i = 0; i < A->n_rows; ++i) {
    const double xi = x[i];
    if (xi == 0.0) continue;
    for (size_t k = A->rowptr[i]; k < A->rowptr[i + 1]; ++k) y[A->cols[k]] += A->vals[k] * xi;
  }
}

/* transpose, sparse.cpp:97-116 */
static csr csr_transpose(const csr* A) {
  csr T = {A->n_cols, A->n_rows, A->nnz, NULL, NULL, NULL};
  T.rowptr = xcalloc(A->n_cols + 1, sizeof(size_t));
  for (size_t k = 0; k < A->nnz; ++k) T.rowptr[A->cols[k] + 1]++;
  for (size_t r = 0; r < T.n_rows; ++r) T.rowptr[r + 1] += T.rowptr[r];
  T.cols = xmalloc(A->nnz * sizeof(size_t));
  T.vals = xmalloc(A->nnz * sizeof(double));
  size_t* fill = xcalloc(T.n_rows, sizeof(size_t));
  for (size_t i = 0; i < A->n_rows; ++i)
    for (size_t k = A->rowptr[i]; k < A->rowptr[i + 1]; ++k) {
      const size_t c = A->cols[k];
      const size_t pos = T.rowptr[c] + fill[c]++;
      T.cols[pos] = i;
      T.vals[pos] = A->vals[k];
    }
  free(fill);
  return T;
}

static int size_cmp(const void* a, const void* b) {
  size_t x = *(const size_t*)a, y = *(const size_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* sparse_matmul, sparse.cpp:118-154: dense accumulator, products added in
 * (A-entry, B-entry) order, output columns sorted. */
static csr csr_matmul(const csr* A, const csr* B) {
  csr C = {A->n_rows, B->n_cols, 0, NULL, NULL, NULL};
  C.rowptr = xcalloc(A->n_rows + 1, sizeof(size_t));
  size_t cap = A->nnz + B->nnz + 16;
  C.cols = xmalloc(cap * sizeof(size_t));
  C.vals = xmalloc(cap * sizeof(double));
  double* accum = xcalloc(B->n_cols, sizeof(double));
  size_t* mark = xmalloc(B->n_cols * sizeof(size_t));
  for (size_t c = 0; c < B->n_cols; ++c) mark[c] = (size_t)-1;
  size_t* marked = xmalloc((B->n_cols + 1) * sizeof(size_t));
  for (size_t i = 0; i < A->n_rows; ++i) {
    size_t nm = 0;
    for (size_t ka = A->rowptr[i]; ka < A->rowptr[i + 1]; ++ka) {
      const size_t j = A->cols[ka];
      const double aij = A->vals[ka];
      for (size_t kb = B->rowptr[j]; kb < B->rowptr[j + 1]; ++kb) {
        const size_t c = B->cols[kb];
        if (mark[c] != i) {
          mark[c] = i;
          accum[c] = 0.0;
          marked[nm++] = c;
        }
        accum[c] += aij * B->vals[kb];
      }
    }
    qsort(marked, nm, sizeof(size_t), size_cmp);
    if (C.nnz + nm > cap) {
      while (C.nnz + nm > cap) cap *= 2;
      C.cols = realloc(C.cols, cap * sizeof(size_t));
      C.vals = realloc(C.vals, cap * sizeof(double));
      if (!C.cols || !C.vals) abort();
    }
    for (size_t q = 0; q < nm; ++q) {
      C.cols[C.nnz] = marked[q];
      C.vals[C.nnz] = accum[marked[q]];
      C.nnz++;
    }
    C.rowptr[i + 1] = C.nnz;
  }
  free(accum);
  free(mark);
  free(marked);
  return C;
}

/* scale_rows, sparse.cpp:156-163 */
static csr csr_scale_rows(const csr* A, const double* s) {
  csr B = csr_copy(A);
  for (size_t i = 0; i < A->n_rows; ++i)
    for (size_t k = B.rowptr[i]; k < B.rowptr[i + 1]; ++k) B.vals[k] *= s[i];
  return B;
}

/* symmetry_error, sparse.cpp:172-179 */
static double csr_symmetry_error(const csr* A) {
  if (A->n_rows != A->n_cols) return INFINITY;
  double err = 0.0;
  for (size_t i = 0; i < A->n_rows; ++i)
    for (size_t k = A->rowptr[i]; k < A->rowptr[i + 1]; ++k) {
      double e = fabs(A->vals[k] - csr_coeff(A, A->cols[k], i));
      if (e > err) err = e;
    }
  return err;
}

/* ------------------------------------------------------------ dense (L0) */
/* dense_cholesky, linalg.cpp:88-105 (reads the lower triangle only) */
static int dense_cholesky(size_t n, const double* C, double* L) {
  memset(L, 0, n * n * sizeof(double));
  for (size_t j = 0; j < n; ++j) {
    double d = C[j * n + j];
    for (size_t k = 0; k < j; ++k) d -= L[j * n + k] * L[j * n + k];
    if (!(d > 0.0)) return fail(ENUM, "dense_cholesky: matrix not positive definite");
    const double ljj = sqrt(d);
    L[j * n + j] = ljj;
    for (size_t i = j + 1; i < n; ++i) {
      double s = C[i * n + j];
      for (size_t k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = s / ljj;
    }
  }
  return 0;
}

/* cholesky_solve_in_place, linalg.cpp:107-123 */
static void cholesky_solve_in_place(size_t n, const double* L, double* x) {
  for (size_t i = 0; i < n; ++i) {
    double s = x[i];
    const double* row = L + i * n;
    for (size_t k = 0; k < i; ++k) s -= row[k] * x[k];
    x[i] = s / row[i];
  }
  for (size_t ii = n; ii-- > 0;) {
    double s = x[ii];
    for (size_t k = ii + 1; k < n; ++k) s -= L[k * n + ii] * x[k];
    x[ii] = s / L[ii * n + ii];
  }
}

/* dot / norm2 / axpy, linalg.cpp:9-21 */
static double vdot(const double* x, const double* y, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}
static double vnorm(const double* x, size_t n) { return sqrt(vdot(x, x, n)); }

/* matvec, linalg.cpp:33-43 (row-major, row-wise sequential sums) */
static void matvec(size_t rows, size_t cols, const double* A, const double* x, double* y) {
  for (size_t i = 0; i < rows; ++i) {
    const double* row = A + i * cols;
    double s = 0.0;
    for (size_t j = 0; j < cols; ++j) s += row[j] * x[j];
    y[i] = s;
  }
}
/* matvec_transpose, linalg.cpp:45-54 */
static void matvec_transpose(size_t rows, size_t cols, const double* A, const double* x,
                             double* y) {
  memset(y, 0, cols * sizeof(double));
  for (size_t i = 0; i < rows; ++i) {
    const double* row = A + i * cols;
    const double xi = x[i];
    for (size_t j = 0; j < cols; ++j) y[j] += row[j] * xi;
  }
}

/* --------------------------------------------------------------- mesh (L3) */
typedef struct {
  size_t nv, nc, ne, nb;
  double* v;        /* 2 per vertex */
  size_t* cells;    /* 3 per cell, CCW after finalize */
  size_t* edges;    /* 2 per edge, low->high */
  size_t* cedges;   /* 3 per cell */
  int* csigns;      /* 3 per cell */
  size_t* bedge;    /* boundary edge ids in edge order */
  int* btag;        /* 0 surface, 1 far */
} mesh_t;

static void mesh_free(mesh_t* m) {
  free(m->v);
  free(m->cells);
  free(m->edges);
  free(m->cedges);
  free(m->csigns);
  free(m->bedge);
  free(m->btag);
}

/* signed_area, mesh.cpp:16-19 */
static double signed_area(const double* a, const double* b, const double* c) {
  return 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]));
}

typedef struct {
  size_t u, v, occ;
} edge_occ;
static int eo_key_cmp(const void* a, const void* b) {
  const edge_occ* x = a;
  const edge_occ* y = b;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  if (x->v != y->v) return x->v < y->v ? -1 : 1;
  return x->occ < y->occ ? -1 : (x->occ > y->occ ? 1 : 0);
}
typedef struct {
  size_t first, group;
} first_occ;
static int fo_cmp(const void* a, const void* b) {
  const first_occ* x = a;
  const first_occ* y = b;
  return x->first < y->first ? -1 : (x->first > y->first ? 1 : 0);
}

/* finalize_mesh, mesh.cpp:85-154.  Edges are numbered by FIRST ENCOUNTER in
 * (cell, local edge) order (the std::map try_emplace at :123); here that order
 * is rebuilt by sorting occurrences by key and the groups by first occurrence. */
static int finalize_mesh(mesh_t* m) {
  double scale = 0.0;
  for (size_t i = 0; i < m->nv; ++i) {
    if (fabs(m->v[2 * i]) > scale) scale = fabs(m->v[2 * i]);
    if (fabs(m->v[2 * i + 1]) > scale) scale = fabs(m->v[2 * i + 1]);
  }
  for (size_t c = 0; c < m->nc; ++c) {
    size_t* t = m->cells + 3 * c;
    for (int k = 0; k < 3; ++k)
      if (t[k] >= m->nv) return fail(EINV, "finalize_mesh: vertex index out of range");
    double area = signed_area(m->v + 2 * t[0], m->v + 2 * t[1], m->v + 2 * t[2]);
    if (area < 0.0) {
      size_t tmp = t[1];
      t[1] = t[2];
      t[2] = tmp;
      area = -area;
    }
    if (!(area > 0.0)) return fail(EINV, "finalize_mesh: degenerate cell");
  }
  const size_t nocc = 3 * m->nc;
  edge_occ* eo = xmalloc(nocc * sizeof(edge_occ));
  for (size_t c = 0; c < m->nc; ++c)
    for (int loc = 0; loc < 3; ++loc) {
      size_t u = m->cells[3 * c + loc], v = m->cells[3 * c + (loc + 1) % 3];
      eo[3 * c + loc] = (edge_occ){u < v ? u : v, u < v ? v : u, 3 * c + loc};
    }
  qsort(eo, nocc, sizeof(edge_occ), eo_key_cmp);
  size_t ngroups = 0;
  for (size_t k = 0; k < nocc; ++k)
    if (k == 0 || eo[k].u != eo[k - 1].u || eo[k].v != eo[k - 1].v) ngroups++;
  first_occ* fo = xmalloc(ngroups * sizeof(first_occ));
  size_t* group_of = xmalloc(nocc * sizeof(size_t)); /* sorted position -> group */
  size_t g = (size_t)-1;
  for (size_t k = 0; k < nocc; ++k) {
    if (k == 0 || eo[k].u != eo[k - 1].u || eo[k].v != eo[k - 1].v) {
      ++g;
      fo[g].first = eo[k].occ; /* occurrences sorted ascending inside a key */
      fo[g].group = g;
    }
    group_of[k] = g;
  }
  qsort(fo, ngroups, sizeof(first_occ), fo_cmp);
  size_t* edge_of_group = xmalloc(ngroups * sizeof(size_t));
  for (size_t e = 0; e < ngroups; ++e) edge_of_group[fo[e].group] = e;
  m->ne = ngroups;
  m->edges = xmalloc(2 * ngroups * sizeof(size_t));
  m->cedges = xmalloc(3 * m->nc * sizeof(size_t));
  m->csigns = xmalloc(3 * m->nc * sizeof(int));
  int* incidence = xcalloc(ngroups, sizeof(int));
  int* sign_sum = xcalloc(ngroups, sizeof(int));
  for (size_t k = 0; k < nocc; ++k) {
    const size_t e = edge_of_group[group_of[k]];
    m->edges[2 * e] = eo[k].u;
    m->edges[2 * e + 1] = eo[k].v;
  }
  for (size_t k = 0; k < nocc; ++k) {
    const size_t occ = eo[k].occ, c = occ / 3;
    const int loc = (int)(occ % 3);
    const size_t u = m->cells[3 * c + loc], v = m->cells[3 * c + (loc + 1) % 3];
    const size_t e = edge_of_group[group_of[k]];
    const int sign = (u < v) ? +1 : -1; /* mesh.cpp:131 */
    m->cedges[occ] = e;
    m->csigns[occ] = sign;
    incidence[e] += 1;
    sign_sum[e] += sign;
  }
  free(eo);
  free(fo);
  free(group_of);
  free(edge_of_group);
  const double surface_tol = 1e-9 * (scale > 0.0 ? scale : 1.0);
  m->bedge = xmalloc((m->ne + 1) * sizeof(size_t));
  m->btag = xmalloc((m->ne + 1) * sizeof(int));
  m->nb = 0;
  int rc = 0;
  for (size_t e = 0; e < m->ne && !rc; ++e) {
    if (incidence[e] == 1) {
      const size_t a = m->edges[2 * e], b = m->edges[2 * e + 1];
      const int on_surface = fabs(m->v[2 * a + 1]) <= surface_tol && fabs(m->v[2 * b + 1]) <= surface_tol;
      m->bedge[m->nb] = e;
      m->btag[m->nb] = on_surface ? 0 : 1;
      m->nb++;
    } else if (incidence[e] == 2) {
      if (sign_sum[e] != 0)
        rc = fail(EINV, "finalize_mesh: interior edge with non-opposing orientations");
    } else {
      rc = fail(EINV, "finalize_mesh: edge shared by more than two cells");
    }
  }
  free(incidence);
  free(sign_sum);
  return rc;
}

/* --------------------------------------------------------- fem_mixed (L3) */
/* assemble_Q, fem_mixed.cpp:29-68 (edge_dof_map = identity: Gamma_N empty,
 * make_mixed_spaces fem_mixed.cpp:8-27) */
static int assemble_Q(const mesh_t* m, csr* Q) {
  triplet* t = xmalloc(9 * m->nc * sizeof(triplet));
  size_t nt = 0;
  for (size_t c = 0; c < m->nc; ++c) {
    const size_t* cv = m->cells + 3 * c;
    const double* pts[3] = {m->v + 2 * cv[0], m->v + 2 * cv[1], m->v + 2 * cv[2]};
    const double area = signed_area(pts[0], pts[1], pts[2]);
    double mids[3][2];
    for (int k = 0; k < 3; ++k) {
      mids[k][0] = 0.5 * (pts[k][0] + pts[(k + 1) % 3][0]);
      mids[k][1] = 0.5 * (pts[k][1] + pts[(k + 1) % 3][1]);
    }
    for (int li = 0; li < 3; ++li) {
      const size_t dof_i = m->cedges[3 * c + li];
      const double* opp_i = pts[(li + 2) % 3];
      const double si = (double)m->csigns[3 * c + li];
      for (int lj = 0; lj < 3; ++lj) {
        const size_t dof_j = m->cedges[3 * c + lj];
        const double* opp_j = pts[(lj + 2) % 3];
        const double sj = (double)m->csigns[3 * c + lj];
        double integral = 0.0;
        for (int q = 0; q < 3; ++q)
          integral += (mids[q][0] - opp_i[0]) * (mids[q][0] - opp_j[0]) +
                      (mids[q][1] - opp_i[1]) * (mids[q][1] - opp_j[1]);
        integral *= area / 3.0;
        t[nt++] = (triplet){dof_i, dof_j, si * sj * integral / (4.0 * area * area)};
      }
    }
  }
  int rc = from_triplets(m->ne, m->ne, t, nt, Q);
  free(t);
  return rc;
}

/* assemble_D, fem_mixed.cpp:70-82 */
static int assemble_D(const mesh_t* m, csr* D) {
  triplet* t = xmalloc(3 * m->nc * sizeof(triplet));
  size_t nt = 0;
  for (size_t c = 0; c < m->nc; ++c)
    for (int loc = 0; loc < 3; ++loc)
      t[nt++] = (triplet){c, m->cedges[3 * c + loc], (double)m->csigns[3 * c + loc]};
  int rc = from_triplets(m->nc, m->ne, t, nt, D);
  free(t);
  return rc;
}

/* assemble_lumped_schur, fem_mixed.cpp:84-94: D * scale_rows(D^T, 1/diag Q) */
static int assemble_lumped_schur(const csr* Q, const csr* D, csr* S) {
  if (Q->n_rows != Q->n_cols || D->n_cols != Q->n_rows)
    return fail(EINV, "assemble_lumped_schur: shape mismatch");
  double* inv = csr_diagonal(Q);
  for (size_t i = 0; i < Q->n_rows; ++i) {
    if (!(inv[i] > 0.0)) {
      free(inv);
      return fail(ENUM, "assemble_lumped_schur: zero diagonal in Q (degenerate cell)");
    }
    inv[i] = 1.0 / inv[i];
  }
  csr Dt = csr_transpose(D);
  csr Ds = csr_scale_rows(&Dt, inv);
  *S = csr_matmul(D, &Ds);
  csr_free(&Dt);
  csr_free(&Ds);
  free(inv);
  return 0;
}

/* --------------------------------------------------------------- amg (L2) */
typedef struct {
  csr A, P;         /* P empty (nnz 0, n_rows 0) on the coarsest level */
  double* inv_diag;
} level_t;

typedef struct {
  orc_amg_opts opts;
  size_t nlev;
  level_t* lev;
  double* coarse_L; /* dense lower Cholesky factor of the coarsest A */
  size_t nc;
} amg_t;

static void amg_free(amg_t* h) {
  for (size_t l = 0; l < h->nlev; ++l) {
    csr_free(&h->lev[l].A);
    csr_free(&h->lev[l].P);
    free(h->lev[l].inv_diag);
  }
  free(h->lev);
  free(h->coarse_L);
  memset(h, 0, sizeof *h);
}

typedef struct {
  double key;
  size_t j;
} nbr_t;
static int nbr_cmp(const void* a, const void* b) {
  const nbr_t* x = a;
  const nbr_t* y = b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->j < y->j ? -1 : (x->j > y->j ? 1 : 0);
}

/* aggregate, amg.cpp:13-68: greedy root aggregation over the strength graph
 * |a_ij| > theta sqrt(|a_ii a_jj|), three passes. */
static size_t* aggregate(const csr* A, const orc_amg_opts* o, size_t* n_agg) {
  const size_t n = A->n_rows;
  const double theta = o->strength;
  double* diag = csr_diagonal(A);
  const size_t kUnset = (size_t)-1;
  size_t* agg = xmalloc(n * sizeof(size_t));
  for (size_t i = 0; i < n; ++i) agg[i] = kUnset;
#define IS_STRONG(i, k)                                 \
  (A->cols[k] != (i) &&                                 \
   fabs(A->vals[k]) > theta * sqrt(fabs(diag[i] * diag[A->cols[k]])))
  size_t na = 0;
  size_t maxrow = 0;
  for (size_t i = 0; i < n; ++i)
    if (A->rowptr[i + 1] - A->rowptr[i] > maxrow) maxrow = A->rowptr[i + 1] - A->rowptr[i];
  nbr_t* nb = xmalloc((maxrow + 1) * sizeof(nbr_t));
  for (size_t i = 0; i < n; ++i) { /* pass 1, amg.cpp:31-49 */
    if (agg[i] != kUnset) continue;
    size_t nn = 0;
    int free_nbhd = 1;
    for (size_t k = A->rowptr[i]; k < A->rowptr[i + 1]; ++k) {
      if (!IS_STRONG(i, k)) continue;
      if (agg[A->cols[k]] != kUnset) {
        free_nbhd = 0;
        break;
      }
      nb[nn++] = (nbr_t){-fabs(A->vals[k]), A->cols[k]};
    }
    if (!free_nbhd || nn == 0) continue;
    qsort(nb, nn, sizeof(nbr_t), nbr_cmp);
    const size_t id = na++;
    agg[i] = id;
    size_t take = o->max_aggregate_size - 1;
    if (nn < take) take = nn;
    for (size_t k = 0; k < take; ++k) agg[nb[k].j] = id;
  }
  for (size_t i = 0; i < n; ++i) { /* pass 2, amg.cpp:51-62 */
    if (agg[i] != kUnset) continue;
    double best = 0.0;
    size_t best_agg = kUnset;
    for (size_t k = A->rowptr[i]; k < A->rowptr[i + 1]; ++k) {
      const size_t j = A->cols[k];
      if (IS_STRONG(i, k) && agg[j] != kUnset && fabs(A->vals[k]) > best) {
        best = fabs(A->vals[k]);
        best_agg = agg[j];
      }
    }
    if (best_agg != kUnset) agg[i] = best_agg;
  }
  for (size_t i = 0; i < n; ++i) /* pass 3, amg.cpp:64-66 */
    if (agg[i] == kUnset) agg[i] = na++;
#undef IS_STRONG
  free(nb);
  free(diag);
  *n_agg = na;
  return agg;
}

/* inverse_diagonal, amg.cpp:81-88 */
static int inverse_diagonal(const csr* A, double** out) {
  double* d = csr_diagonal(A);
  for (size_t i = 0; i < A->n_rows; ++i) {
    if (!(d[i] > 0.0)) {
      free(d);
      return fail(EINV, "amg_setup: non-positive diagonal entry");
    }
    d[i] = 1.0 / d[i];
  }
  *out = d;
  return 0;
}

/* amg_setup, amg.cpp:115-187 */
static int amg_setup(const csr* S, const orc_amg_opts* o, amg_t* h) {
  memset(h, 0, sizeof *h);
  if (S->n_rows != S->n_cols) return fail(EINV, "amg_setup: matrix not square");
  double max_abs = 0.0;
  for (size_t k = 0; k < S->nnz; ++k)
    if (fabs(S->vals[k]) > max_abs) max_abs = fabs(S->vals[k]);
  if (csr_symmetry_error(S) > 1e-12 * (max_abs > 1.0 ? max_abs : 1.0))
    return fail(EINV, "amg_setup: matrix not symmetric");
  h->opts = *o;
  size_t cap = o->max_levels + 1;
  h->lev = xcalloc(cap, sizeof(level_t));
  csr cur = csr_copy(S);
  int rc = 0;
  while (h->nlev + 1 < o->max_levels && cur.n_rows > o->coarse_threshold) {
    size_t n_agg = 0;
    size_t* agg = aggregate(&cur, o, &n_agg);
    if (n_agg >= cur.n_rows) {
      free(agg);
      break;
    }
    /* tentative_prolongator, amg.cpp:70-79 */
    size_t* count = xcalloc(n_agg, sizeof(size_t));
    for (size_t i = 0; i < cur.n_rows; ++i) count[agg[i]]++;
    triplet* tt = xmalloc(cur.n_rows * sizeof(triplet));
    for (size_t i = 0; i < cur.n_rows; ++i)
      tt[i] = (triplet){i, agg[i], 1.0 / sqrt((double)count[agg[i]])};
    csr T;
    from_triplets(cur.n_rows, n_agg, tt, cur.n_rows, &T);
    free(tt);
    free(count);
    free(agg);
    double* inv_diag = NULL;
    if ((rc = inverse_diagonal(&cur, &inv_diag))) {
      csr_free(&T);
      break;
    }
    /* filtered, lumped operator, amg.cpp:141-166 */
    csr F = csr_copy(&cur);
    {
      double* diag = csr_diagonal(&cur);
      double* lumped = xcalloc(cur.n_rows, sizeof(double));
      for (size_t i = 0; i < cur.n_rows; ++i)
        for (size_t k = F.rowptr[i]; k < F.rowptr[i + 1]; ++k) {
          const size_t j = F.cols[k];
          if (j == i) continue;
          if (fabs(F.vals[k]) <= o->strength * sqrt(fabs(diag[i] * diag[j]))) {
            lumped[i] += F.vals[k];
            F.vals[k] = 0.0;
          }
        }
      for (size_t i = 0; i < cur.n_rows; ++i)
        for (size_t k = F.rowptr[i]; k < F.rowptr[i + 1]; ++k)
          if (F.cols[k] == i) {
            F.vals[k] += lumped[i];
            break;
          }
      free(diag);
      free(lumped);
    }
    double* scaled = NULL;
    if ((rc = inverse_diagonal(&F, &scaled))) {
      csr_free(&T);
      csr_free(&F);
      free(inv_diag);
      break;
    }
    for (size_t i = 0; i < cur.n_rows; ++i) scaled[i] *= o->prolongation_damping;
    csr Fs = csr_scale_rows(&F, scaled);
    csr AT = csr_matmul(&Fs, &T);
    /* P = T - AT via triplets, amg.cpp:168-177 */
    triplet* pt = xmalloc((T.nnz + AT.nnz) * sizeof(triplet));
    size_t np = 0;
    for (size_t i = 0; i < T.n_rows; ++i) {
      for (size_t k = T.rowptr[i]; k < T.rowptr[i + 1]; ++k) pt[np++] = (triplet){i, T.cols[k], T.vals[k]};
      for (size_t k = AT.rowptr[i]; k < AT.rowptr[i + 1]; ++k) pt[np++] = (triplet){i, AT.cols[k], -AT.vals[k]};
    }
    csr P;
    from_triplets(T.n_rows, T.n_cols, pt, np, &P);
    free(pt);
    /* Galerkin coarse operator P^T (A P), amg.cpp:179 */
    csr AP = csr_matmul(&cur, &P);
    csr Pt = csr_transpose(&P);
    csr coarse = csr_matmul(&Pt, &AP);
    csr_free(&AP);
    csr_free(&Pt);
    csr_free(&Fs);
    csr_free(&AT);
    csr_free(&F);
    csr_free(&T);
    free(scaled);
    level_t* L = &h->lev[h->nlev++];
    L->A = cur;
    L->P = P;
    L->inv_diag = inv_diag;
    cur = coarse;
  }
  if (rc) {
    csr_free(&cur);
    amg_free(h);
    return rc;
  }
  level_t* L = &h->lev[h->nlev++];
  L->A = cur;
  memset(&L->P, 0, sizeof L->P);
  if ((rc = inverse_diagonal(&L->A, &L->inv_diag))) {
    amg_free(h);
    return rc;
  }
  /* to_dense + dense_cholesky, amg.cpp:185 */
  const size_t nc = L->A.n_rows;
  double* Dn = xcalloc(nc * nc, sizeof(double));
  for (size_t i = 0; i < nc; ++i)
    for (size_t k = L->A.rowptr[i]; k < L->A.rowptr[i + 1]; ++k) Dn[i * nc + L->A.cols[k]] += L->A.vals[k];
  h->coarse_L = xmalloc(nc * nc * sizeof(double));
  h->nc = nc;
  rc = dense_cholesky(nc, Dn, h->coarse_L);
  free(Dn);
  if (rc) amg_free(h);
  return rc;
}

/* cycle, amg.cpp:90-111: one symmetric V-cycle, damped Jacobi pre/post */
static void amg_cycle(const amg_t* h, size_t level, const double* r, double* x) {
  const level_t* lv = &h->lev[level];
  const size_t n = lv->A.n_rows;
  if (level + 1 == h->nlev) {
    memcpy(x, r, n * sizeof(double));
    cholesky_solve_in_place(n, h->coarse_L, x);
    return;
  }
  const double omega = h->opts.jacobi_damping;
  for (size_t i = 0; i < n; ++i) x[i] = omega * lv->inv_diag[i] * r[i];
  double* resid = xmalloc(n * sizeof(double));
  memcpy(resid, r, n * sizeof(double));
  spmv_add(&lv->A, x, -1.0, resid);
  const size_t nc = lv->P.n_cols;
  double* rc = xmalloc(nc * sizeof(double));
  double* ec = xmalloc(nc * sizeof(double));
  spmv_transpose(&lv->P, resid, rc);
  amg_cycle(h, level + 1, rc, ec);
  spmv_add(&lv->P, ec, 1.0, x);
  memcpy(resid, r, n * sizeof(double));
  spmv_add(&lv->A, x, -1.0, resid);
  for (size_t i = 0; i < n; ++i) x[i] += omega * lv->inv_diag[i] * resid[i];
  free(resid);
  free(rc);
  free(ec);
}

/* ----------------------------------------------------- inversion (L4) */
struct orc_problem {
  int mixed;
  mesh_t mesh;
  csr Q, D, S;
  double* qinv;
  amg_t amg;
  size_t K, N;
  /* Woodbury state */
  int pc_laplace; /* Alg. 4: J in the operator, Laplace preconditioner */
  size_t m;
  double beta;
  double* J; /* m x N */
  double* H; /* N x m */
  double* L; /* m x m */
};

static orc_amg_opts default_opts(const orc_amg_opts* o) {
  if (o) return *o;
  orc_amg_opts d = {64, 0.08, 2.0 / 3.0, 2.0 / 3.0, 3, 25}; /* amg.hpp:11-21 */
  return d;
}

orc_problem* orc_create_mixed(const double* vertices, uint64_t n_vertices, const int64_t* cells,
                              uint64_t n_cells, const orc_amg_opts* opts) {
  orc_problem* p = xcalloc(1, sizeof *p);
  p->mixed = 1;
  p->beta = 1.0;
  mesh_t* m = &p->mesh;
  m->nv = n_vertices;
  m->nc = n_cells;
  m->v = xmalloc(2 * n_vertices * sizeof(double));
  memcpy(m->v, vertices, 2 * n_vertices * sizeof(double));
  m->cells = xmalloc(3 * n_cells * sizeof(size_t));
  for (size_t k = 0; k < 3 * n_cells; ++k) m->cells[k] = (size_t)cells[k];
  orc_amg_opts o = default_opts(opts);
  int rc = finalize_mesh(m);
  if (!rc) rc = assemble_Q(m, &p->Q);
  if (!rc) rc = assemble_D(m, &p->D);
  if (!rc) {
    /* inversion.cpp:210-211 */
    p->qinv = csr_diagonal(&p->Q);
    for (size_t i = 0; i < p->Q.n_rows; ++i) p->qinv[i] = 1.0 / p->qinv[i];
    rc = assemble_lumped_schur(&p->Q, &p->D, &p->S);
  }
  if (!rc) rc = amg_setup(&p->S, &o, &p->amg);
  if (rc) {
    orc_destroy(p);
    return NULL;
  }
  p->K = m->ne;
  p->N = m->nc;
  return p;
}

orc_problem* orc_create_amg_csr(uint64_t n, const int64_t* rowptr, const int64_t* cols,
                                const double* vals, const orc_amg_opts* opts) {
  orc_problem* p = xcalloc(1, sizeof *p);
  size_t nnz = (size_t)rowptr[n];
  triplet* t = xmalloc(nnz * sizeof(triplet));
  for (size_t i = 0; i < n; ++i)
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) t[k] = (triplet){i, (size_t)cols[k], vals[k]};
  orc_amg_opts o = default_opts(opts);
  int rc = from_triplets(n, n, t, nnz, &p->S);
  free(t);
  if (!rc) rc = amg_setup(&p->S, &o, &p->amg);
  if (rc) {
    orc_destroy(p);
    return NULL;
  }
  p->N = n;
  return p;
}

void orc_destroy(orc_problem* p) {
  if (!p) return;
  mesh_free(&p->mesh);
  csr_free(&p->Q);
  csr_free(&p->D);
  csr_free(&p->S);
  free(p->qinv);
  amg_free(&p->amg);
  free(p->J);
  free(p->H);
  free(p->L);
  free(p);
}

int orc_sizes(const orc_problem* p, uint64_t s[8]) {
  memset(s, 0, 8 * sizeof(uint64_t));
  s[0] = p->K;
  s[1] = p->N;
  s[2] = p->mesh.nv;
  s[3] = p->mesh.nc;
  s[4] = p->mesh.ne;
  s[5] = p->amg.nlev;
  s[6] = p->mesh.nb;
  s[7] = p->amg.nc;
  return 0;
}

int orc_mesh(const orc_problem* p, int64_t* cells, int64_t* edges, int64_t* cell_edges,
             int32_t* signs, int64_t* bedges, int32_t* btags) {
  if (!p->mixed) return fail(EINV, "orc_mesh: not a mixed problem");
  const mesh_t* m = &p->mesh;
  for (size_t k = 0; k < 3 * m->nc; ++k) {
    if (cells) cells[k] = (int64_t)m->cells[k];
    if (cell_edges) cell_edges[k] = (int64_t)m->cedges[k];
    if (signs) signs[k] = m->csigns[k];
  }
  for (size_t k = 0; k < 2 * m->ne; ++k)
    if (edges) edges[k] = (int64_t)m->edges[k];
  for (size_t b = 0; b < m->nb; ++b) {
    if (bedges) bedges[b] = (int64_t)m->bedge[b];
    if (btags) btags[b] = m->btag[b];
  }
  return 0;
}

int orc_csr(const orc_problem* p, int which, uint64_t level, uint64_t* n_rows, uint64_t* n_cols,
            uint64_t* nnz, int64_t* rowptr, int64_t* cols, double* vals) {
  const csr* A = NULL;
  switch (which) {
    case 0: A = &p->Q; break;
    case 1: A = &p->D; break;
    case 2: A = &p->S; break;
    case 3:
    case 4:
      if (level >= p->amg.nlev) return fail(EINV, "orc_csr: level out of range");
      A = which == 3 ? &p->amg.lev[level].A : &p->amg.lev[level].P;
      break;
    default: return fail(EINV, "orc_csr: bad selector");
  }
  if (n_rows) *n_rows = A->n_rows;
  if (n_cols) *n_cols = A->n_cols;
  if (nnz) *nnz = A->nnz;
  if (rowptr) {
    if (A->rowptr)
      for (size_t i = 0; i <= A->n_rows; ++i) rowptr[i] = (int64_t)A->rowptr[i];
    else
      rowptr[0] = 0;
  }
  if (cols)
    for (size_t k = 0; k < A->nnz; ++k) cols[k] = (int64_t)A->cols[k];
  if (vals && A->nnz) memcpy(vals, A->vals, A->nnz * sizeof(double));
  return 0;
}

int orc_level_inv_diag(const orc_problem* p, uint64_t level, double* out) {
  if (level >= p->amg.nlev) return fail(EINV, "orc_level_inv_diag: level out of range");
  memcpy(out, p->amg.lev[level].inv_diag, p->amg.lev[level].A.n_rows * sizeof(double));
  return 0;
}

int orc_coarse_cholesky(const orc_problem* p, double* out) {
  memcpy(out, p->amg.coarse_L, p->amg.nc * p->amg.nc * sizeof(double));
  return 0;
}

int orc_q_diag_inv(const orc_problem* p, double* out) {
  memcpy(out, p->qinv, p->K * sizeof(double));
  return 0;
}

/* amg_apply, amg.cpp:189-194 */
int orc_amg_apply(const orc_problem* p, const double* r, double* z) {
  if (p->amg.nlev == 0) return fail(EINV, "amg_apply: empty hierarchy");
  amg_cycle(&p->amg, 0, r, z);
  return 0;
}

/* build_woodbury_preconditioner, inversion.cpp:91-124 (+ capacitance_matrix
 * :37-43 and cholesky_with_retry :21-35) */
int orc_set_jacobian(orc_problem* p, const double* J, uint64_t m, double beta, double timings[3]) {
  if (!p->mixed) return fail(EINV, "orc_set_jacobian: not a mixed problem");
  free(p->J);
  free(p->H);
  free(p->L);
  p->J = p->H = p->L = NULL;
  p->m = 0;
  p->beta = beta;
  if (timings) timings[0] = timings[1] = timings[2] = 0.0;
  if (m == 0) return 0; /* plain Laplace preconditioner, inversion.cpp:251-256 */
  if (!(beta > 0.0)) return fail(EINV, "build_woodbury_preconditioner: beta <= 0");
  const size_t N = p->N;
  p->m = m;
  p->J = xmalloc(m * N * sizeof(double));
  memcpy(p->J, J, m * N * sizeof(double));
  if (p->pc_laplace) return 0; /* inversion.cpp:251-256 */
  double t0 = now_s();
  p->H = xmalloc(N * m * sizeof(double));
  double* col = xmalloc(N * sizeof(double));
  double* h = xmalloc(N * sizeof(double));
  for (size_t i = 0; i < m; ++i) {
    for (size_t c = 0; c < N; ++c) col[c] = J[i * N + c];
    amg_cycle(&p->amg, 0, col, h);
    for (size_t c = 0; c < N; ++c) p->H[c * m + i] = h[c];
  }
  free(col);
  free(h);
  if (timings) timings[0] = now_s() - t0;
  t0 = now_s();
  /* capacitance_matrix: C = matmul(J, H) (i-k-j, zero a_ik skipped,
   * linalg.cpp:56-70), then /beta, then +1 on the diagonal */
  double* C = xcalloc(m * m, sizeof(double));
  for (size_t i = 0; i < m; ++i) {
    double* crow = C + i * m;
    for (size_t k = 0; k < N; ++k) {
      const double aik = J[i * N + k];
      if (aik == 0.0) continue;
      const double* brow = p->H + k * m;
      for (size_t j = 0; j < m; ++j) crow[j] += aik * brow[j];
    }
  }
  for (size_t k = 0; k < m * m; ++k) C[k] /= beta;
  for (size_t i = 0; i < m; ++i) C[i * m + i] += 1.0;
  if (timings) timings[1] = now_s() - t0;
  t0 = now_s();
  p->L = xmalloc(m * m * sizeof(double));
  int rc = dense_cholesky(m, C, p->L);
  if (rc) { /* cholesky_with_retry: symmetrize once, inversion.cpp:24-33 */
    for (size_t i = 0; i < m; ++i)
      for (size_t j = i + 1; j < m; ++j) {
        const double v = 0.5 * (C[i * m + j] + C[j * m + i]);
        C[i * m + j] = v;
        C[j * m + i] = v;
      }
    rc = dense_cholesky(m, C, p->L);
  }
  free(C);
  if (timings) timings[2] = now_s() - t0;
  return rc;
}

int orc_set_pc_laplace(orc_problem* p, int laplace) {
  p->pc_laplace = laplace != 0;
  return 0;
}

int orc_get_H(const orc_problem* p, double* out) {
  memcpy(out, p->H, p->N * p->m * sizeof(double));
  return 0;
}
int orc_get_L(const orc_problem* p, double* out) {
  memcpy(out, p->L, p->m * p->m * sizeof(double));
  return 0;
}

/* SaddleOperator::apply, inversion.cpp:47-69 */
static void saddle_apply(const orc_problem* p, const double* x, double* out) {
  const size_t K = p->K, N = p->N;
  const double* zeta = x;
  const double* dm = x + K;
  memset(out, 0, (K + N) * sizeof(double));
  double* out1 = out;
  double* out2 = out + K;
  spmv_add(&p->Q, zeta, 1.0, out1);
  double* dt = xmalloc(K * sizeof(double));
  spmv_transpose(&p->D, dm, dt);
  for (size_t i = 0; i < K; ++i) out1[i] += 1.0 * dt[i];
  free(dt);
  spmv_add(&p->D, zeta, 1.0, out2);
  if (p->m > 0) {
    double* jdm = xmalloc(p->m * sizeof(double));
    double* jt = xmalloc(N * sizeof(double));
    matvec(p->m, N, p->J, dm, jdm);
    matvec_transpose(p->m, N, p->J, jdm, jt);
    const double a = -1.0 / p->beta;
    for (size_t i = 0; i < N; ++i) out2[i] += a * jt[i];
    free(jdm);
    free(jt);
  }
}

/* WoodburyPreconditioner::apply, inversion.cpp:71-89 */
static void woodbury_apply(const orc_problem* p, const double* y, double* out) {
  const size_t K = p->K, N = p->N;
  for (size_t i = 0; i < K; ++i) out[i] = p->qinv[i] * y[i];
  const double* y2 = y + K;
  double* s = out + K;
  amg_cycle(&p->amg, 0, y2, s);
  if (p->m > 0 && !p->pc_laplace) {
    double* t = xmalloc(p->m * sizeof(double));
    double* w = xmalloc(N * sizeof(double));
    matvec_transpose(N, p->m, p->H, y2, t);
    cholesky_solve_in_place(p->m, p->L, t);
    matvec(N, p->m, p->H, t, w);
    const double a = -1.0 / p->beta;
    for (size_t i = 0; i < N; ++i) s[i] += a * w[i];
    free(t);
    free(w);
  }
}

int orc_apply_operator(const orc_problem* p, const double* x, double* y) {
  if (!p->mixed) return fail(EINV, "SaddleOperator: not a mixed problem");
  saddle_apply(p, x, y);
  return 0;
}

int orc_precondition(const orc_problem* p, const double* y, double* z) {
  if (!p->mixed) return fail(EINV, "WoodburyPreconditioner: not a mixed problem");
  woodbury_apply(p, y, z);
  return 0;
}

/* assemble_gn_rhs, inversion.cpp:126-146 */
int orc_assemble_rhs(const orc_problem* p, const double* m, const double* m_ref, const double* g,
                     const double* g_obs, double* rhs) {
  const size_t K = p->K, N = p->N, M = p->m;
  double* dm = xmalloc(N * sizeof(double));
  for (size_t i = 0; i < N; ++i) dm[i] = m[i] - m_ref[i];
  double* dt = xmalloc(K * sizeof(double));
  spmv_transpose(&p->D, dm, dt);
  for (size_t i = 0; i < K; ++i) rhs[i] = -dt[i];
  double* dg = xmalloc((M ? M : 1) * sizeof(double));
  for (size_t i = 0; i < M; ++i) dg[i] = g[i] - g_obs[i];
  double* jt = xcalloc(N, sizeof(double));
  if (M) matvec_transpose(M, N, p->J, dg, jt);
  for (size_t i = 0; i < N; ++i) rhs[K + i] = jt[i] / p->beta;
  free(dm);
  free(dt);
  free(dg);
  free(jt);
  return 0;
}

/* combine, minres.cpp:11-16 */
static void combine(size_t n, const double* a, double ca, const double* b, double cb,
                    const double* c, double cc, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = ca * a[i] + cb * b[i] + cc * c[i];
}

/* residual r = b - A x */
static void true_residual(const orc_problem* p, const double* b, const double* x, double* r, size_t n) {
  saddle_apply(p, x, r);
  for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
}

/* minres, minres.cpp:20-155 */
int orc_minres(const orc_problem* p, const double* b, const double* x0, double tol, uint64_t maxit,
               double* x, orc_minres_report* rep, double* he, double* hp, uint64_t cap) {
  if (!(tol > 0.0)) return fail(EINV, "minres: tol must be positive");
  if (!p->mixed) return fail(EINV, "minres: not a mixed problem");
  const size_t n = p->K + p->N;
  memset(rep, 0, sizeof *rep);
  memcpy(x, x0, n * sizeof(double));
  size_t nh = 0;
#define PUSH(e, pn)                  \
  do {                               \
    if (nh < cap) {                  \
      if (he) he[nh] = (e);          \
      if (hp) hp[nh] = (pn);         \
    }                                \
    ++nh;                            \
  } while (0)
#define SET_BACK(e) \
  do {              \
    if (nh - 1 < cap && he) he[nh - 1] = (e); \
  } while (0)

  const double bnorm = vnorm(b, n);
  double* V = xmalloc(14 * n * sizeof(double));
  double *r = V, *z = V + n, *v_prev = V + 2 * n, *v_cur = V + 3 * n, *w_prev = V + 4 * n,
         *w_cur = V + 5 * n, *u_prev = V + 6 * n, *u_cur = V + 7 * n, *zhat = V + 8 * n,
         *Az = V + 9 * n, *v_next = V + 10 * n, *z_next = V + 11 * n, *w_next = V + 12 * n,
         *u_next = V + 13 * n;
  int rc = 0;
  if (bnorm == 0.0) { /* minres.cpp:32-39 */
    saddle_apply(p, x, r);
    rep->converged = vnorm(r, n) == 0.0;
    PUSH(0.0, 0.0);
    rep->n_hist = nh;
    free(V);
    return 0;
  }
  true_residual(p, b, x, r, n);
  woodbury_apply(p, r, z);
  const double gamma_sq0 = vdot(r, z, n);
  if (gamma_sq0 < 0.0) {
    free(V);
    return fail(ENUM, "minres: preconditioner is not positive definite");
  }
  const double gamma1 = sqrt(gamma_sq0);
  double rel0 = vnorm(r, n) / bnorm;
  PUSH(rel0, 1.0);
  if (rel0 <= tol) {
    rep->converged = 1;
    rep->true_relative_residual = rel0;
    rep->n_hist = nh;
    free(V);
    return 0;
  }
  if (gamma1 == 0.0) {
    free(V);
    return fail(ENUM, "minres: breakdown (zero preconditioned residual, nonzero residual)");
  }
  memset(v_prev, 0, n * sizeof(double));
  memcpy(v_cur, r, n * sizeof(double));
  memset(w_prev, 0, n * sizeof(double));
  memset(w_cur, 0, n * sizeof(double));
  memset(u_prev, 0, n * sizeof(double));
  memset(u_cur, 0, n * sizeof(double));
  double gamma_prev = 1.0, gamma_cur = gamma1;
  double c_prev = 1.0, c_cur = 1.0, s_prev = 0.0, s_cur = 0.0;
  double eta = gamma1;
  const double exhausted_tol = 1e-13 * gamma1;

  for (uint64_t j = 1; j <= maxit; ++j) {
    const double ig = 1.0 / gamma_cur;
    for (size_t i = 0; i < n; ++i) zhat[i] = z[i] * ig;
    saddle_apply(p, zhat, Az);
    const double delta = vdot(Az, zhat, n);
    combine(n, Az, 1.0, v_cur, -delta / gamma_cur, v_prev, -gamma_cur / gamma_prev, v_next);
    woodbury_apply(p, v_next, z_next);
    const double gamma_sq = vdot(z_next, v_next, n);
    if (gamma_sq < -1e-12 * (vnorm(z_next, n) * vnorm(v_next, n) + 1.0)) {
      rc = fail(ENUM, "minres: preconditioner is not positive definite");
      break;
    }
    const double gamma_next = sqrt(gamma_sq > 0.0 ? gamma_sq : 0.0);
    const double alpha0 = c_cur * delta - c_prev * s_cur * gamma_cur;
    const double alpha1 = sqrt(alpha0 * alpha0 + gamma_next * gamma_next);
    const double alpha2 = s_cur * delta + c_prev * c_cur * gamma_cur;
    const double alpha3 = s_prev * gamma_cur;
    if (alpha1 == 0.0) {
      rc = fail(ENUM, "minres: breakdown (stagnated rotation)");
      break;
    }
    const double c_next = alpha0 / alpha1;
    const double s_next = gamma_next / alpha1;
    const double ia = 1.0 / alpha1;
    combine(n, zhat, 1.0, w_prev, -alpha3, w_cur, -alpha2, w_next);
    for (size_t i = 0; i < n; ++i) w_next[i] *= ia;
    combine(n, Az, 1.0, u_prev, -alpha3, u_cur, -alpha2, u_next);
    for (size_t i = 0; i < n; ++i) u_next[i] *= ia;
    const double tau = c_next * eta;
    for (size_t i = 0; i < n; ++i) x[i] += tau * w_next[i];
    const double mtau = -tau;
    for (size_t i = 0; i < n; ++i) r[i] += mtau * u_next[i];
    eta = -s_next * eta;
    rep->iterations = j;
    const double rel = vnorm(r, n) / bnorm;
    PUSH(rel, fabs(eta) / gamma1);
    if (rel <= tol) { /* minres.cpp:108-120 */
      true_residual(p, b, x, r, n);
      const double rel_true = vnorm(r, n) / bnorm;
      SET_BACK(rel_true);
      if (rel_true <= 10.0 * tol) {
        rep->converged = 1;
        rep->true_relative_residual = rel_true;
        rep->n_hist = nh;
        free(V);
        return 0;
      }
    }
    if (gamma_next <= exhausted_tol) { /* minres.cpp:122-133 */
      double* rt = xmalloc(n * sizeof(double));
      true_residual(p, b, x, rt, n);
      const double rel_true = vnorm(rt, n) / bnorm;
      free(rt);
      rep->true_relative_residual = rel_true;
      rep->n_hist = nh;
      if (rel_true <= 10.0 * tol) {
        rep->converged = 1;
        free(V);
        return 0;
      }
      free(V);
      return fail(ENUM, "minres: breakdown (Krylov space exhausted before convergence)");
    }
    /* rotate, minres.cpp:135-148 */
    double* t;
    t = v_prev; v_prev = v_cur; v_cur = v_next; v_next = t;
    t = z; z = z_next; z_next = t;
    gamma_prev = gamma_cur;
    gamma_cur = gamma_next;
    c_prev = c_cur;
    c_cur = c_next;
    s_prev = s_cur;
    s_cur = s_next;
    t = w_prev; w_prev = w_cur; w_cur = w_next; w_next = t;
    t = u_prev; u_prev = u_cur; u_cur = u_next; u_next = t;
  }
  if (rc) {
    free(V);
    rep->n_hist = nh;
    return rc;
  }
  /* maxit exhausted, minres.cpp:150-154 */
  true_residual(p, b, x, r, n);
  rep->true_relative_residual = vnorm(r, n) / bnorm;
  rep->converged = 0;
  rep->n_hist = nh;
  free(V);
  return 0;
#undef PUSH
#undef SET_BACK
}

int orc_dense_cholesky(uint64_t n, const double* C, double* L) { return dense_cholesky(n, C, L); }

/* ------------------------------------------------------------ ERT (C4/C5) */
static double dist3(const double* p, const double* q) {
  return sqrt((p[0] - q[0]) * (p[0] - q[0]) + (p[1] - q[1]) * (p[1] - q[1]) + (p[2] - q[2]) * (p[2] - q[2]));
}

/* geometric_factor, survey.cpp:22-46 */
int orc_geometric_factor(const double a[3], const double* b, const double m[3], const double n[3], int dim,
                         double* k) {
  if (dim != 2 && dim != 3) return fail(EINV, "geometric_factor: dim must be 2 or 3");
  const double am = dist3(a, m), an = dist3(a, n);
  if (am == 0.0 || an == 0.0 || dist3(m, n) == 0.0 ||
      (b && (dist3(b, m) == 0.0 || dist3(b, n) == 0.0 || dist3(a, b) == 0.0)))
    return fail(EINV, "geometric_factor: coincident electrodes");
  const double pi = 3.14159265358979323846;
  double denom;
  if (dim == 2) {
    denom = -log(am) + log(an);
    if (b) denom += log(dist3(b, m)) - log(dist3(b, n));
    if (fabs(denom) < 1e-14) return fail(ENUM, "geometric_factor: degenerate configuration (zero log ratio)");
    *k = pi / denom;
    return 0;
  }
  denom = 1.0 / am - 1.0 / an;
  if (b) denom += -1.0 / dist3(b, m) + 1.0 / dist3(b, n);
  if (fabs(denom) < 1e-14) return fail(ENUM, "geometric_factor: degenerate configuration (zero denominator)");
  *k = 2.0 * pi / denom;
  return 0;
}

/* Banded LU without pivoting of an SPD CSR matrix (exact solver standing in for
 * the reference's Eigen SparseLU, factorization.cpp:14-45). */
typedef struct {
  size_t n, bw;
  double* band; /* row i holds columns [i-bw, i+bw] */
} band_t;
#define BAND(f, i, j) ((f)->band[(i) * (2 * (f)->bw + 1) + ((j) + (f)->bw - (i))])

static int band_factor(const csr* A, band_t* f) {
  size_t bw = 0;
  for (size_t i = 0; i < A->n_rows; ++i)
    for (size_t k = A->rowptr[i]; k < A->rowptr[i + 1]; ++k) {
      size_t j = A->cols[k];
      size_t d = j > i ? j - i : i - j;
      if (d > bw) bw = d;
    }
  f->n = A->n_rows;
  f->bw = bw;
  f->band = xcalloc(f->n * (2 * bw + 1), sizeof(double));
  for (size_t i = 0; i < A->n_rows; ++i)
    for (size_t k = A->rowptr[i]; k < A->rowptr[i + 1]; ++k) BAND(f, i, A->cols[k]) += A->vals[k];
  for (size_t k = 0; k < f->n; ++k) {
    const double piv = BAND(f, k, k);
    if (!(fabs(piv) > 0.0)) return fail(ENUM, "sparse_factorize: numerically singular pivot");
    const size_t iend = k + bw + 1 < f->n ? k + bw + 1 : f->n;
    for (size_t i = k + 1; i < iend; ++i) {
      const double l = BAND(f, i, k) / piv;
      if (l == 0.0) continue;
      BAND(f, i, k) = l;
      for (size_t j = k + 1; j < iend; ++j) BAND(f, i, j) -= l * BAND(f, k, j);
    }
  }
  return 0;
}

static void band_solve(const band_t* f, double* x) {
  for (size_t i = 0; i < f->n; ++i) {
    const size_t j0 = i > f->bw ? i - f->bw : 0;
    double s = x[i];
    for (size_t j = j0; j < i; ++j) s -= BAND(f, i, j) * x[j];
    x[i] = s;
  }
  for (size_t ii = f->n; ii-- > 0;) {
    const size_t j1 = ii + f->bw + 1 < f->n ? ii + f->bw + 1 : f->n;
    double s = x[ii];
    for (size_t j = ii + 1; j < j1; ++j) s -= BAND(f, ii, j) * x[j];
    x[ii] = s / BAND(f, ii, ii);
  }
}

/* assemble_forward (forward.cpp:39-81), solve_unit_pole (:83-98) and
 * evaluate_response_and_jacobian (:100-172) */
int orc_response_jacobian(orc_problem* p, const int64_t* nodes, uint64_t n_nodes, const int64_t* a, const int64_t* b,
                          const int64_t* m, const int64_t* n, const double* k, uint64_t n_cfg, const double* model,
                          double* J, double* g) {
  if (!p->mixed) return fail(EINV, "orc_response_jacobian: not a mixed problem");
  const mesh_t* me = &p->mesh;
  double scale = 0.0;
  for (size_t i = 0; i < 2 * me->nv; ++i)
    if (fabs(me->v[i]) > scale) scale = fabs(me->v[i]);
  for (uint64_t e = 0; e < n_nodes; ++e)
    if (nodes[e] < 0 || (size_t)nodes[e] >= me->nv || fabs(me->v[2 * nodes[e] + 1]) > 1e-9 * scale)
      return fail(EINV, "evaluate_response_and_jacobian: survey electrode is not a mesh node");
  for (uint64_t i = 0; i < n_cfg; ++i)
    if (a[i] < 0 || (uint64_t)a[i] >= n_nodes || m[i] < 0 || (uint64_t)m[i] >= n_nodes || n[i] < 0 ||
        (uint64_t)n[i] >= n_nodes || (b[i] != -1 && (b[i] < 0 || (uint64_t)b[i] >= n_nodes)))
      return fail(EINV, "attach_electrode_positions: electrode index out of range");
  /* grounded nodes: vertices of FAR boundary edges (forward.cpp:44-56) */
  long long* n2f = xcalloc(me->nv, sizeof(long long));
  for (size_t bi = 0; bi < me->nb; ++bi)
    if (me->btag[bi] == 1) {
      n2f[me->edges[2 * me->bedge[bi]]] = -1;
      n2f[me->edges[2 * me->bedge[bi] + 1]] = -1;
    }
  size_t nf = 0;
  for (size_t v = 0; v < me->nv; ++v)
    if (n2f[v] == 0) n2f[v] = (long long)nf++;
    else n2f[v] = -1;
  /* cell geometry (forward.cpp:17-36) */
  double* area = xmalloc(me->nc * sizeof(double));
  double* grad = xmalloc(6 * me->nc * sizeof(double));
  for (size_t c = 0; c < me->nc; ++c) {
    const double* p0 = me->v + 2 * me->cells[3 * c];
    const double* p1 = me->v + 2 * me->cells[3 * c + 1];
    const double* p2 = me->v + 2 * me->cells[3 * c + 2];
    area[c] = signed_area(p0, p1, p2);
    const double inv2a = 1.0 / (2.0 * area[c]);
    double* gr = grad + 6 * c;
    gr[0] = -(p2[1] - p1[1]) * inv2a;
    gr[1] = (p2[0] - p1[0]) * inv2a;
    gr[2] = -(p0[1] - p2[1]) * inv2a;
    gr[3] = (p0[0] - p2[0]) * inv2a;
    gr[4] = -(p1[1] - p0[1]) * inv2a;
    gr[5] = (p1[0] - p0[0]) * inv2a;
  }
  /* stiffness triplets (forward.cpp:58-78) */
  triplet* t = xmalloc(9 * me->nc * sizeof(triplet));
  size_t nt = 0;
  for (size_t c = 0; c < me->nc; ++c) {
    const double sigma = exp(model[c]);
    const double* gr = grad + 6 * c;
    for (int i = 0; i < 3; ++i) {
      const long long fi = n2f[me->cells[3 * c + i]];
      if (fi < 0) continue;
      for (int j = 0; j < 3; ++j) {
        const long long fj = n2f[me->cells[3 * c + j]];
        if (fj < 0) continue;
        t[nt++] = (triplet){(size_t)fi, (size_t)fj,
                            sigma * area[c] * (gr[2 * i] * gr[2 * j] + gr[2 * i + 1] * gr[2 * j + 1])};
      }
    }
  }
  csr Kst;
  int rc = from_triplets(nf, nf, t, nt, &Kst);
  free(t);
  band_t f = {0, 0, NULL};
  if (!rc) rc = band_factor(&Kst, &f);
  csr_free(&Kst);
  /* used electrodes, pole solves and cellwise gradients (forward.cpp:115-143) */
  char* used = xcalloc(n_nodes, 1);
  for (uint64_t i = 0; i < n_cfg; ++i) {
    used[a[i]] = used[m[i]] = used[n[i]] = 1;
    if (b[i] != -1) used[b[i]] = 1;
  }
  double* gx = xcalloc(n_nodes * me->nc, sizeof(double));
  double* gz = xcalloc(n_nodes * me->nc, sizeof(double));
  double* rhs = xmalloc((nf ? nf : 1) * sizeof(double));
  double* u = xmalloc(me->nv * sizeof(double));
  for (uint64_t e = 0; e < n_nodes && !rc; ++e) {
    if (!used[e]) continue;
    const long long fr = n2f[nodes[e]];
    if (fr < 0) {
      rc = fail(EINV, "solve_unit_pole: electrode sits on the grounded boundary");
      break;
    }
    memset(rhs, 0, nf * sizeof(double));
    rhs[fr] = 1.0;
    band_solve(&f, rhs);
    for (size_t v = 0; v < me->nv; ++v) u[v] = n2f[v] >= 0 ? rhs[n2f[v]] : 0.0;
    for (size_t c = 0; c < me->nc; ++c) {
      double sx = 0.0, sz = 0.0;
      for (int i = 0; i < 3; ++i) {
        sx += u[me->cells[3 * c + i]] * grad[6 * c + 2 * i];
        sz += u[me->cells[3 * c + i]] * grad[6 * c + 2 * i + 1];
      }
      gx[e * me->nc + c] = sx;
      gz[e * me->nc + c] = sz;
    }
  }
  /* J rows and response (forward.cpp:145-171) */
  for (uint64_t i = 0; i < n_cfg && !rc; ++i) {
    double gi = 0.0;
    for (size_t c = 0; c < me->nc; ++c) {
      double tx = gx[a[i] * me->nc + c], tz = gz[a[i] * me->nc + c];
      if (b[i] != -1) {
        tx -= gx[b[i] * me->nc + c];
        tz -= gz[b[i] * me->nc + c];
      }
      const double rx = gx[m[i] * me->nc + c] - gx[n[i] * me->nc + c];
      const double rz = gz[m[i] * me->nc + c] - gz[n[i] * me->nc + c];
      const double term = k[i] * exp(model[c]) * area[c] * (tx * rx + tz * rz);
      gi += term;
      J[i * me->nc + c] = -term;
    }
    g[i] = gi;
    if (!isfinite(gi)) rc = fail(ENUM, "evaluate_response_and_jacobian: non-finite response");
  }
  free(f.band);
  free(n2f);
  free(area);
  free(grad);
  free(used);
  free(gx);
  free(gz);
  free(rhs);
  free(u);
  return rc;
}
