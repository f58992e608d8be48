// partition.cpp -- see partition.hpp.
#include "partition.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

namespace gnw::host {

std::vector<int32_t> owners_from_ranges(const std::vector<long long>& lo, int64_t n) {
  std::vector<int32_t> own(static_cast<size_t>(n));
  const int P = static_cast<int>(lo.size()) - 1;
  for (int r = 0; r < P; ++r)
    for (long long i = lo[r]; i < lo[r + 1]; ++i) own[static_cast<size_t>(i)] = r;
  return own;
}

std::vector<int32_t> edge_owners(const Mesh& mesh, const std::vector<int32_t>& cell_owner) {
  std::vector<int32_t> own(static_cast<size_t>(mesh.ne), -1);
  for (int64_t c = 0; c < mesh.nc; ++c)  // cells ascending: the first cell that touches an edge wins
    for (int k = 0; k < 3; ++k) {
      int32_t& o = own[static_cast<size_t>(mesh.cell_edges[3 * c + k])];
      if (o < 0) o = cell_owner[static_cast<size_t>(c)];
    }
  for (int32_t o : own)
    if (o < 0) throw std::invalid_argument("partition: edge outside every cell");
  return own;
}

std::vector<int32_t> coarse_owners(const Csr& P, const std::vector<int32_t>& fine_owner) {
  std::vector<double> best(static_cast<size_t>(P.n_cols), -1.0);
  std::vector<int32_t> own(static_cast<size_t>(P.n_cols), -1);
  for (int64_t i = 0; i < P.n_rows; ++i)  // rows ascending: ties keep the smallest fine row
    for (int64_t k = P.rowptr[i]; k < P.rowptr[i + 1]; ++k) {
      const int32_t c = P.cols[static_cast<size_t>(k)];
      const double a = std::fabs(P.vals[static_cast<size_t>(k)]);
      if (a > best[static_cast<size_t>(c)]) {
        best[static_cast<size_t>(c)] = a;
        own[static_cast<size_t>(c)] = fine_owner[static_cast<size_t>(i)];
      }
    }
  for (int32_t& o : own)
    if (o < 0) o = 0;  // an empty prolongator column (never from amg_setup): rank 0
  return own;
}

std::vector<int64_t> owned(const std::vector<int32_t>& owner, int r) {
  std::vector<int64_t> out;
  for (size_t i = 0; i < owner.size(); ++i)
    if (owner[i] == r) out.push_back(static_cast<int64_t>(i));
  return out;
}

void append_refs(const Csr& A, const std::vector<int64_t>& rows, std::vector<int64_t>& out) {
  for (int64_t i : rows)
    for (int64_t k = A.rowptr[static_cast<size_t>(i)]; k < A.rowptr[static_cast<size_t>(i) + 1]; ++k)
      out.push_back(A.cols[static_cast<size_t>(k)]);
}

std::vector<Halo> build_halos(const std::vector<int32_t>& owner, int P, const std::vector<std::vector<int64_t>>& refs,
                              int me) {
  const int64_t n = static_cast<int64_t>(owner.size());
  std::vector<Halo> h(static_cast<size_t>(P));
  std::vector<std::vector<int64_t>> own_of(static_cast<size_t>(P));
  for (int64_t i = 0; i < n; ++i) own_of[static_cast<size_t>(owner[static_cast<size_t>(i)])].push_back(i);
  std::vector<int64_t> pos(static_cast<size_t>(n));  // global -> index among its owner's entries
  for (int r = 0; r < P; ++r)
    for (size_t k = 0; k < own_of[static_cast<size_t>(r)].size(); ++k)
      pos[static_cast<size_t>(own_of[static_cast<size_t>(r)][k])] = static_cast<int64_t>(k);
  for (int r = 0; r < P; ++r) {
    Halo& H = h[static_cast<size_t>(r)];
    H.P = P;
    H.rank = r;
    H.n_global = n;
    H.own_global = own_of[static_cast<size_t>(r)];
    H.n_own = static_cast<int64_t>(H.own_global.size());
    std::vector<int64_t> g;
    for (int64_t c : refs[static_cast<size_t>(r)]) {
      if (c < 0 || c >= n) throw std::invalid_argument("partition: column out of range");
      if (owner[static_cast<size_t>(c)] != r) g.push_back(c);
    }
    std::sort(g.begin(), g.end(), [&](int64_t a, int64_t b) {
      const int32_t oa = owner[static_cast<size_t>(a)], ob = owner[static_cast<size_t>(b)];
      return oa != ob ? oa < ob : a < b;
    });
    g.erase(std::unique(g.begin(), g.end()), g.end());
    H.ghost_global = g;
    H.recv_off.assign(static_cast<size_t>(P) + 1, 0);
    for (int64_t c : g) ++H.recv_off[static_cast<size_t>(owner[static_cast<size_t>(c)]) + 1];
    for (int q = 0; q < P; ++q) H.recv_off[static_cast<size_t>(q) + 1] += H.recv_off[static_cast<size_t>(q)];
    if (r != me) continue;
    H.g2l.assign(static_cast<size_t>(n), -1);
    for (int64_t k = 0; k < H.n_own; ++k) H.g2l[static_cast<size_t>(H.own_global[static_cast<size_t>(k)])] = k;
    for (size_t k = 0; k < g.size(); ++k) H.g2l[static_cast<size_t>(g[k])] = H.n_own + static_cast<int64_t>(k);
  }
  // send lists: what rank q receives from r, in q's ghost order, as r's local indices
  for (int r = 0; r < P; ++r) {
    Halo& H = h[static_cast<size_t>(r)];
    H.send_off.assign(static_cast<size_t>(P) + 1, 0);
    for (int q = 0; q < P; ++q) {
      const Halo& Q = h[static_cast<size_t>(q)];
      for (int64_t k = Q.recv_off[static_cast<size_t>(r)]; k < Q.recv_off[static_cast<size_t>(r) + 1]; ++k)
        H.send_idx.push_back(static_cast<int32_t>(pos[static_cast<size_t>(Q.ghost_global[static_cast<size_t>(k)])]));
      H.send_off[static_cast<size_t>(q) + 1] = static_cast<int64_t>(H.send_idx.size());
    }
  }
  return h;
}

Csr localize(const Csr& A, const std::vector<int64_t>& rows, const Halo& cols, int64_t col_offset,
             int64_t local_shift) {
  Csr L;
  L.n_rows = static_cast<int64_t>(rows.size());
  L.n_cols = cols.n_local();
  L.rowptr.assign(rows.size() + 1, 0);
  for (size_t k = 0; k < rows.size(); ++k) {
    const int64_t i = rows[k];
    for (int64_t e = A.rowptr[static_cast<size_t>(i)]; e < A.rowptr[static_cast<size_t>(i) + 1]; ++e) {
      const int64_t c = cols.g2l[static_cast<size_t>(A.cols[static_cast<size_t>(e)] + col_offset)];
      if (c < 0) throw std::logic_error("partition: column without a local index");
      L.cols.push_back(static_cast<int32_t>(c - local_shift));
      L.vals.push_back(A.vals[static_cast<size_t>(e)]);
    }
    L.rowptr[k + 1] = static_cast<int64_t>(L.vals.size());
  }
  return L;
}

SaddlePartition partition_saddle(const Mesh& mesh, const Csr& Q, const Csr& D, const std::vector<long long>& cell_lo,
                                 int me) {
  const int P = static_cast<int>(cell_lo.size()) - 1;
  const int64_t K = Q.n_rows, N = D.n_rows;
  SaddlePartition sp;
  sp.cell_lo = cell_lo;
  sp.cell_owner = owners_from_ranges(cell_lo, N);
  const std::vector<int32_t> edge_own = edge_owners(mesh, sp.cell_owner);
  std::vector<int32_t> own(static_cast<size_t>(K + N));
  std::copy(edge_own.begin(), edge_own.end(), own.begin());
  std::copy(sp.cell_owner.begin(), sp.cell_owner.end(), own.begin() + K);
  const Csr Dt = transpose(D);
  std::vector<std::vector<int64_t>> refs(static_cast<size_t>(P)), my_e(static_cast<size_t>(P)),
      my_c(static_cast<size_t>(P));
  sp.edge_lo.assign(static_cast<size_t>(P) + 1, 0);
  for (int r = 0; r < P; ++r) {
    my_e[r] = owned(edge_own, r);
    my_c[r] = owned(sp.cell_owner, r);
    if (!my_e[r].empty() && my_e[r].back() - my_e[r].front() + 1 != static_cast<int64_t>(my_e[r].size()))
      throw std::logic_error("partition: own edges are not contiguous");
    sp.edge_lo[r + 1] = sp.edge_lo[r] + static_cast<long long>(my_e[r].size());
    append_refs(Q, my_e[r], refs[r]);  // Q: edge columns
    const size_t k0 = refs[r].size();
    append_refs(Dt, my_e[r], refs[r]);  // D^T: cell columns -> K + c
    for (size_t k = k0; k < refs[r].size(); ++k) refs[r][k] += K;
    append_refs(D, my_c[r], refs[r]);  // D: edge columns
  }
  std::vector<Halo> H = build_halos(own, P, refs, me);
  sp.halo = std::move(H[static_cast<size_t>(me)]);
  sp.K_l = static_cast<int64_t>(my_e[me].size());
  sp.N_l = static_cast<int64_t>(my_c[me].size());
  sp.Q = localize(Q, my_e[me], sp.halo);
  sp.D = localize(D, my_c[me], sp.halo);
  sp.Dt = localize(Dt, my_e[me], sp.halo, K, sp.K_l);
  return sp;
}

}  // namespace gnw::host
