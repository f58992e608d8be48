// partition.hpp -- host-side row partition of the GN-step solve over P ranks (SURVEY.md 8(e):
// "MINRES vectors by mesh rows with halo exchange").
//
// Every rank runs the same (replicated, deterministic) host setup, so every rank can derive
// every other rank's partition and halo lists without communicating.
//
// A partitioned vector space (the saddle unknowns [edges; cells], or one AMG level) gives each
// global index one owning rank.  On its owner the entry lives at a LOCAL index: the owned
// entries first, in ascending global order, then the ghosts (entries owned elsewhere that the
// rank's rows read), grouped by owning rank.  A halo exchange sends every rank the current
// values of its ghosts; a local matrix is the rank's owned rows with their columns mapped to
// local indices, entry order unchanged, so each row sums the same terms in the same order as
// the global matrix (bit-identical rows).
//
// Ownership:
//   cells   contiguous ranges of the cell numbering (partition_cells: multiples of 64 cells,
//           i.e. whole mesh rows of a unit-square mesh for 2n | 64 k);
//   edges   the owner of the first cell that contains the edge -- edges are numbered by first
//           encounter in cell order (mesh.cpp:116-137), so these are contiguous ranges too;
//   AMG level l+1: the owner of the fine row holding the largest |P_l(i, c)| of coarse column c
//           (the aggregate's own rows dominate its smoothed prolongator column).
#pragma once

#include <cstdint>
#include <vector>

#include "setup.hpp"

namespace gnw::host {

struct Halo {
  int P = 1, rank = 0;
  int64_t n_global = 0, n_own = 0;
  std::vector<int64_t> own_global;    // local k < n_own -> global index (ascending)
  std::vector<int64_t> ghost_global;  // local n_own + k -> global, grouped by owner rank
  std::vector<int64_t> recv_off;      // P + 1: ghosts owned by rank q at [recv_off[q], recv_off[q+1])
  std::vector<int32_t> send_idx;      // local (owned) indices other ranks read, grouped by destination
  std::vector<int64_t> send_off;      // P + 1
  std::vector<int64_t> g2l;           // global -> local (-1: neither owned nor a ghost)
  int64_t n_local() const { return n_own + static_cast<int64_t>(ghost_global.size()); }
};

// Halos of every rank of one space: refs[r] = global indices read by rank r's rows (any order,
// duplicates allowed).  Owned indices in refs are ignored.  Only rank `me` gets its g2l map.
std::vector<Halo> build_halos(const std::vector<int32_t>& owner, int P, const std::vector<std::vector<int64_t>>& refs,
                              int me);

// Rank r's rows of A (global rows `rows`, in that order) with column j mapped to
// cols.g2l[j + col_offset] - local_shift (a referenced column without a local index throws).
// The offsets place a block of a combined space: D^T's cell columns live at K + c of the saddle
// space, and the kernels add the local edge count back (x[K_r + col]).
Csr localize(const Csr& A, const std::vector<int64_t>& rows, const Halo& cols, int64_t col_offset = 0,
             int64_t local_shift = 0);

// Column references of the given rows of A (for build_halos).
void append_refs(const Csr& A, const std::vector<int64_t>& rows, std::vector<int64_t>& out);

// Owners of the cells (contiguous, partition_cells), edges (first containing cell) and of
// AMG level l+1 from P_l and the owners of level l.
std::vector<int32_t> owners_from_ranges(const std::vector<long long>& lo, int64_t n);
std::vector<int32_t> edge_owners(const Mesh& mesh, const std::vector<int32_t>& cell_owner);
std::vector<int32_t> coarse_owners(const Csr& P, const std::vector<int32_t>& fine_owner);

// Owned global indices of rank r, ascending.
std::vector<int64_t> owned(const std::vector<int32_t>& owner, int r);

// Rank `me`'s part of the saddle system [[Q, D^T], [D, 0]] on P ranks: the halo of the combined
// space (edge e -> e, cell c -> K + c) and the local operators.  Local layout
// [own edges (K_l) | own cells (N_l) | ghosts]; Dt's columns are stored minus K_l (the kernels
// address cell columns as x[K_l + col]).
struct SaddlePartition {
  std::vector<long long> cell_lo, edge_lo;  // P + 1 contiguous ranges
  std::vector<int32_t> cell_owner;
  Halo halo;
  Csr Q, D, Dt;
  int64_t K_l = 0, N_l = 0;
};
SaddlePartition partition_saddle(const Mesh& mesh, const Csr& Q, const Csr& D, const std::vector<long long>& cell_lo,
                                 int me);

}  // namespace gnw::host
