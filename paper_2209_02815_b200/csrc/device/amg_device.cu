// amg_device.cu -- device SA-AMG hierarchy and V-cycle orchestration (amg.cpp:90-111).
#include "amg_device.cuh"
#include "minres_persistent.cuh"
#include "sparse_device.cuh"

#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unordered_map>
#include <unordered_set>

namespace gnw {

void DeviceMemory::release_all() {
  for (void* p : ptrs) cudaFree(p);
  ptrs.clear();
  bytes = 0;
}

DCsr upload_csr(DeviceMemory& mem, const host::Csr& A, cudaStream_t s) {
  DCsr d;
  if (A.nnz() > 0x7fffffffLL || A.n_rows > 0x7fffffffLL) throw std::invalid_argument("matrix too large for int32 indices");
  d.n_rows = static_cast<int>(A.n_rows);
  d.n_cols = static_cast<int>(A.n_cols);
  d.nnz = static_cast<int>(A.nnz());
  std::vector<int> rp(A.rowptr.size());
  for (size_t i = 0; i < rp.size(); ++i) rp[i] = static_cast<int>(A.rowptr[i]);
  d.rowptr = mem.alloc<int>(rp.size());
  d.cols = mem.alloc<int>(A.cols.size());
  d.vals = mem.alloc<double>(A.vals.size());
  GNW_CUDA_CHECK(cudaMemcpyAsync(d.rowptr, rp.data(), rp.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  if (A.nnz()) {
    GNW_CUDA_CHECK(cudaMemcpyAsync(d.cols, A.cols.data(), A.cols.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    GNW_CUDA_CHECK(cudaMemcpyAsync(d.vals, A.vals.data(), A.vals.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));  // host vectors are temporaries
  return d;
}

namespace {
// The distinct values of v (as bit patterns, ascending) if there are at most `cap` of them;
// empty + false otherwise.  Chunks are scanned in parallel, each bailing out early.
bool distinct_values(const std::vector<double>& v, size_t cap, std::vector<uint64_t>& out) {
  out.clear();
  const int nt = std::max(1, omp_get_max_threads());
  std::vector<std::unordered_set<uint64_t>> local(nt);
  std::vector<char> over(nt, 0);
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    const size_t a = v.size() * t / nt, b = v.size() * (t + 1) / nt;
    std::unordered_set<uint64_t>& mine = local[t];
    uint64_t last = 0;
    bool have_last = false;
    for (size_t k = a; k < b; ++k) {
      uint64_t bits;
      std::memcpy(&bits, &v[k], sizeof bits);
      if (have_last && bits == last) continue;
      last = bits;
      have_last = true;
      if (mine.insert(bits).second && mine.size() > cap) {
        over[t] = 1;
        break;
      }
    }
  }
  for (int t = 0; t < nt; ++t)
    if (over[t]) return false;
  for (int t = 0; t < nt; ++t) out.insert(out.end(), local[t].begin(), local[t].end());
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  if (out.size() > cap) {
    out.clear();
    return false;
  }
  return true;
}
}  // namespace

DSell upload_sell(DeviceMemory& mem, const host::Csr& A, cudaStream_t s, int encode) {
  DSell d;
  int64_t w = 0;
  for (int64_t r = 0; r < A.n_rows; ++r) w = std::max(w, A.rowptr[r + 1] - A.rowptr[r]);
  if (A.n_rows == 0 || w == 0 || w > kSellMaxWidth || A.n_rows > 0x7fffffffLL) return d;
  // the value encoding (common.cuh DSell): signs in the columns, or one-byte codes
  std::vector<double> table;
  std::unordered_map<uint64_t, unsigned char> code_of;  // value bits -> code
  auto bits = [](double v) {
    uint64_t b;
    std::memcpy(&b, &v, sizeof b);
    return b;
  };
  if (encode == 1)
    for (double v : A.vals)
      if (v != 1.0 && v != -1.0) encode = 2;
  if (encode == 2) {
    std::vector<uint64_t> dv;
    if (distinct_values(A.vals, 256, dv)) {
      for (uint64_t b : dv) {
        double v;
        std::memcpy(&v, &b, sizeof v);
        code_of[b] = static_cast<unsigned char>(table.size());
        table.push_back(v);
      }
    } else {
      encode = 0;
    }
  }
  const int64_t slices = (A.n_rows + 31) / 32;
  const size_t len = static_cast<size_t>(slices * 32 * w);
  std::vector<int> cols(len, -1);
  std::vector<double> vals(encode == 0 ? len : 0, 0.0);
  std::vector<unsigned char> codes(encode == 2 ? len : 0, 0);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < A.n_rows; ++r) {
    const int64_t base = (r / 32) * 32 * w + (r % 32);
    for (int64_t k = A.rowptr[r]; k < A.rowptr[r + 1]; ++k) {
      const size_t at = static_cast<size_t>(base + 32 * (k - A.rowptr[r]));
      const int c = A.cols[static_cast<size_t>(k)];
      const double v = A.vals[static_cast<size_t>(k)];
      if (encode == 1) {
        cols[at] = v == 1.0 ? c : -c - 2;
      } else if (encode == 2) {
        cols[at] = c;
        codes[at] = code_of.at(bits(v));
      } else {
        cols[at] = c;
        vals[at] = v;
      }
    }
  }
  int* dc = mem.alloc<int>(len);
  GNW_CUDA_CHECK(cudaMemcpyAsync(dc, cols.data(), len * sizeof(int), cudaMemcpyHostToDevice, s));
  if (encode == 0) {
    double* dv = mem.alloc<double>(len);
    GNW_CUDA_CHECK(cudaMemcpyAsync(dv, vals.data(), len * sizeof(double), cudaMemcpyHostToDevice, s));
    d.vals = dv;
  } else if (encode == 2) {
    unsigned char* dh = mem.alloc<unsigned char>(len);
    double* dt = mem.alloc<double>(table.size());
    GNW_CUDA_CHECK(cudaMemcpyAsync(dh, codes.data(), len, cudaMemcpyHostToDevice, s));
    GNW_CUDA_CHECK(cudaMemcpyAsync(dt, table.data(), table.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    d.codes = dh;
    d.table = dt;
  }
  d.signed_cols = encode == 1 ? 1 : 0;
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));  // host vectors are temporaries
  d.n_rows = static_cast<int>(A.n_rows);
  d.width = static_cast<int>(w);
  d.cols = dc;
  return d;
}

DLell upload_lell(DeviceMemory& mem, const host::Csr& A, int G, cudaStream_t s) {
  DLell d;
  int64_t longest = 0;
  for (int64_t r = 0; r < A.n_rows; ++r) longest = std::max(longest, A.rowptr[r + 1] - A.rowptr[r]);
  if (A.n_rows == 0 || longest == 0 || G < 1 || G > 32) return d;
  const int64_t W = (longest + G - 1) / G, rpw = 32 / G;
  const int64_t slices = ((A.n_rows + rpw - 1) / rpw + 7) / 8 * 8;  // every warp of the grid's CTAs
  const int64_t len = slices * W * 32;
  // a level whose padding would more than triple the entries keeps its CSR kernels
  if (len > 3 * A.nnz() + 8192 || len > 0x7fffffffLL) return d;
  std::unordered_map<uint64_t, unsigned> code_of;  // value bits -> code
  std::vector<double> table;
  int col_bits = 1;
  while ((int64_t{1} << col_bits) < A.n_cols) ++col_bits;
  const size_t max_codes = col_bits >= 31 ? 0 : size_t{1} << (31 - col_bits);
  {
    std::vector<uint64_t> dv;
    if (max_codes == 0 || !distinct_values(A.vals, max_codes, dv)) return d;  // too many distinct values for a 32-bit entry
    for (uint64_t b : dv) {
      double v;
      std::memcpy(&v, &b, sizeof v);
      code_of[b] = static_cast<unsigned>(table.size());
      table.push_back(v);
    }
  }
  std::vector<unsigned> words(static_cast<size_t>(len), 0xffffffffu);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < A.n_rows; ++r) {
    const int64_t base = (r / rpw) * W * 32 + (r % rpw) * G;
    for (int64_t k = A.rowptr[r]; k < A.rowptr[r + 1]; ++k) {
      const int64_t e = k - A.rowptr[r];
      const double v = A.vals[static_cast<size_t>(k)];
      uint64_t b;
      std::memcpy(&b, &v, sizeof b);
      words[static_cast<size_t>(base + (e / G) * 32 + e % G)] =
          (code_of.at(b) << col_bits) | static_cast<unsigned>(A.cols[static_cast<size_t>(k)]);
    }
  }
  unsigned* dw = mem.alloc<unsigned>(words.size());
  double* dt = mem.alloc<double>(table.size());
  GNW_CUDA_CHECK(cudaMemcpyAsync(dw, words.data(), words.size() * sizeof(unsigned), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dt, table.data(), table.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));  // host vectors are temporaries
  d.n_rows = static_cast<int>(A.n_rows);
  d.width = static_cast<int>(W);
  d.lanes = G;
  d.shift = col_bits;
  d.mask = (1u << col_bits) - 1u;
  d.words = dw;
  d.table = dt;
  return d;
}

int DeviceAmg::collapse_max() {
  static const int v = [] {
    const char* e = std::getenv("GNW_VC_COLLAPSE_MAX");
    return e ? std::atoi(e) : 3072;  // C1: level 1 (2058 rows, 34 MB) -> 0.051 -> 0.047 ms per iteration
  }();
  return v;
}

void DeviceAmg::reset() {
  bmem_.reset();
  bmem_b_ = 0;
  collapse_l_ = -1;
  collapse_M_ = nullptr;
  lv_.clear();
  mem_.release_all();
}

void DeviceAmg::upload(const host::AmgHierarchy& h, cudaStream_t s, int min_collapse_level,
                       std::vector<DevFusedOps>* fused_dev) {
  reset();
  min_collapse_ = min_collapse_level;
  const double omega = h.options.jacobi_damping;
  const size_t L = h.levels.size();
  // the dense tail starts at the collapse level (build_collapse's rule) or the coarsest level;
  // the levels above it get the fused operators (env GNW_VC_FUSED=0: the four-pass levels)
  const char* fe = std::getenv("GNW_VC_FUSED");
  const bool fused_on = !(fe && std::atoi(fe) == 0);
  int stop = static_cast<int>(L) - 1;
  for (int l = min_collapse_; l + 1 < static_cast<int>(L); ++l)
    if (h.levels[l].A.n_rows <= collapse_max()) {
      stop = l;
      break;
    }
  if (const char* e = std::getenv("GNW_VC_COLLAPSE"))
    if (std::atoi(e) == 0) stop = static_cast<int>(L) - 1;
  // Small hierarchies (candidates for the persistent MINRES kernel, minres_persistent.cu) also
  // get a SECOND, deeper dense tail: every pass of that kernel streams the tail's matrix from L2
  // (34 MB at C1's level 1), while a level of grid barriers costs ~4 us -- so its tail starts at
  // the first level with <= 640 rows (C1: level 2, 2 MB), and the levels in between get their
  // one-pass operators too.
  pstop_ = -1;
  if (fused_on && stop < static_cast<int>(L) - 1 && h.levels[0].A.n_rows <= 65536 && h.levels[stop].A.n_rows > 640)
    for (int l = stop + 1; l + 1 < static_cast<int>(L); ++l)
      if (h.levels[l].A.n_rows <= 640) {
        pstop_ = l;
        break;
      }
  const int fused_stop = pstop_ > stop ? pstop_ : stop;
  fused_ = false;
  const bool timing = [] {
    const char* e = std::getenv("GNW_SETUP_TIMING");
    return e != nullptr && std::atoi(e) != 0;
  }();
  double t_csr = 0, t_sell = 0, t_fops = 0, t_fup = 0, t_lell = 0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  vr_.assign(L, nullptr);
  ve_.assign(L, nullptr);
  vres_.assign(L, nullptr);
  vx_.assign(L, nullptr);
  for (size_t l = 0; l < L; ++l) {
    const host::AmgLevel& H = h.levels[l];
    DLevel d;
    d.n = static_cast<int>(H.A.n_rows);
    if (l + 1 < L) {
      auto ta = now();
      d.A = upload_csr(mem_, H.A, s);
      d.P = upload_csr(mem_, H.P, s);
      const host::Csr Rt = host::transpose(H.P);
      d.R = upload_csr(mem_, Rt, s);
      auto tb = now();
      t_csr += ms(ta, tb);
      if (!std::getenv("GNW_VC_CSR")) {  // experiment switch: CSR thread-per-row kernels
        d.As = upload_sell(mem_, H.A, s);
        d.Ps = upload_sell(mem_, H.P, s);
        d.Rs = upload_sell(mem_, Rt, s);
      }
      t_sell += ms(tb, now());
      d.gA = vc_group_lanes(H.A.nnz(), H.A.n_rows);
      d.gP = vc_group_lanes(H.P.nnz(), H.P.n_rows);
      d.gR = vc_group_lanes(H.P.nnz(), H.P.n_cols);
      std::vector<double> wd(H.inv_diag.size());
      for (size_t i = 0; i < wd.size(); ++i) wd[i] = omega * H.inv_diag[i];  // amg.cpp:98 (omega*inv_diag)*r
      d.wd = mem_.alloc<double>(wd.size());
      GNW_CUDA_CHECK(cudaMemcpyAsync(d.wd, wd.data(), wd.size() * sizeof(double), cudaMemcpyHostToDevice, s));
      GNW_CUDA_CHECK(cudaStreamSynchronize(s));
      if (fused_on && static_cast<int>(l) < fused_stop) {
        fused_ = true;  // levels above the dense tail (vcycle_fused.cu)
        auto tc = now();
        const char* le = std::getenv("GNW_VC_LELL");  // experiment switch: 0 keeps the CSR loops
        const bool lell_on = !(le && std::atoi(le) == 0);
        if (fused_dev != nullptr && l < fused_dev->size()) {
          // formed by the device setup (amg_setup_device.cu): adopted where they are, and their
          // lane-ELL copies are built on the device
          DevFusedOps& fd = (*fused_dev)[l];
          const long long nnz_st = fd.S.nnz + fd.T.nnz, nnz_tt = fd.Tt.nnz, rows_tt = fd.Tt.n_rows;
          d.S = adopt_csr(mem_, fd.S, s);
          d.T = adopt_csr(mem_, fd.T, s);
          d.Tt = adopt_csr(mem_, fd.Tt, s);
          d.gS = vc_group_lanes(nnz_st, d.n);
          d.gTt = vc_group_lanes(nnz_tt, rows_tt);
          auto te = now();
          t_fup += ms(tc, te);
          if (lell_on) {
            d.Sl = build_lell_device(mem_, d.S, d.gS, s);
            d.Tl = build_lell_device(mem_, d.T, d.gS, s);
            d.Ttl = build_lell_device(mem_, d.Tt, d.gTt, s);
          }
          t_lell += ms(te, now());
        } else {
          const host::FusedCycleOps f = host::fused_cycle_ops(H.A, H.P, wd);
          auto td = now();
          t_fops += ms(tc, td);
          d.S = upload_csr(mem_, f.S, s);
          d.T = upload_csr(mem_, f.T, s);
          d.Tt = upload_csr(mem_, f.Tt, s);
          d.gS = vc_group_lanes(f.S.nnz() + f.T.nnz(), f.S.n_rows);
          d.gTt = vc_group_lanes(f.Tt.nnz(), f.Tt.n_rows);
          auto te = now();
          t_fup += ms(td, te);
          if (lell_on) {
            d.Sl = upload_lell(mem_, f.S, d.gS, s);
            d.Tl = upload_lell(mem_, f.T, d.gS, s);
            d.Ttl = upload_lell(mem_, f.Tt, d.gTt, s);
          }
          t_lell += ms(te, now());
        }
        d.fused = 1;
      }
      vres_[l] = mem_.alloc<double>(d.n);
      vx_[l] = mem_.alloc<double>(d.n);
    }
    if (l > 0) {
      vr_[l] = mem_.alloc<double>(d.n);
      ve_[l] = mem_.alloc<double>(d.n);
    }
    lv_.push_back(d);
  }
  nc_ = static_cast<int>(h.nc);
  const std::vector<double> inv = host::cholesky_inverse(h.nc, h.coarse_chol);
  coarse_inv_ = mem_.alloc<double>(inv.size());
  coarse_L_ = mem_.alloc<double>(h.coarse_chol.size());
  GNW_CUDA_CHECK(cudaMemcpyAsync(coarse_inv_, inv.data(), inv.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(coarse_L_, h.coarse_chol.data(), h.coarse_chol.size() * sizeof(double),
                                 cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  auto tf = now();
  build_collapse(s);
  if (timing)
    std::fprintf(stderr,
                 "[gnw setup] device hierarchy: CSR uploads %.1f ms, SELL copies %.1f ms, fused ops (host) %.1f ms, "
                 "fused uploads %.1f ms, lane-ELL %.1f ms, collapsed tail %.1f ms\n",
                 t_csr, t_sell, t_fops, t_fup, t_lell, ms(tf, now()));
}

// Collapsed coarse tail.  Below some level the V-cycle is a small LINEAR map of that
// level's residual (Jacobi smoothing, Galerkin restriction, coarse solve, prolongation --
// amg.cpp:90-111 is linear in r), but it costs ~4 dependent launches per level.  At C2
// levels 4..9 (1147 -> 171 rows) are 21 launches; the map itself is one 1147 x 1147 matrix
// (10.5 MB, L2-resident) applied by one warp-per-row launch.  M is formed once per
// hierarchy by running the sub-cycle on the unit vectors.  Default mode only: the exact
// mode keeps the reference's level-by-level order.  Env GNW_VC_COLLAPSE=0 disables it.
double* DeviceAmg::collapse_matrix(int lc, cudaStream_t s) {
  const int n = lv_[lc].n;
  DeviceMemory tmp;
  double* I = tmp.alloc<double>(static_cast<size_t>(n) * n);
  double* MT = tmp.alloc<double>(static_cast<size_t>(n) * n);
  identity_rows(I, n, s);
  for (int j = 0; j < n; ++j)  // row j of MT = sub-cycle(e_j) = column j of M
    cycle_levels(lc, vfixed(I + static_cast<size_t>(j) * n), MT + static_cast<size_t>(j) * n, nullptr, 0, false, s);
  double* M = mem_.alloc<double>(static_cast<size_t>(n) * n);
  transpose_square(MT, M, n, s);
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  return M;
}

void DeviceAmg::build_collapse(cudaStream_t s) {
  collapse_l_ = -1;
  collapse_M_ = nullptr;
  pcollapse_M_ = nullptr;
  if (const char* e = std::getenv("GNW_VC_COLLAPSE"))
    if (std::atoi(e) == 0) {
      pstop_ = -1;
      return;
    }
  const int L = static_cast<int>(lv_.size());
  int lc = -1;
  for (int l = min_collapse_; l < L - 1; ++l)
    if (lv_[l].n <= collapse_max()) {
      lc = l;
      break;
    }
  if (lc < 0) {
    pstop_ = -1;
    return;
  }
  // collapse_l_ stays -1 while the matrices are formed: cycle_levels then runs every level
  if (pstop_ > lc) pcollapse_M_ = collapse_matrix(pstop_, s);
  collapse_M_ = collapse_matrix(lc, s);
  collapse_l_ = lc;
}

void DeviceAmg::cycle_levels(int l0, VSel r, double* out, const MinresState* st, int exact, bool collapse,
                             cudaStream_t s) {
  const int L = static_cast<int>(lv_.size());
  const int stop = (collapse && collapse_l_ >= l0) ? collapse_l_ : L - 1;
  auto at = [&](int l) { return l == l0 ? r : vfixed(vr_[l]); };
  for (int l = l0; l < stop; ++l) {
    const DLevel lev = level(l, exact);
    vc_down(lev, at(l), vres_[l], st, s);
    vc_restrict(lev, vres_[l], vr_[l + 1], s);
  }
  double* e_stop = stop == l0 ? out : ve_[stop];
  if (stop == L - 1) {
    if (exact)
      coarse_cholesky(coarse_L_, nc_, at(stop), e_stop, st, 1, 1, s);
    else
      coarse_inverse(coarse_inv_, nc_, at(stop), e_stop, st, 1, s);
  } else {
    coarse_inverse(collapse_M_, lv_[stop].n, at(stop), e_stop, st, 1, s);
  }
  for (int l = stop - 1; l >= l0; --l) {
    const DLevel lev = level(l, exact);
    vc_up1(lev, at(l), ve_[l + 1], vx_[l], st, s);
    vc_up2(lev, at(l), vx_[l], l == l0 ? out : ve_[l], st, s);
  }
}

bool DeviceAmg::fill_persist(PersistArgs& a) const {
  if (lv_.empty() || (!fused_ && lv_.size() > 1)) return false;
  const int L = static_cast<int>(lv_.size());
  const bool deep = pstop_ > 0 && pcollapse_M_ != nullptr;  // the persistent kernel's own, deeper tail
  const int stop = deep ? pstop_ : (collapse_l_ >= 0 ? collapse_l_ : L - 1);
  if (stop > kPersistMaxLevels) return false;
  for (int l = 0; l < stop; ++l) {
    const DLevel& d = lv_[l];
    if (!d.fused || !d.Sl.words || !d.Tl.words || !d.Ttl.words) return false;
    a.S[l] = d.Sl;
    a.T[l] = d.Tl;
    a.Tt[l] = d.Ttl;
    a.gS[l] = d.gS;
    a.gTt[l] = d.gTt;
  }
  for (int l = 1; l <= stop; ++l) {
    a.vr[l] = vr_[l];
    a.ve[l] = ve_[l];
  }
  a.nlev = stop;
  a.M = deep ? pcollapse_M_ : (collapse_l_ >= 0 ? collapse_M_ : coarse_inv_);
  a.nM = lv_[stop].n;
  return a.M != nullptr;
}

// Level l as launched: the reference-order (thread-per-row) kernels everywhere in
// exact mode, warp-per-row kernels on wide levels otherwise.
DLevel DeviceAmg::level(int l, int exact) const {
  DLevel d = lv_[l];
  if (exact) {
    d.gA = d.gP = d.gR = 1;
  }
  return d;
}

// amg.cpp:90-111, one symmetric V-cycle; level 0 input may be a ring slot.
void DeviceAmg::vcycle(VSel r0, double* out0, const MinresState* st, int exact, cudaStream_t s) {
  if (lv_.size() == 1) {
    if (exact)
      coarse_cholesky(coarse_L_, nc_, r0, out0, st, 1, 1, s);
    else
      coarse_inverse(coarse_inv_, nc_, r0, out0, st, 1, s);
    return;
  }
  if (!exact && fused_) {  // one pass per level each way (vcycle_fused.cu)
    const int L = static_cast<int>(lv_.size());
    const int stop = collapse_l_ >= 0 ? collapse_l_ : L - 1;
    auto at = [&](int l) { return l == 0 ? r0 : vfixed(vr_[l]); };
    for (int l = 0; l < stop; ++l) vcf_restrict(lv_[l], at(l), vr_[l + 1], st, s);
    coarse_inverse(collapse_l_ >= 0 ? collapse_M_ : coarse_inv_, lv_[stop].n, at(stop), stop == 0 ? out0 : ve_[stop],
                   st, 1, s);
    for (int l = stop - 1; l >= 0; --l) vcf_up(lv_[l], at(l), ve_[l + 1], l == 0 ? out0 : ve_[l], st, s);
    return;
  }
  cycle_levels(0, r0, out0, st, exact, !exact && collapse_l_ >= 0, s);
}

// Persistent work arrays of the batched V-cycle (b interleaved columns).
void DeviceAmg::ensure_batch(int b) {
  if (bmem_ && bmem_b_ >= b) return;
  bmem_.reset();
  bmem_ = std::make_unique<DeviceMemory>();
  const int L = static_cast<int>(lv_.size());
  mr_.assign(L, nullptr);
  me_.assign(L, nullptr);
  mres_.assign(L, nullptr);
  mx_.assign(L, nullptr);
  for (int l = 0; l < L; ++l) {
    const size_t nl = static_cast<size_t>(lv_[l].n) * b;
    if (l > 0) {
      mr_[l] = bmem_->alloc<double>(nl);
      me_[l] = bmem_->alloc<double>(nl);
    }
    if (l + 1 < L) {
      mres_[l] = bmem_->alloc<double>(nl);
      mx_[l] = bmem_->alloc<double>(nl);
    }
  }
  bR0_ = bmem_->alloc<double>(static_cast<size_t>(n()) * b);
  bX0_ = bmem_->alloc<double>(static_cast<size_t>(n()) * b);
  bmem_b_ = b;
}

// Multi-RHS V-cycle over b interleaved columns: r0/out0 are n x b.  Every level uses the
// thread-per-(row, column) kernels with the reference's sequential row sums (coalesced over
// the columns, few registers).  In exact mode that makes each column of H bit-identical to
// the reference's amg_apply; in the default mode it agrees with the loop's single-RHS cycle
// (warp-per-row on wide levels, dense collapsed tail) to rounding.  (A 32-partial emulation
// of the warp lanes kept the two bitwise equal but ran the C2 setup at 1/3 of its roofline.)
bool DeviceAmg::vcycle_batch(const double* r0, int b, double* out0, int exact, const MinresState* st_plain,
                             cudaStream_t s, double* ht, long long ldh) {
  const int L = static_cast<int>(lv_.size());
  ensure_batch(b);
  auto coarse = [&](const double* r, double* x) {
    if (exact)
      coarse_cholesky(coarse_L_, nc_, vfixed(const_cast<double*>(r)), x, st_plain, b, b, s);
    else
      mcoarse_inverse(coarse_inv_, nc_, r, x, b, s);
  };
  if (L == 1) {
    coarse(r0, out0);
    return false;
  }
  const int stop = (!exact && collapse_l_ >= 0) ? collapse_l_ : L - 1;  // as in cycle_levels
  const double* r_stop = stop == 0 ? r0 : mr_[stop];
  double* e_stop = stop == 0 ? out0 : me_[stop];
  if (!exact && fused_) {  // one pass per level each way (vcycle_fused.cu)
    for (int l = 0; l < stop; ++l) mvcf_restrict(lv_[l], l == 0 ? r0 : mr_[l], mr_[l + 1], b, s);
    if (stop == L - 1)
      coarse(r_stop, e_stop);
    else
      dense_seq_batch(collapse_M_, lv_[stop].n, r_stop, e_stop, b, s);
    bool rows = false;
    for (int l = stop - 1; l >= 0; --l)
      rows = mvcf_up(lv_[l], l == 0 ? r0 : mr_[l], me_[l + 1], l == 0 ? out0 : me_[l], b, l == 0 ? ht : nullptr,
                     ldh, s);
    return rows;
  }
  for (int l = 0; l < stop; ++l) {
    const double* rl = l == 0 ? r0 : mr_[l];
    const DLevel lev = level(l, 1);  // sequential row order on every level (see below)
    mvc_down(lev, rl, b, mres_[l], b, s);
    mvc_restrict(lev, mres_[l], mr_[l + 1], b, s);
  }
  if (stop == L - 1)
    coarse(r_stop, e_stop);
  else
    dense_seq_batch(collapse_M_, lv_[stop].n, r_stop, e_stop, b, s);
  bool to_rows = false;
  for (int l = stop - 1; l >= 0; --l) {
    const double* rl = l == 0 ? r0 : mr_[l];
    const DLevel lev = level(l, 1);
    mvc_up1(lev, rl, b, me_[l + 1], mx_[l], b, s);
    if (l == 0 && ht != nullptr && mvc2_up2_rows(lev, rl, b, mx_[l], ht, ldh, b, s))
      to_rows = true;
    else
      mvc_up2(lev, rl, b, mx_[l], l == 0 ? out0 : me_[l], b, b, s);
  }
  return to_rows;
}

}  // namespace gnw
