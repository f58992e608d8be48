// amg_setup_device.cu -- amg_setup (proj/src/amg.cpp:115-187) with every level product on the
// device.  Per level: the strength filter with weak couplings lumped into
// the diagonal (amg.cpp:141-166), the tentative prolongator (amg.cpp:70-79), the smoothing
// product A_F T, the merge P = T - A_F T (amg.cpp:168-177), P^T, A P and the Galerkin product
// P^T (A P) (amg.cpp:179) all run on device-resident matrices (sparse_device.cuh); the one-pass
// V-cycle operators T_l = P - Wd (A P), S_l = 2 Wd - Wd A Wd (host::fused_cycle_ops) reuse the
// Galerkin product's A P.  Only the greedy aggregation (amg.cpp:13-68) stays on the host: it is
// sequential by definition (hard part 1) and runs on each level's downloaded matrix
// while the device filters that level.  Every per-row loop is the host loop with one thread per
// row, so the hierarchy is bit-identical to host::amg_setup and to the reference
// (tests/test_gpu_setup.py, tests/test_hierarchy_baseline.py hashes).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "sparse_device.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {

inline unsigned blocks(long long n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

template <class T>
struct Tmp {  // one stream-ordered temporary
  T* p = nullptr;
  cudaStream_t s;
  Tmp(size_t n, cudaStream_t st) : s(st) {
    void* q = nullptr;
    GNW_CUDA_CHECK(cudaMallocAsync(&q, std::max<size_t>(n, 1) * sizeof(T), s));
    p = static_cast<T*>(q);
  }
  Tmp(const Tmp&) = delete;
  Tmp& operator=(const Tmp&) = delete;
  ~Tmp() { cudaFreeAsync(p, s); }
};

// diagonal(A), sparse.cpp:165-170: A(i, i) or 0.0
__global__ void k_diagonal(const long long* __restrict__ rp, const int* __restrict__ col, const double* __restrict__ val,
                           long long n, double* __restrict__ d) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = 0.0;
  for (long long k = rp[i]; k < rp[i + 1]; ++k)
    if (col[k] == i) {
      v = val[k];
      break;
    }
  d[i] = v;
}

// amg.cpp:141-166 + inverse_diagonal(F) * prolongation_damping + scale_rows: out = diag-scaled A_F
__global__ void k_filter_scale(const long long* __restrict__ rp, const int* __restrict__ col,
                               const double* __restrict__ val, const double* __restrict__ diag, long long n,
                               double strength, double damping, double* __restrict__ out, int* __restrict__ bad) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long k0 = rp[i], k1 = rp[i + 1];
  double lumped = 0.0;
  long long kd = -1;
  for (long long k = k0; k < k1; ++k) {
    const int j = col[k];
    double v = val[k];
    if (j == i) {
      if (kd < 0) kd = k;
    } else if (fabs(v) <= strength * sqrt(fabs(diag[i] * diag[j]))) {
      lumped += v;
      v = 0.0;
    }
    out[k] = v;
  }
  double fd = 0.0;
  if (kd >= 0) {
    fd = val[kd] + lumped;
    out[kd] = fd;
  }
  if (!(fd > 0.0)) {  // inverse_diagonal: "amg_setup: non-positive diagonal entry"
    *bad = 1;
    return;
  }
  double sc = 1.0 / fd;
  sc *= damping;
  for (long long k = k0; k < k1; ++k) out[k] = out[k] * sc;
}

// tentative prolongator, amg.cpp:70-79
__global__ void k_tentative(const int* __restrict__ agg, const long long* __restrict__ count, long long n,
                            long long* __restrict__ rp, int* __restrict__ col, double* __restrict__ val) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i > n) return;
  rp[i] = i;
  if (i == n) return;
  const int a = agg[i];
  col[i] = a;
  val[i] = 1.0 / sqrt(static_cast<double>(count[a]));
}

// P = T - AT (amg.cpp:168-177): row lengths, then the merged rows
__global__ void k_pmerge_len(const int* __restrict__ tcol, const long long* __restrict__ arp,
                             const int* __restrict__ acol, long long n, long long* __restrict__ len) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {
    len[i] = 0;
    return;
  }
  const int tc = tcol[i];
  bool hit = false;
  for (long long k = arp[i]; k < arp[i + 1]; ++k) hit |= (acol[k] == tc);
  len[i] = (arp[i + 1] - arp[i]) + (hit ? 0 : 1);
}
__global__ void k_pmerge_fill(const int* __restrict__ tcol, const double* __restrict__ tval,
                              const long long* __restrict__ arp, const int* __restrict__ acol,
                              const double* __restrict__ aval, long long n, const long long* __restrict__ prp,
                              int* __restrict__ pcol, double* __restrict__ pval) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int tc = tcol[i];
  const double tv = tval[i];
  long long out = prp[i];
  bool done = false;
  for (long long k = arp[i]; k < arp[i + 1]; ++k) {
    const int c = acol[k];
    if (!done && tc < c) {
      pcol[out] = tc;
      pval[out++] = 0.0 + tv;
      done = true;
    }
    if (c == tc) {
      double v = 0.0;
      v += tv;
      v += -aval[k];
      pcol[out] = c;
      pval[out++] = v;
      done = true;
    } else {
      pcol[out] = c;
      pval[out++] = 0.0 + -aval[k];
    }
  }
  if (!done) {
    pcol[out] = tc;
    pval[out++] = 0.0 + tv;
  }
}

// host::fused_cycle_ops: S = 2 Wd - Wd A Wd on A's pattern
__global__ void k_fused_s(const long long* __restrict__ rp, const int* __restrict__ col, const double* __restrict__ val,
                          const double* __restrict__ wd, long long n, double* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (long long k = rp[i]; k < rp[i + 1]; ++k) {
    const int j = col[k];
    const double v = -(wd[i] * val[k] * wd[j]);
    out[k] = (i == j) ? 2.0 * wd[i] + v : v;
  }
}
// T = P - Wd (A P): union of the two sorted column lists per row
__global__ void k_fused_t_len(const long long* __restrict__ prp, const int* __restrict__ pcol,
                              const long long* __restrict__ qrp, const int* __restrict__ qcol, long long n,
                              long long* __restrict__ len) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {
    len[i] = 0;
    return;
  }
  long long a = prp[i], b = qrp[i], c = 0;
  const long long a1 = prp[i + 1], b1 = qrp[i + 1];
  while (a < a1 || b < b1) {
    const int ca = a < a1 ? pcol[a] : 0x7fffffff;
    const int cb = b < b1 ? qcol[b] : 0x7fffffff;
    if (ca <= cb) ++a;
    if (cb <= ca) ++b;
    ++c;
  }
  len[i] = c;
}
__global__ void k_fused_t_fill(const long long* __restrict__ prp, const int* __restrict__ pcol,
                               const double* __restrict__ pval, const long long* __restrict__ qrp,
                               const int* __restrict__ qcol, const double* __restrict__ qval,
                               const double* __restrict__ wd, long long n, const long long* __restrict__ trp,
                               int* __restrict__ tcol, double* __restrict__ tval) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long a = prp[i], b = qrp[i], o = trp[i];
  const long long a1 = prp[i + 1], b1 = qrp[i + 1];
  while (a < a1 || b < b1) {
    const int ca = a < a1 ? pcol[a] : 0x7fffffff;
    const int cb = b < b1 ? qcol[b] : 0x7fffffff;
    double v = 0.0;
    if (ca <= cb) v = pval[a++];
    if (cb <= ca) v = v - wd[i] * qval[b++];
    tcol[o] = ca < cb ? ca : cb;
    tval[o++] = v;
  }
}

__global__ void k_scale_rows(const long long* __restrict__ rp, double* __restrict__ val, const double* __restrict__ sc,
                             long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (long long k = rp[i]; k < rp[i + 1]; ++k) val[k] *= sc[i];
}


__global__ void k_rowptr_to_int(const long long* __restrict__ in, long long n1, int* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n1) out[i] = static_cast<int>(in[i]);
}

__global__ void k_longest_row(const int* __restrict__ rp, int n, int* __restrict__ longest) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicMax(longest, rp[i + 1] - rp[i]);
}

__global__ void k_value_bits(const double* __restrict__ val, long long nnz, unsigned long long* __restrict__ bits) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < nnz) bits[k] = static_cast<unsigned long long>(__double_as_longlong(val[k]));
}

// lane-ELL words of one row per thread (common.cuh DLell): code = rank of the value's bits
__global__ void k_lell_fill(const int* __restrict__ rp, const int* __restrict__ col, const double* __restrict__ val,
                            int n, int G, int W, int shift, const unsigned long long* __restrict__ table, int ntab,
                            unsigned* __restrict__ words) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int rpw = 32 / G;
  const long long base = static_cast<long long>(r / rpw) * W * 32 + (r % rpw) * G;
  const int k0 = rp[r];
  for (int k = k0; k < rp[r + 1]; ++k) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(val[k]));
    int lo = 0, hi = ntab - 1;  // the value is in the table
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (table[mid] < b)
        lo = mid + 1;
      else
        hi = mid;
    }
    const int e = k - k0;
    words[base + static_cast<long long>(e / G) * 32 + e % G] =
        (static_cast<unsigned>(lo) << shift) | static_cast<unsigned>(col[k]);
  }
}

void scan_ll(const long long* in, long long* out, long long n, cudaStream_t s) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s);
  Tmp<unsigned char> tmp(bytes, s);
  cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, s);
}

template <class T>
T* salloc(size_t count, cudaStream_t s) {
  void* p = nullptr;
  GNW_CUDA_CHECK(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), s));
  return static_cast<T*>(p);
}

long long read_ll(const long long* p, cudaStream_t s) {
  long long v = 0;
  GNW_CUDA_CHECK(cudaMemcpyAsync(&v, p, 8, cudaMemcpyDeviceToHost, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  return v;
}

// keep freed stream-ordered blocks in the pool across the setup's syncs (the default threshold
// of 0 returns them to the driver at every synchronisation)
void keep_pool(cudaStream_t) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  unsigned long long thr = ~0ULL;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}
void trim_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  cudaMemPoolTrimTo(pool, 0);
}

struct Lap {
  bool on;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  Lap(cudaStream_t st) : s(st) {
    const char* e = std::getenv("GNW_SETUP_TIMING");
    on = e != nullptr && std::atoi(e) != 0;
  }
  void operator()(const char* what, long long level) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gnw setup/device] %-26s level %2lld  %8.1f ms\n", what, level,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

}  // namespace


DCsr adopt_csr(DeviceMemory& mem, DevCsr& A, cudaStream_t s) {
  if (A.nnz > 0x7fffffffLL || A.n_rows > 0x7fffffffLL) throw std::invalid_argument("matrix too large for int32 indices");
  DCsr d;
  d.n_rows = static_cast<int>(A.n_rows);
  d.n_cols = static_cast<int>(A.n_cols);
  d.nnz = static_cast<int>(A.nnz);
  d.rowptr = mem.alloc<int>(A.n_rows + 1);
  k_rowptr_to_int<<<blocks(A.n_rows + 1), 256, 0, s>>>(A.rp, A.n_rows + 1, d.rowptr);
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  // the column and value arrays change owner (cudaFree accepts stream-ordered allocations)
  d.cols = A.col;
  d.vals = A.val;
  if (A.col) mem.ptrs.push_back(A.col);
  if (A.val) mem.ptrs.push_back(A.val);
  mem.bytes += static_cast<size_t>(A.nnz) * 12;
  A.col = nullptr;
  A.val = nullptr;
  A.release();
  A.nnz = 0;
  return d;
}

DLell build_lell_device(DeviceMemory& mem, const DCsr& A, int G, cudaStream_t s) {
  DLell d;
  if (A.n_rows == 0 || A.nnz == 0 || G < 1 || G > 32) return d;
  Tmp<int> dl(1, s);
  GNW_CUDA_CHECK(cudaMemsetAsync(dl.p, 0, 4, s));
  k_longest_row<<<blocks(A.n_rows), 256, 0, s>>>(A.rowptr, A.n_rows, dl.p);
  int longest = 0;
  GNW_CUDA_CHECK(cudaMemcpyAsync(&longest, dl.p, 4, cudaMemcpyDeviceToHost, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  if (longest == 0) return d;
  const long long W = (longest + G - 1) / G, rpw = 32 / G;
  const long long slices = ((A.n_rows + rpw - 1) / rpw + 7) / 8 * 8;
  const long long len = slices * W * 32;
  if (len > 3LL * A.nnz + 8192 || len > 0x7fffffffLL) return d;
  int col_bits = 1;
  while ((1LL << col_bits) < A.n_cols) ++col_bits;
  const long long max_codes = col_bits >= 31 ? 0 : 1LL << (31 - col_bits);
  // the distinct values: sort the bit patterns, keep one of each
  Tmp<unsigned long long> bits(A.nnz, s), sorted(A.nnz, s), uniq(A.nnz, s);
  Tmp<long long> nuniq(1, s);
  k_value_bits<<<blocks(A.nnz), 256, 0, s>>>(A.vals, A.nnz, bits.p);
  {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, bits.p, sorted.p, static_cast<long long>(A.nnz), 0, 64, s);
    Tmp<unsigned char> tmp(bytes, s);
    cub::DeviceRadixSort::SortKeys(tmp.p, bytes, bits.p, sorted.p, static_cast<long long>(A.nnz), 0, 64, s);
  }
  {
    size_t bytes = 0;
    cub::DeviceSelect::Unique(nullptr, bytes, sorted.p, uniq.p, nuniq.p, static_cast<long long>(A.nnz), s);
    Tmp<unsigned char> tmp(bytes, s);
    cub::DeviceSelect::Unique(tmp.p, bytes, sorted.p, uniq.p, nuniq.p, static_cast<long long>(A.nnz), s);
  }
  const long long ntab = read_ll(nuniq.p, s);
  if (ntab > max_codes) return d;  // too many distinct values for a 32-bit entry
  unsigned* words = mem.alloc<unsigned>(static_cast<size_t>(len));
  double* table = mem.alloc<double>(static_cast<size_t>(ntab));
  GNW_CUDA_CHECK(cudaMemsetAsync(words, 0xff, static_cast<size_t>(len) * 4, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(table, uniq.p, ntab * 8, cudaMemcpyDeviceToDevice, s));
  k_lell_fill<<<blocks(A.n_rows), 256, 0, s>>>(A.rowptr, A.cols, A.vals, A.n_rows, G, static_cast<int>(W), col_bits,
                                               uniq.p, static_cast<int>(ntab), words);
  note_launch("lell_fill");
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  d.n_rows = A.n_rows;
  d.width = static_cast<int>(W);
  d.lanes = G;
  d.shift = col_bits;
  d.mask = (1u << col_bits) - 1u;
  d.words = words;
  d.table = table;
  return d;
}

void device_setup_trim() {
  cudaDeviceSynchronize();
  trim_pool();
}

host::Csr device_lumped_schur(const host::Csr& Q, const host::Csr& D, cudaStream_t s) {
  if (Q.n_rows != Q.n_cols || D.n_cols != Q.n_rows)
    throw std::invalid_argument("assemble_lumped_schur: shape mismatch");
  keep_pool(s);
  std::vector<double> inv = host::diagonal(Q);
  for (double& v : inv) {
    if (!(v > 0.0)) throw std::runtime_error("assemble_lumped_schur: zero diagonal in Q (degenerate cell)");
    v = 1.0 / v;
  }
  const DevCsr dD = dev_upload(D, s);
  DevCsr dDt = dev_transpose(dD, s);
  Tmp<double> dinv(inv.size(), s);
  dev_upload_array(dinv.p, inv.data(), inv.size() * 8, s);
  k_scale_rows<<<blocks(dDt.n_rows), 256, 0, s>>>(dDt.rp, dDt.val, dinv.p, dDt.n_rows);
  const DevCsr dS = dev_spgemm(dD, dDt, s);
  return dev_download(dS, s);
}

host::AmgHierarchy device_amg_setup(const host::Csr& S, const host::AmgOptions& o, cudaStream_t s,
                                    std::vector<DevFusedOps>* fused, int collapse_max) {
  const long long host_rows = [] {
    const char* e = std::getenv("GNW_DEVICE_SETUP_MIN_ROWS");
    return e ? std::atoll(e) : 100000LL;
  }();
  Lap lap(s);
  keep_pool(s);
  if (S.n_rows != S.n_cols) throw std::invalid_argument("amg_setup: matrix not square");
  double max_abs = 0.0;
  for (double v : S.vals) max_abs = std::max(max_abs, std::abs(v));
  if (host::symmetry_error(S) > 1e-12 * std::max(max_abs, 1.0))
    throw std::invalid_argument("amg_setup: matrix not symmetric");
  host::AmgHierarchy h;
  h.options = o;
  if (fused) fused->clear();
  host::Csr cur = S;  // the host copy: aggregation input and the hierarchy's level matrix
  DevCsr dcur = dev_upload(cur, s);
  lap("symmetry check + upload", 0);
  Tmp<int> bad(1, s);
  GNW_CUDA_CHECK(cudaMemsetAsync(bad.p, 0, 4, s));
  bool fused_more = fused != nullptr;
  while (static_cast<int64_t>(h.levels.size()) + 1 < o.max_levels && cur.n_rows > o.coarse_threshold) {
    const long long lev = static_cast<long long>(h.levels.size());
    const long long n = cur.n_rows;
    if (n <= host_rows) {  // the remaining (small) levels on the host, appended as they are
      host::AmgOptions rest = o;
      rest.max_levels = o.max_levels - static_cast<int64_t>(h.levels.size());
      host::AmgHierarchy tail = host::amg_setup(cur, rest, false);
      for (auto& L : tail.levels) h.levels.push_back(std::move(L));
      h.coarse_chol = std::move(tail.coarse_chol);
      h.nc = tail.nc;
      lap("remaining levels (host)", lev);
      return h;
    }
    // the fused one-pass operators exist on the levels above the dense collapsed tail
    // (DeviceAmg::upload's rule: the tail starts at the first level >= 1 with <= collapse_max rows)
    if (lev >= 1 && n <= collapse_max) fused_more = false;
    // device: diag(A), filtered + scaled A_F (independent of the aggregation)
    Tmp<double> diag(n, s);
    k_diagonal<<<blocks(n), 256, 0, s>>>(dcur.rp, dcur.col, dcur.val, n, diag.p);
    DevCsr AF;
    AF.s = s;
    AF.n_rows = AF.n_cols = n;
    AF.nnz = dcur.nnz;
    AF.rp = salloc<long long>(n + 1, s);
    AF.col = salloc<int>(dcur.nnz, s);
    AF.val = salloc<double>(dcur.nnz, s);
    GNW_CUDA_CHECK(cudaMemcpyAsync(AF.rp, dcur.rp, (n + 1) * 8, cudaMemcpyDeviceToDevice, s));
    GNW_CUDA_CHECK(cudaMemcpyAsync(AF.col, dcur.col, dcur.nnz * 4, cudaMemcpyDeviceToDevice, s));
    k_filter_scale<<<blocks(n), 256, 0, s>>>(dcur.rp, dcur.col, dcur.val, diag.p, n, o.strength,
                                             o.prolongation_damping, AF.val, bad.p);
    note_launch("amg_filter_scale");
    // host, meanwhile: the sequential greedy aggregation
    int64_t n_agg = 0;
    const std::vector<int64_t> agg = host::aggregate(cur, o, n_agg);
    lap("aggregate (host) | filter", lev);
    if (n_agg >= cur.n_rows) break;
    std::vector<double> inv_diag = host::inverse_diagonal(cur);  // throws on a non-positive diagonal
    std::vector<long long> count(n_agg, 0);
    std::vector<int> agg32(n);
    for (long long i = 0; i < n; ++i) {
      ++count[agg[i]];
      agg32[i] = static_cast<int>(agg[i]);
    }
    Tmp<int> dagg(n, s);
    Tmp<long long> dcount(n_agg, s);
    dev_upload_array(dagg.p, agg32.data(), n * 4, s);
    dev_upload_array(dcount.p, count.data(), n_agg * 8, s);
    int hbad = 0;
    GNW_CUDA_CHECK(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, s));
    GNW_CUDA_CHECK(cudaStreamSynchronize(s));
    if (hbad) throw std::invalid_argument("amg_setup: non-positive diagonal entry");
    DevCsr T;
    T.s = s;
    T.n_rows = n;
    T.n_cols = n_agg;
    T.nnz = n;
    T.rp = salloc<long long>(n + 1, s);
    T.col = salloc<int>(n, s);
    T.val = salloc<double>(n, s);
    k_tentative<<<blocks(n + 1), 256, 0, s>>>(dagg.p, dcount.p, n, T.rp, T.col, T.val);
    DevCsr AT = dev_spgemm(AF, T, s);
    AF.release();
    lap("tentative + A_F T", lev);
    DevCsr P;
    P.s = s;
    P.n_rows = n;
    P.n_cols = n_agg;
    P.rp = salloc<long long>(n + 1, s);
    {
      Tmp<long long> len(n + 1, s);
      k_pmerge_len<<<blocks(n + 1), 256, 0, s>>>(T.col, AT.rp, AT.col, n, len.p);
      scan_ll(len.p, P.rp, n + 1, s);
      P.nnz = read_ll(P.rp + n, s);
      P.col = salloc<int>(P.nnz, s);
      P.val = salloc<double>(P.nnz, s);
      k_pmerge_fill<<<blocks(n), 256, 0, s>>>(T.col, T.val, AT.rp, AT.col, AT.val, n, P.rp, P.col, P.val);
      note_launch("amg_pmerge");
    }
    AT.release();
    T.release();
    lap("P merge", lev);
    DevCsr Pt = dev_transpose(P, s);
    DevCsr AP = dev_spgemm(dcur, P, s);
    DevCsr coarse = dev_spgemm(Pt, AP, s);  // Galerkin, amg.cpp:179
    Pt.release();
    lap("galerkin P^T (A P)", lev);
    host::Csr hP = dev_download(P, s);
    if (fused_more) {
      DevFusedOps f;
      std::vector<double> wd(n);
      for (long long i = 0; i < n; ++i) wd[i] = o.jacobi_damping * inv_diag[i];  // amg.cpp:98
      Tmp<double> dwd(n, s);
      dev_upload_array(dwd.p, wd.data(), n * 8, s);
      // S = 2 Wd - Wd A Wd on A's pattern
      f.S.s = s;
      f.S.n_rows = f.S.n_cols = n;
      f.S.nnz = dcur.nnz;
      f.S.rp = salloc<long long>(n + 1, s);
      f.S.col = salloc<int>(dcur.nnz, s);
      f.S.val = salloc<double>(dcur.nnz, s);
      GNW_CUDA_CHECK(cudaMemcpyAsync(f.S.rp, dcur.rp, (n + 1) * 8, cudaMemcpyDeviceToDevice, s));
      GNW_CUDA_CHECK(cudaMemcpyAsync(f.S.col, dcur.col, dcur.nnz * 4, cudaMemcpyDeviceToDevice, s));
      k_fused_s<<<blocks(n), 256, 0, s>>>(dcur.rp, dcur.col, dcur.val, dwd.p, n, f.S.val);
      f.T.s = s;
      f.T.n_rows = n;
      f.T.n_cols = n_agg;
      f.T.rp = salloc<long long>(n + 1, s);
      {
        Tmp<long long> len(n + 1, s);
        k_fused_t_len<<<blocks(n + 1), 256, 0, s>>>(P.rp, P.col, AP.rp, AP.col, n, len.p);
        scan_ll(len.p, f.T.rp, n + 1, s);
        f.T.nnz = read_ll(f.T.rp + n, s);
        f.T.col = salloc<int>(f.T.nnz, s);
        f.T.val = salloc<double>(f.T.nnz, s);
        k_fused_t_fill<<<blocks(n), 256, 0, s>>>(P.rp, P.col, P.val, AP.rp, AP.col, AP.val, dwd.p, n, f.T.rp, f.T.col,
                                                 f.T.val);
        note_launch("amg_fused_t");
      }
      f.Tt = dev_transpose(f.T, s);
      fused->push_back(std::move(f));
      lap("fused S, T, T^T (device)", lev);
    }
    AP.release();
    P.release();
    host::Csr hcoarse = dev_download(coarse, s);
    lap("download P, A_coarse", lev);
    h.levels.push_back({std::move(cur), std::move(hP), std::move(inv_diag)});
    cur = std::move(hcoarse);
    dcur = std::move(coarse);
  }
  std::vector<double> inv_last = host::inverse_diagonal(cur);
  const int64_t nc = cur.n_rows;
  std::vector<double> dense(nc * nc, 0.0);
  for (int64_t i = 0; i < nc; ++i)
    for (int64_t k = cur.rowptr[i]; k < cur.rowptr[i + 1]; ++k) dense[i * nc + cur.cols[k]] += cur.vals[k];
  h.levels.push_back({std::move(cur), host::Csr{}, std::move(inv_last)});
  h.coarse_chol = host::dense_cholesky(nc, dense);
  h.nc = nc;
  lap("coarse cholesky (host)", static_cast<long long>(h.levels.size()) - 1);
  GNW_CUDA_CHECK(cudaGetLastError());
  return h;
}

}  // namespace gnw
