// spgemm.cu -- device-resident sparse building blocks of the SA-AMG setup:
// sparse_matmul (proj/src/sparse.cpp:118-154) and transpose (sparse.cpp:97-116), bit-identical
// to the host/reference code, on matrices that stay on the device (sparse_device.cuh).  The
// products are the lumped Schur complement D diag(Q)^-1 D^T (fem_mixed.cpp:84-94), the smoothing
// product A_F T and the Galerkin product P^T (A P) (amg.cpp:168-179).
//
// The reference accumulates, for every row i, the products a_ik b_kj over the entries k of
// A's row in order and, inside each, over B's row k in order, into accum[j] (reset to 0.0 at
// the first touch), then emits the row's columns sorted.  Expand-sort-compress keeps exactly
// that order:
//   expand   one record (key = (i, j), value = a_ik * b_kj) per product, written in (i, k, kb)
//            order -- the position of a product is an exclusive scan of len_B over A's nonzeros;
//   sort     a STABLE radix sort by key, so equal (i, j) keep their expansion order;
//   compress one thread per run of equal keys sums its values sequentially from 0.0.
// The host code is compiled with -ffp-contract=off and this file with --fmad=false, so each
// product and each addition rounds the same way.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "sparse_device.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {

__global__ void k_products_per_entry(const int* __restrict__ Acol, const long long* __restrict__ Brp, long long nnzA,
                                     long long* __restrict__ cnt) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nnzA) return;
  const int j = Acol[k];
  cnt[k] = Brp[j + 1] - Brp[j];
}

// row of every nonzero (for the keys)
__global__ void k_entry_rows(const long long* __restrict__ Arp, long long na, int* __restrict__ row_of) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= na) return;
  for (long long k = Arp[i]; k < Arp[i + 1]; ++k) row_of[k] = static_cast<int>(i);
}

__global__ void k_expand(const int* __restrict__ row_of, const int* __restrict__ Acol, const double* __restrict__ Aval,
                         long long nnzA, const long long* __restrict__ Brp, const int* __restrict__ Bcol,
                         const double* __restrict__ Bval, const long long* __restrict__ off, int colbits,
                         unsigned long long* __restrict__ keys, double* __restrict__ vals) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nnzA) return;
  const int j = Acol[k];
  const double a = Aval[k];
  const unsigned long long rk = static_cast<unsigned long long>(row_of[k]) << colbits;
  long long o = off[k];
  for (long long kb = Brp[j]; kb < Brp[j + 1]; ++kb, ++o) {
    keys[o] = rk | static_cast<unsigned long long>(Bcol[kb]);
    vals[o] = a * Bval[kb];
  }
}

__global__ void k_run_heads(const unsigned long long* __restrict__ keys, long long n, int* __restrict__ head) {
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  head[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

// run r covers [start, next start); its sum in order from 0.0 (accum[c] = 0.0; accum[c] += ...)
__global__ void k_compress(const unsigned long long* __restrict__ keys, const double* __restrict__ vals, long long n,
                           const int* __restrict__ head, const long long* __restrict__ run_id, int colbits,
                           unsigned long long colmask, int* __restrict__ ccol, double* __restrict__ cval,
                           long long* __restrict__ row_count) {
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n || !head[p]) return;
  const unsigned long long key = keys[p];
  double s = 0.0;
  long long q = p;
  do {
    s += vals[q];
    ++q;
  } while (q < n && keys[q] == key);
  const long long r = run_id[p];
  ccol[r] = static_cast<int>(key & colmask);
  cval[r] = s;
  atomicAdd(reinterpret_cast<unsigned long long*>(row_count + (key >> colbits)), 1ULL);
}

__global__ void k_iota(int* __restrict__ p, long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = static_cast<int>(i);
}

__global__ void k_col_hist(const int* __restrict__ col, long long nnz, long long* __restrict__ cnt) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < nnz) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + col[k]), 1ULL);
}

__global__ void k_permute_transpose(const int* __restrict__ perm, const int* __restrict__ row_of,
                                    const double* __restrict__ val, long long nnz, int* __restrict__ ocol,
                                    double* __restrict__ oval) {
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const int k = perm[p];
  ocol[p] = row_of[k];
  oval[p] = val[k];
}

inline unsigned blocks(long long n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

// stream-ordered temporaries (cudaMallocAsync pool): no device-wide sync per free
struct StreamMemory {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit StreamMemory(cudaStream_t st) : s(st) {}
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    GNW_CUDA_CHECK(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), s));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~StreamMemory() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

template <class T>
T* salloc(size_t count, cudaStream_t s) {
  void* p = nullptr;
  GNW_CUDA_CHECK(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), s));
  return static_cast<T*>(p);
}

int bits_for(long long n) {
  int b = 1;
  while ((1LL << b) < n) ++b;
  return b;
}

void exclusive_scan_ll(const long long* in, long long* out, long long n, StreamMemory& mem, cudaStream_t s) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s);
  void* tmp = mem.alloc<unsigned char>(bytes);
  cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, s);
}

// pinned double buffer shared by the transfers of a process (setup runs once per mesh)
struct PinnedStage {
  static constexpr size_t kChunk = size_t{64} << 20;
  unsigned char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  std::mutex mu;
  void ensure() {
    if (buf[0]) return;
    for (int i = 0; i < 2; ++i) {
      GNW_CUDA_CHECK(cudaMallocHost(reinterpret_cast<void**>(&buf[i]), kChunk));
      GNW_CUDA_CHECK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
  }
};
PinnedStage& stage() {
  static PinnedStage st;
  return st;
}

void par_copy(void* dst, const void* src, size_t bytes) {
  const int nt = std::max(1, std::min(omp_get_max_threads(), 8));
  if (bytes < (size_t{1} << 20) || nt == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int t = 0; t < nt; ++t) {
    const size_t a = bytes * t / nt, b = bytes * (t + 1) / nt;
    std::memcpy(static_cast<unsigned char*>(dst) + a, static_cast<const unsigned char*>(src) + a, b - a);
  }
}

}  // namespace

void dev_upload_array(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  PinnedStage& st = stage();
  std::lock_guard<std::mutex> lock(st.mu);
  st.ensure();
  int b = 0;
  bool used[2] = {false, false};
  for (size_t o = 0; o < bytes; o += PinnedStage::kChunk, b ^= 1) {
    const size_t n = std::min(PinnedStage::kChunk, bytes - o);
    if (used[b]) GNW_CUDA_CHECK(cudaEventSynchronize(st.ev[b]));
    par_copy(st.buf[b], static_cast<const unsigned char*>(src) + o, n);
    GNW_CUDA_CHECK(cudaMemcpyAsync(static_cast<unsigned char*>(dst) + o, st.buf[b], n, cudaMemcpyHostToDevice, s));
    GNW_CUDA_CHECK(cudaEventRecord(st.ev[b], s));
    used[b] = true;
  }
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
}

void dev_download_array(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  PinnedStage& st = stage();
  std::lock_guard<std::mutex> lock(st.mu);
  st.ensure();
  const size_t nchunks = (bytes + PinnedStage::kChunk - 1) / PinnedStage::kChunk;
  auto issue = [&](size_t c) {
    const size_t o = c * PinnedStage::kChunk, n = std::min(PinnedStage::kChunk, bytes - o);
    GNW_CUDA_CHECK(cudaMemcpyAsync(st.buf[c & 1], static_cast<const unsigned char*>(src) + o, n, cudaMemcpyDeviceToHost, s));
    GNW_CUDA_CHECK(cudaEventRecord(st.ev[c & 1], s));
  };
  issue(0);
  for (size_t c = 0; c < nchunks; ++c) {
    GNW_CUDA_CHECK(cudaEventSynchronize(st.ev[c & 1]));
    if (c + 1 < nchunks) issue(c + 1);  // the other buffer fills while this one is copied out
    const size_t o = c * PinnedStage::kChunk, n = std::min(PinnedStage::kChunk, bytes - o);
    par_copy(static_cast<unsigned char*>(dst) + o, st.buf[c & 1], n);
  }
}

DevCsr dev_upload(const host::Csr& A, cudaStream_t s) {
  if (A.n_rows > 0x7fffffffLL || A.n_cols > 0x7fffffffLL) throw std::invalid_argument("matrix too large for int32 indices");
  DevCsr d;
  d.s = s;
  d.n_rows = A.n_rows;
  d.n_cols = A.n_cols;
  d.nnz = A.nnz();
  d.rp = salloc<long long>(A.n_rows + 1, s);
  d.col = salloc<int>(d.nnz, s);
  d.val = salloc<double>(d.nnz, s);
  static_assert(sizeof(long long) == sizeof(int64_t), "rowptr layout");
  dev_upload_array(d.rp, A.rowptr.data(), (A.n_rows + 1) * 8, s);
  dev_upload_array(d.col, A.cols.data(), d.nnz * 4, s);
  dev_upload_array(d.val, A.vals.data(), d.nnz * 8, s);
  return d;
}

host::Csr dev_download(const DevCsr& A, cudaStream_t s) {
  host::Csr C;
  C.n_rows = A.n_rows;
  C.n_cols = A.n_cols;
  C.rowptr.resize(A.n_rows + 1);
  C.cols.resize(A.nnz);
  C.vals.resize(A.nnz);
  dev_download_array(C.rowptr.data(), A.rp, (A.n_rows + 1) * 8, s);
  dev_download_array(C.cols.data(), A.col, A.nnz * 4, s);
  dev_download_array(C.vals.data(), A.val, A.nnz * 8, s);
  return C;
}

DevCsr dev_spgemm(const DevCsr& A, const DevCsr& B, cudaStream_t s) {
  if (A.n_cols != B.n_rows) throw std::invalid_argument("sparse_matmul: dimension mismatch");
  const long long na = A.n_rows, nnzA = A.nnz;
  DevCsr C;
  C.s = s;
  C.n_rows = na;
  C.n_cols = B.n_cols;
  C.rp = salloc<long long>(na + 1, s);
  GNW_CUDA_CHECK(cudaMemsetAsync(C.rp, 0, (na + 1) * 8, s));
  if (nnzA == 0 || B.nnz == 0) return C;
  const int rowbits = bits_for(std::max<long long>(na, 2)), colbits = bits_for(std::max<long long>(B.n_cols, 2));
  if (rowbits + colbits > 64 || na > 0x7fffffffLL || B.n_cols > 0x7fffffffLL)
    throw std::invalid_argument("device_spgemm: matrix too large");
  StreamMemory mem(s);
  // product offsets: exclusive scan of len_B over A's nonzeros in CSR order = (i, k, kb) order
  long long* cnt = mem.alloc<long long>(nnzA + 1);
  long long* off = mem.alloc<long long>(nnzA + 1);
  k_products_per_entry<<<blocks(nnzA), 256, 0, s>>>(A.col, B.rp, nnzA, cnt);
  GNW_CUDA_CHECK(cudaMemsetAsync(cnt + nnzA, 0, 8, s));
  exclusive_scan_ll(cnt, off, nnzA + 1, mem, s);
  long long nprod = 0;
  GNW_CUDA_CHECK(cudaMemcpyAsync(&nprod, off + nnzA, 8, cudaMemcpyDeviceToHost, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  if (nprod == 0) return C;  // every product row empty

  int* row_of = mem.alloc<int>(nnzA);
  k_entry_rows<<<blocks(na), 256, 0, s>>>(A.rp, na, row_of);
  unsigned long long* keys = mem.alloc<unsigned long long>(nprod);
  unsigned long long* keys2 = mem.alloc<unsigned long long>(nprod);
  double* vals = mem.alloc<double>(nprod);
  double* vals2 = mem.alloc<double>(nprod);
  k_expand<<<blocks(nnzA), 256, 0, s>>>(row_of, A.col, A.val, nnzA, B.rp, B.col, B.val, off, colbits, keys, vals);
  note_launch("spgemm_expand");

  // stable sort by (row, column): equal keys keep the expansion (accumulation) order
  cub::DoubleBuffer<unsigned long long> kb(keys, keys2);
  cub::DoubleBuffer<double> vb(vals, vals2);
  size_t sort_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, kb, vb, nprod, 0, rowbits + colbits, s);
  void* stmp = mem.alloc<unsigned char>(sort_bytes);
  cub::DeviceRadixSort::SortPairs(stmp, sort_bytes, kb, vb, nprod, 0, rowbits + colbits, s);
  const unsigned long long* sk = kb.Current();
  const double* sv = vb.Current();

  int* head = mem.alloc<int>(nprod);
  long long* run_id = mem.alloc<long long>(nprod);
  k_run_heads<<<blocks(nprod), 256, 0, s>>>(sk, nprod, head);
  size_t scan2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan2, head, run_id, nprod, s);
  void* tmp2 = mem.alloc<unsigned char>(scan2);
  cub::DeviceScan::ExclusiveSum(tmp2, scan2, head, run_id, nprod, s);
  long long nnzC = 0;
  int last_head = 0;
  GNW_CUDA_CHECK(cudaMemcpyAsync(&nnzC, run_id + nprod - 1, 8, cudaMemcpyDeviceToHost, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(&last_head, head + nprod - 1, 4, cudaMemcpyDeviceToHost, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  nnzC += last_head;

  C.nnz = nnzC;
  C.col = salloc<int>(nnzC, s);
  C.val = salloc<double>(nnzC, s);
  long long* rcount = mem.alloc<long long>(na + 1);
  GNW_CUDA_CHECK(cudaMemsetAsync(rcount, 0, (na + 1) * 8, s));
  k_compress<<<blocks(nprod), 256, 0, s>>>(sk, sv, nprod, head, run_id, colbits, (1ULL << colbits) - 1, C.col, C.val,
                                           rcount);
  note_launch("spgemm_compress");
  exclusive_scan_ll(rcount, C.rp, na + 1, mem, s);
  GNW_CUDA_CHECK(cudaGetLastError());
  return C;
}

DevCsr dev_transpose(const DevCsr& A, cudaStream_t s) {
  DevCsr T;
  T.s = s;
  T.n_rows = A.n_cols;
  T.n_cols = A.n_rows;
  T.nnz = A.nnz;
  T.rp = salloc<long long>(T.n_rows + 1, s);
  T.col = salloc<int>(T.nnz, s);
  T.val = salloc<double>(T.nnz, s);
  StreamMemory mem(s);
  long long* cnt = mem.alloc<long long>(T.n_rows + 1);
  GNW_CUDA_CHECK(cudaMemsetAsync(cnt, 0, (T.n_rows + 1) * 8, s));
  if (A.nnz == 0) {
    GNW_CUDA_CHECK(cudaMemsetAsync(T.rp, 0, (T.n_rows + 1) * 8, s));
    return T;
  }
  if (A.nnz > 0x7fffffffLL) throw std::invalid_argument("device transpose: matrix too large");
  k_col_hist<<<blocks(A.nnz), 256, 0, s>>>(A.col, A.nnz, cnt);
  exclusive_scan_ll(cnt, T.rp, T.n_rows + 1, mem, s);
  // stable sort of the entry indices by column: each output row keeps ascending source rows
  int* row_of = mem.alloc<int>(A.nnz);
  k_entry_rows<<<blocks(A.n_rows), 256, 0, s>>>(A.rp, A.n_rows, row_of);
  int* keys = mem.alloc<int>(A.nnz);
  int* keys2 = mem.alloc<int>(A.nnz);
  int* idx = mem.alloc<int>(A.nnz);
  int* idx2 = mem.alloc<int>(A.nnz);
  GNW_CUDA_CHECK(cudaMemcpyAsync(keys, A.col, A.nnz * 4, cudaMemcpyDeviceToDevice, s));
  k_iota<<<blocks(A.nnz), 256, 0, s>>>(idx, A.nnz);
  cub::DoubleBuffer<int> kb(keys, keys2);
  cub::DoubleBuffer<int> vb(idx, idx2);
  size_t sort_bytes = 0;
  const int bits = bits_for(std::max<long long>(A.n_cols, 2));
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, kb, vb, A.nnz, 0, bits, s);
  void* stmp = mem.alloc<unsigned char>(sort_bytes);
  cub::DeviceRadixSort::SortPairs(stmp, sort_bytes, kb, vb, A.nnz, 0, bits, s);
  k_permute_transpose<<<blocks(A.nnz), 256, 0, s>>>(vb.Current(), row_of, A.val, A.nnz, T.col, T.val);
  note_launch("transpose_device");
  GNW_CUDA_CHECK(cudaGetLastError());
  return T;
}

host::Csr device_spgemm(const host::Csr& A, const host::Csr& B, cudaStream_t s) {
  if (A.n_cols != B.n_rows) throw std::invalid_argument("sparse_matmul: dimension mismatch");
  const DevCsr dA = dev_upload(A, s), dB = dev_upload(B, s);
  const DevCsr dC = dev_spgemm(dA, dB, s);
  return dev_download(dC, s);
}

}  // namespace gnw
