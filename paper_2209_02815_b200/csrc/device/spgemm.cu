// spgemm.cu -- sparse_matmul (proj/src/sparse.cpp:118-154) on the device, bit-identical to the
// host/reference product, for the SA-AMG setup: the lumped Schur
// complement D diag(Q)^-1 D^T (fem_mixed.cpp:84-94), the smoothing product A_F T and the
// Galerkin product P^T (A P) (amg.cpp:168-179).  Those products were 70-85 % of the host setup.
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

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <vector>

#include "amg_device.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {

__global__ void k_products_per_entry(const long long* __restrict__ Arp, const int* __restrict__ Acol, long long na,
                                     const long long* __restrict__ Brp, long long nnzA, long long* __restrict__ cnt) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nnzA) return;
  const int j = Acol[k];
  cnt[k] = Brp[j + 1] - Brp[j];
}

// row of every A nonzero (for the key)
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

int bits_for(long long n) {
  int b = 1;
  while ((1LL << b) < n) ++b;
  return b;
}

}  // namespace

host::Csr device_spgemm(const host::Csr& A, const host::Csr& B, cudaStream_t s) {
  if (A.n_cols != B.n_rows) throw std::invalid_argument("sparse_matmul: dimension mismatch");
  host::Csr C;
  C.n_rows = A.n_rows;
  C.n_cols = B.n_cols;
  const long long na = A.n_rows, nnzA = A.nnz();
  C.rowptr.assign(na + 1, 0);
  if (nnzA == 0 || B.nnz() == 0) return C;
  const int rowbits = bits_for(std::max<long long>(na, 2)), colbits = bits_for(std::max<long long>(B.n_cols, 2));
  if (rowbits + colbits > 64 || na > 0x7fffffffLL || B.n_cols > 0x7fffffffLL)
    throw std::invalid_argument("device_spgemm: matrix too large");
  const bool timing = [] {
    const char* e = std::getenv("GNW_SETUP_TIMING");
    return e != nullptr && std::atoi(e) != 0;
  }();
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    GNW_CUDA_CHECK(cudaStreamSynchronize(s));
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gnw setup]   device spgemm %-10s %8.1f ms (%lld x %lld, nnz %lld)\n", what,
                 std::chrono::duration<double, std::milli>(t1 - tp).count(), static_cast<long long>(A.n_rows),
                 static_cast<long long>(B.n_cols), static_cast<long long>(A.nnz()));
    tp = t1;
  };
  StreamMemory mem(s);
  long long* dArp = mem.alloc<long long>(na + 1);
  int* dAcol = mem.alloc<int>(nnzA);
  double* dAval = mem.alloc<double>(nnzA);
  long long* dBrp = mem.alloc<long long>(B.n_rows + 1);
  int* dBcol = mem.alloc<int>(B.nnz());
  double* dBval = mem.alloc<double>(B.nnz());
  static_assert(sizeof(long long) == sizeof(int64_t), "rowptr layout");
  GNW_CUDA_CHECK(cudaMemcpyAsync(dArp, A.rowptr.data(), (na + 1) * 8, cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dAcol, A.cols.data(), nnzA * 4, cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dAval, A.vals.data(), nnzA * 8, cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dBrp, B.rowptr.data(), (B.n_rows + 1) * 8, cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dBcol, B.cols.data(), B.nnz() * 4, cudaMemcpyHostToDevice, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(dBval, B.vals.data(), B.nnz() * 8, cudaMemcpyHostToDevice, s));

  lap("upload");
  // product offsets: exclusive scan of len_B over A's nonzeros in CSR order = (i, k, kb) order
  long long* cnt = mem.alloc<long long>(nnzA + 1);
  long long* off = mem.alloc<long long>(nnzA + 1);
  k_products_per_entry<<<blocks(nnzA), 256, 0, s>>>(dArp, dAcol, na, dBrp, nnzA, cnt);
  GNW_CUDA_CHECK(cudaMemsetAsync(cnt + nnzA, 0, 8, s));
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off, nnzA + 1, s);
  void* tmp = mem.alloc<unsigned char>(tmp_bytes);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, nnzA + 1, s);
  long long nprod = 0;
  GNW_CUDA_CHECK(cudaMemcpyAsync(&nprod, off + nnzA, 8, cudaMemcpyDeviceToHost, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  if (nprod == 0) return C;  // every product row empty

  int* row_of = mem.alloc<int>(nnzA);
  k_entry_rows<<<blocks(na), 256, 0, s>>>(dArp, na, row_of);
  unsigned long long* keys = mem.alloc<unsigned long long>(nprod);
  unsigned long long* keys2 = mem.alloc<unsigned long long>(nprod);
  double* vals = mem.alloc<double>(nprod);
  double* vals2 = mem.alloc<double>(nprod);
  k_expand<<<blocks(nnzA), 256, 0, s>>>(row_of, dAcol, dAval, nnzA, dBrp, dBcol, dBval, off, colbits, keys, vals);
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

  int* ccol = mem.alloc<int>(nnzC);
  double* cval = mem.alloc<double>(nnzC);
  long long* rcount = mem.alloc<long long>(na + 1);
  GNW_CUDA_CHECK(cudaMemsetAsync(rcount, 0, (na + 1) * 8, s));
  k_compress<<<blocks(nprod), 256, 0, s>>>(sk, sv, nprod, head, run_id, colbits, (1ULL << colbits) - 1, ccol, cval,
                                           rcount);
  note_launch("spgemm_compress");
  lap("compute");
  std::vector<long long> counts(na);
  C.cols.resize(nnzC);
  C.vals.resize(nnzC);
  GNW_CUDA_CHECK(cudaMemcpyAsync(counts.data(), rcount, na * 8, cudaMemcpyDeviceToHost, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(C.cols.data(), ccol, nnzC * 4, cudaMemcpyDeviceToHost, s));
  GNW_CUDA_CHECK(cudaMemcpyAsync(C.vals.data(), cval, nnzC * 8, cudaMemcpyDeviceToHost, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  GNW_CUDA_CHECK(cudaGetLastError());
  for (long long i = 0; i < na; ++i) C.rowptr[i + 1] = C.rowptr[i] + counts[i];
  lap("download");
  return C;
}

}  // namespace gnw
