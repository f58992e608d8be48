// ert_gmg.cu -- geometric multigrid preconditioner for the ERT pole solves on the structured
// unit-square mesh (BASELINE C4/C5; forward.cpp:39-98 is the operator being solved).
//
// The reference factorises the P1 stiffness K(sigma) exactly (Eigen SparseLU).  The device
// path solves all poles as one batched PCG; its preconditioner used to be an SA-AMG
// hierarchy of K built on the host per model (amg_setup: 0.11 s at C4, 2.2 s at C5, the
// dominant part of t_J).  On make_unit_square_mesh meshes the P1 spaces of the meshes with
// n, n/2, n/4, ... squares per side are nested (each coarse triangle is the union of four
// fine ones, diagonals aligned), so the Galerkin coarse operator P^T K P with P = P1
// interpolation is exactly the P1 stiffness of the coarse mesh with sigma averaged over
// the four children.  Every level is therefore a structured stencil built on the device in
// microseconds, and the hierarchy needs no host setup at all.
//
// Stencil: on these right-isoceles triangles the hypotenuse coupling vanishes, so the P1
// stiffness at free node (i, j) is the 5-point stencil (cells: L = lower (i,j),(i+1,j),(i+1,j+1),
// U = upper (i,j),(i+1,j+1),(i,j+1) of square (i,j); element matrices sigma/2 [[1,-1,0],[-1,2,-1],
// [0,-1,1]] for L and sigma/2 [[1,0,-1],[0,1,-1],[-1,-1,2]] for U, independent of h):
//   C = (L(i,j) + U(i,j) + L(i-1,j-1) + U(i-1,j-1)) / 2 + L(i-1,j) + U(i,j-1)
//   E = -(L(i,j) + U(i,j-1)) / 2      W = -(L(i-1,j) + U(i-1,j-1)) / 2
//   N = -(U(i,j) + L(i-1,j)) / 2      S = -(U(i,j-1) + L(i-1,j-1)) / 2
// with absent cells (j - 1 < 0) contributing nothing.  Grounded nodes (the FAR boundary:
// i = 0, i = n, j = n) are not unknowns; free node (i, j), 1 <= i <= n-1, 0 <= j <= n-1, has
// index j (n-1) + i - 1 (assemble_forward's vertex order).  The PCG operator itself stays the
// exact host-assembled K; the stencil only preconditions.
//
// Cycle: symmetric V(2,2), damped Jacobi (omega = 0.8), full-weighting restriction = P^T,
// P1 prolongation; the coarsest level (n <= 16) is solved with its explicit inverse.
#include <cuda_runtime.h>

#include <cmath>
#include <stdexcept>

#include "ert_gmg.cuh"
#include "kernels.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {

constexpr double kOmega = 0.8;
constexpr int kCoarseN = 16;

__device__ __forceinline__ double sig(const double* s, int n, int i, int j, int t) {
  return (i < 0 || j < 0 || i >= n || j >= n) ? 0.0 : s[2 * (static_cast<long long>(j) * n + i) + t];
}

}  // namespace

__global__ void k_gmg_sigma(const double* __restrict__ m, long long nc, double* __restrict__ s) {
  const long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c < nc) s[c] = exp(m[c]);
}

// coarse cell (I, J, t) = mean of its four children (see the header)
__global__ void k_gmg_coarsen(const double* __restrict__ sf, int nf, double* __restrict__ sc, int ncs) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= 2LL * ncs * ncs) return;
  const int t = static_cast<int>(k & 1);
  const long long sq = k >> 1;
  const int I = static_cast<int>(sq % ncs), J = static_cast<int>(sq / ncs);
  const int i = 2 * I, j = 2 * J;
  double v;
  if (t == 0)  // lower: L(i,j), L(i+1,j), L(i+1,j+1), U(i+1,j)
    v = sig(sf, nf, i, j, 0) + sig(sf, nf, i + 1, j, 0) + sig(sf, nf, i + 1, j + 1, 0) + sig(sf, nf, i + 1, j, 1);
  else  // upper: U(i,j), U(i+1,j+1), U(i,j+1), L(i,j+1)
    v = sig(sf, nf, i, j, 1) + sig(sf, nf, i + 1, j + 1, 1) + sig(sf, nf, i, j + 1, 1) + sig(sf, nf, i, j + 1, 0);
  sc[k] = 0.25 * v;
}

// 5-point stencil (C, W, E, S, N) per free node
__global__ void k_gmg_stencil(const double* __restrict__ s, int n, double* __restrict__ st) {
  const long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long nfree = static_cast<long long>(n - 1) * n;
  if (f >= nfree) return;
  const int i = static_cast<int>(f % (n - 1)) + 1, j = static_cast<int>(f / (n - 1));
  const double Lij = sig(s, n, i, j, 0), Uij = sig(s, n, i, j, 1);
  const double Lw = sig(s, n, i - 1, j, 0), Us = sig(s, n, i, j - 1, 1);
  const double Lsw = sig(s, n, i - 1, j - 1, 0), Usw = sig(s, n, i - 1, j - 1, 1);
  double* o = st + 5 * f;
  o[0] = 0.5 * (Lij + Uij + Lsw + Usw) + Lw + Us;
  o[1] = -0.5 * (Lw + Usw);
  o[2] = -0.5 * (Lij + Us);
  o[3] = -0.5 * (Us + Lsw);
  o[4] = -0.5 * (Uij + Lw);
}

// (A x)(f, q) from the stencil; grounded / absent neighbours are skipped
__device__ __forceinline__ double apply5(const double* __restrict__ st, const double* __restrict__ x, int n,
                                         long long f, int i, int j, int b, int q) {
  const double* o = st + 5 * f;
  const long long w = n - 1;
  double y = o[0] * x[f * b + q];
  if (i > 1) y += o[1] * x[(f - 1) * b + q];
  if (i < n - 1) y += o[2] * x[(f + 1) * b + q];
  if (j > 0) y += o[3] * x[(f - w) * b + q];
  if (j < n - 1) y += o[4] * x[(f + w) * b + q];
  return y;
}

// mode 0: out = omega B / C;  mode 1: out = X + omega (B - A X) / C;  mode 2: out = B - A X
template <int MODE>
__global__ void __launch_bounds__(256) k_gmg_sweep(const double* __restrict__ st, int n, const double* __restrict__ B,
                                                   const double* __restrict__ X, double* __restrict__ out, int b) {
  griddep_wait();
  const long long nfree = static_cast<long long>(n - 1) * n;
  const long long f = static_cast<long long>(blockIdx.x) * blockDim.y + threadIdx.y;
  const int q = blockIdx.y * 32 + threadIdx.x;
  if (f >= nfree || q >= b) return;
  const long long k = f * b + q;
  if (MODE == 0) {
    out[k] = kOmega * B[k] / st[5 * f];
    return;
  }
  const int i = static_cast<int>(f % (n - 1)) + 1, j = static_cast<int>(f / (n - 1));
  const double ax = apply5(st, X, n, f, i, j, b, q);
  if (MODE == 1)
    out[k] = X[k] + kOmega * (B[k] - ax) / st[5 * f];
  else
    out[k] = B[k] - ax;
}

// coarse (I, J) = r(2I, 2J) + (r at the six adjacent midpoints) / 2   (P^T, P = P1 interpolation)
__global__ void __launch_bounds__(256) k_gmg_restrict(const double* __restrict__ r, int nf, double* __restrict__ rc,
                                                      int nc, int b) {
  griddep_wait();
  const long long nfree_c = static_cast<long long>(nc - 1) * nc;
  const long long F = static_cast<long long>(blockIdx.x) * blockDim.y + threadIdx.y;
  const int q = blockIdx.y * 32 + threadIdx.x;
  if (F >= nfree_c || q >= b) return;
  const int I = static_cast<int>(F % (nc - 1)) + 1, J = static_cast<int>(F / (nc - 1));
  const int i = 2 * I, j = 2 * J;
  auto at = [&](int ii, int jj) -> double {
    if (ii < 1 || ii > nf - 1 || jj < 0 || jj > nf - 1) return 0.0;
    return r[(static_cast<long long>(jj) * (nf - 1) + ii - 1) * b + q];
  };
  rc[F * b + q] = at(i, j) + 0.5 * (at(i - 1, j) + at(i + 1, j) + at(i, j - 1) + at(i, j + 1) + at(i + 1, j + 1) +
                                    at(i - 1, j - 1));
}

// x(i, j) += (P e)(i, j)
__global__ void __launch_bounds__(256) k_gmg_prolong(const double* __restrict__ e, int nc, double* __restrict__ x,
                                                     int nf, int b) {
  griddep_wait();
  const long long nfree = static_cast<long long>(nf - 1) * nf;
  const long long f = static_cast<long long>(blockIdx.x) * blockDim.y + threadIdx.y;
  const int q = blockIdx.y * 32 + threadIdx.x;
  if (f >= nfree || q >= b) return;
  const int i = static_cast<int>(f % (nf - 1)) + 1, j = static_cast<int>(f / (nf - 1));
  auto at = [&](int I, int J) -> double {
    if (I < 1 || I > nc - 1 || J < 0 || J > nc - 1) return 0.0;  // grounded coarse node
    return e[(static_cast<long long>(J) * (nc - 1) + I - 1) * b + q];
  };
  const int I = i >> 1, J = j >> 1;
  double v;
  if (!(i & 1) && !(j & 1))
    v = at(I, J);
  else if ((i & 1) && !(j & 1))
    v = 0.5 * (at(I, J) + at(I + 1, J));
  else if (!(i & 1) && (j & 1))
    v = 0.5 * (at(I, J) + at(I, J + 1));
  else
    v = 0.5 * (at(I, J) + at(I + 1, J + 1));
  x[f * b + q] += v;
}

// dense coarsest operator from its stencil (row-major, free x free)
__global__ void k_gmg_dense(const double* __restrict__ st, int n, double* __restrict__ A) {
  const long long nfree = static_cast<long long>(n - 1) * n;
  const long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= nfree) return;
  const int i = static_cast<int>(f % (n - 1)) + 1, j = static_cast<int>(f / (n - 1));
  const double* o = st + 5 * f;
  double* row = A + f * nfree;
  for (long long c = 0; c < nfree; ++c) row[c] = 0.0;
  row[f] = o[0];
  if (i > 1) row[f - 1] = o[1];
  if (i < n - 1) row[f + 1] = o[2];
  if (j > 0) row[f - (n - 1)] = o[3];
  if (j < n - 1) row[f + (n - 1)] = o[4];
}

// ----------------------------------------------------------------------------- host side
int ErtGmg::structured_n(const host::Mesh& mesh, const host::ForwardStructure& fwd) {
  const int64_t nc = mesh.nc;
  int64_t n = static_cast<int64_t>(std::llround(std::sqrt(static_cast<double>(nc) / 2.0)));
  if (n < 2 || 2 * n * n != nc || mesh.nv != (n + 1) * (n + 1)) return 0;
  auto v = [n](int64_t i, int64_t j) { return j * (n + 1) + i; };
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      const int64_t c = 2 * (j * n + i);
      const int64_t* L = &mesh.cells[3 * c];
      const int64_t* U = &mesh.cells[3 * (c + 1)];
      if (L[0] != v(i, j) || L[1] != v(i + 1, j) || L[2] != v(i + 1, j + 1)) return 0;
      if (U[0] != v(i, j) || U[1] != v(i + 1, j + 1) || U[2] != v(i, j + 1)) return 0;
    }
  if (fwd.n_free != (n - 1) * n) return 0;
  for (int64_t j = 0; j <= n; ++j)
    for (int64_t i = 0; i <= n; ++i) {
      const bool grounded = i == 0 || i == n || j == n;
      const int64_t want = grounded ? -1 : j * (n - 1) + i - 1;
      if (fwd.node_to_free[v(i, j)] != want) return 0;
    }
  // at least one coarsening: n even and above the coarsest size
  return (n > kCoarseN && n % 2 == 0) ? static_cast<int>(n) : 0;
}

void ErtGmg::build(int n, const double* m_dev, int b, int* dflag, cudaStream_t s) {
  if (n_ != n || b_ != b) {
    mem_ = std::make_unique<DeviceMemory>();
    n_ = n;
    b_ = b;
    lv_.clear();
    for (int nl = n;; nl /= 2) {
      Level L;
      L.n = nl;
      L.nfree = static_cast<long long>(nl - 1) * nl;
      L.sigma = mem_->alloc<double>(2LL * nl * nl);
      L.st = mem_->alloc<double>(5 * L.nfree);
      const size_t nb = static_cast<size_t>(L.nfree) * b;
      L.X = mem_->alloc<double>(nb);
      L.T = mem_->alloc<double>(nb);
      L.R = mem_->alloc<double>(nb);
      L.B = mem_->alloc<double>(nb);
      lv_.push_back(L);
      if (nl <= kCoarseN || nl % 2 != 0) break;
    }
    const long long nc = lv_.back().nfree;
    Adense_ = mem_->alloc<double>(nc * nc);
    W_ = mem_->alloc<double>(nc * nc);
    L_ = mem_->alloc<double>(nc * nc);
    Ainv_ = mem_->alloc<double>(nc * nc);
    Y_ = mem_->alloc<double>(nc * nc);
  }
  const long long nc0 = 2LL * n * n;
  k_gmg_sigma<<<static_cast<unsigned>((nc0 + 255) / 256), 256, 0, s>>>(m_dev, nc0, lv_[0].sigma);
  note_launch("gmg_sigma");
  for (size_t l = 0; l < lv_.size(); ++l) {
    Level& L = lv_[l];
    if (l > 0) {
      const long long k = 2LL * L.n * L.n;
      k_gmg_coarsen<<<static_cast<unsigned>((k + 255) / 256), 256, 0, s>>>(lv_[l - 1].sigma, lv_[l - 1].n, L.sigma,
                                                                          L.n);
      note_launch("gmg_coarsen");
    }
    k_gmg_stencil<<<static_cast<unsigned>((L.nfree + 255) / 256), 256, 0, s>>>(L.sigma, L.n, L.st);
    note_launch("gmg_stencil");
  }
  const Level& C = lv_.back();
  const int ncf = static_cast<int>(C.nfree);
  k_gmg_dense<<<(ncf + 127) / 128, 128, 0, s>>>(C.st, C.n, Adense_);
  note_launch("gmg_dense");
  cholesky_blocked(Adense_, W_, L_, ncf, dflag, s);
  cholesky_inverse(L_, Y_, Ainv_, ncf, s);
  GNW_CUDA_CHECK(cudaGetLastError());
}

static dim3 bgrid(long long rows, int b) {
  return dim3(static_cast<unsigned>((rows + 7) / 8), static_cast<unsigned>((b + 31) / 32));
}

void ErtGmg::cycle(size_t l, const double* B, double* out, cudaStream_t s) {
  const Level& L = lv_[l];
  const int b = b_;
  const dim3 g = bgrid(L.nfree, b), blk(32, 8);
  if (l + 1 == lv_.size()) {
    mcoarse_inverse(Ainv_, static_cast<int>(L.nfree), B, out, b, s);
    return;
  }
  const Level& Cl = lv_[l + 1];
  // pre-smoothing: X = omega B / C, T = X + omega (B - A X) / C
  GNW_LAUNCH(launch_k(k_gmg_sweep<0>, g, blk, 0, s, L.st, L.n, B, static_cast<const double*>(nullptr), L.X, b));
  GNW_LAUNCH(launch_k(k_gmg_sweep<1>, g, blk, 0, s, L.st, L.n, B, static_cast<const double*>(L.X), L.T, b));
  // residual, restriction, coarse correction
  GNW_LAUNCH(launch_k(k_gmg_sweep<2>, g, blk, 0, s, L.st, L.n, B, static_cast<const double*>(L.T), L.R, b));
  GNW_LAUNCH(launch_k(k_gmg_restrict, bgrid(Cl.nfree, b), blk, 0, s, static_cast<const double*>(L.R), L.n, Cl.B,
                      Cl.n, b));
  // the coarse cycle returns in Cl.R: its X and T are its own scratch, R is free again once
  // it has restricted its residual
  cycle(l + 1, Cl.B, Cl.R, s);
  GNW_LAUNCH(launch_k(k_gmg_prolong, g, blk, 0, s, static_cast<const double*>(Cl.R), Cl.n, L.T, L.n, b));
  // post-smoothing (same sweeps: the cycle stays symmetric for CG)
  GNW_LAUNCH(launch_k(k_gmg_sweep<1>, g, blk, 0, s, L.st, L.n, B, static_cast<const double*>(L.T), L.X, b));
  GNW_LAUNCH(launch_k(k_gmg_sweep<1>, g, blk, 0, s, L.st, L.n, B, static_cast<const double*>(L.X), out, b));
  for (int k = 0; k < 7; ++k) note_launch("gmg_cycle");
}

void ErtGmg::vcycle(const double* r, double* z, cudaStream_t s) { cycle(0, r, z, s); }

}  // namespace gnw
