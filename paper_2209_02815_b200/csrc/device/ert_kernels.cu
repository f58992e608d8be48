// ert_kernels.cu -- device kernels of the ERT forward model (forward.cpp:83-172):
// batched PCG for the unit-pole solves K u_e = e_e (one column per used electrode,
// columns interleaved X[row * b + q]), cellwise potential gradients, and the
// sensitivity rows J(i, c) = -k_i sigma_c area_c grad(u_A - u_B) . grad(u_M - u_N)
// with the response g_i = sum_c of the same terms.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "ert_kernels.cuh"

namespace gnw {

void note_launch(const char* what);

namespace {
constexpr int kT = 256;
inline unsigned cdiv(long long a, long long b) { return static_cast<unsigned>((a + b - 1) / b); }
}  // namespace

// Y = A X, b interleaved columns (thread per (row, column))
__global__ void __launch_bounds__(256) k_spmm(DCsr A, const double* __restrict__ X, double* __restrict__ Y, int b) {
  griddep_wait();
  const int i = blockIdx.x * 8 + threadIdx.y;
  const int q = blockIdx.y * 32 + threadIdx.x;
  if (i >= A.n_rows || q >= b) return;
  double s = 0.0;
  for (int k = A.rowptr[i]; k < A.rowptr[i + 1]; ++k)
    s = s + __ldg(&A.vals[k]) * X[static_cast<long long>(A.cols[k]) * b + q];
  Y[static_cast<long long>(i) * b + q] = s;
}

// out[q] = sum_i X[i, q] Y[i, q] (and out[b + q] = sum_i X[i, q]^2 when both), fixed-order
// two-stage reduction: rows split in chunks, last block sums the chunk partials.
__global__ void __launch_bounds__(256) k_col_dots(const double* __restrict__ X, const double* __restrict__ Y, long long n,
                                                  int b, int rows_per_chunk, double* __restrict__ part,
                                                  unsigned* counter, double* __restrict__ out, int with_xx) {
  griddep_wait();
  __shared__ double sm[2][8][33];
  __shared__ bool last;
  const int q = blockIdx.y * 32 + threadIdx.x;
  const long long r0 = static_cast<long long>(blockIdx.x) * rows_per_chunk;
  const long long r1 = min(n, r0 + rows_per_chunk);
  double xy = 0.0, xx = 0.0;
  if (q < b)
    for (long long i = r0 + threadIdx.y; i < r1; i += 8) {
      const double x = X[i * b + q];
      xy = xy + x * Y[i * b + q];
      xx = xx + x * x;
    }
  sm[0][threadIdx.y][threadIdx.x] = xy;
  sm[1][threadIdx.y][threadIdx.x] = xx;
  __syncthreads();
  if (threadIdx.y == 0 && q < b) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < 8; ++w) {
      s0 += sm[0][w][threadIdx.x];
      s1 += sm[1][w][threadIdx.x];
    }
    part[(static_cast<long long>(blockIdx.x) * 2 + 0) * b + q] = s0;
    part[(static_cast<long long>(blockIdx.x) * 2 + 1) * b + q] = s1;
  }
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int t = threadIdx.y * 32 + threadIdx.x;
  for (int qq = t; qq < b; qq += 256) {
    double s0 = 0.0, s1 = 0.0;
    for (unsigned c = 0; c < gridDim.x; ++c) {
      s0 += __ldcg(&part[(static_cast<long long>(c) * 2 + 0) * b + qq]);
      s1 += __ldcg(&part[(static_cast<long long>(c) * 2 + 1) * b + qq]);
    }
    out[qq] = s0;
    if (with_xx) out[b + qq] = s1;
  }
  if (t == 0) *counter = 0u;
}

// x += alpha_q p ; r -= alpha_q Ap   (alpha_q = rz_q / pAp_q, frozen columns skip)
__global__ void __launch_bounds__(256) k_pcg_xr(double* __restrict__ x, double* __restrict__ r,
                                                const double* __restrict__ p, const double* __restrict__ Ap,
                                                const double* __restrict__ rz, const double* __restrict__ pap,
                                                const int* __restrict__ active, long long n, int b) {
  griddep_wait();
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * b) return;
  const int q = static_cast<int>(e % b);
  if (!active[q]) return;
  const double alpha = rz[q] / pap[q];
  x[e] = x[e] + alpha * p[e];
  r[e] = r[e] - alpha * Ap[e];
}

// p = z + beta_q p, beta_q = rz_new / rz_old
__global__ void __launch_bounds__(256) k_pcg_p(double* __restrict__ p, const double* __restrict__ z,
                                               const double* __restrict__ rz_new, const double* __restrict__ rz_old,
                                               const int* __restrict__ active, long long n, int b) {
  griddep_wait();
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * b) return;
  const int q = static_cast<int>(e % b);
  if (!active[q]) return;
  p[e] = z[e] + (rz_new[q] / rz_old[q]) * p[e];
}

// cellwise gradients of the pole potentials (forward.cpp:128-143):
// gx[q][c] = sum_i u_q[t_i] grad_i(c).x, grounded nodes carry u = 0
__global__ void __launch_bounds__(256) k_cell_grad(const int64_t* __restrict__ cells, const int64_t* __restrict__ node_to_free,
                                                   const double* __restrict__ grad, const double* __restrict__ X, int b,
                                                   long long nc, double* __restrict__ gx, double* __restrict__ gz) {
  griddep_wait();
  const long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  long long f[3];
  for (int i = 0; i < 3; ++i) f[i] = node_to_free[cells[3 * c + i]];
  const double* g = grad + 6 * c;
  for (int q = 0; q < b; ++q) {
    double sx = 0.0, sz = 0.0;
    for (int i = 0; i < 3; ++i) {
      const double u = f[i] >= 0 ? X[f[i] * b + q] : 0.0;
      sx = sx + u * g[2 * i];
      sz = sz + u * g[2 * i + 1];
    }
    gx[static_cast<long long>(q) * nc + c] = sx;
    gz[static_cast<long long>(q) * nc + c] = sz;
  }
}

// J rows and response partials (forward.cpp:145-167).  grid = (config groups of 32, cell chunks
// of 256): the config groups of one cell chunk run back to back, so the chunk's gradient
// columns are re-read from L2, not DRAM (the other order re-streamed gx/gz, 2 GB at C5, once
// per group: 42 ms for the 63 GB J).
__global__ void __launch_bounds__(256) k_jacobian(const ErtCfgDev* __restrict__ cfg, int n_cfg,
                                                  const int* __restrict__ col_of_electrode, const double* __restrict__ gx,
                                                  const double* __restrict__ gz, const double* __restrict__ mdl,
                                                  const double* __restrict__ area, long long nc, double* __restrict__ J,
                                                  long long ldj, double* __restrict__ gpart) {
  griddep_wait();
  __shared__ double red[8][33];
  const long long c = static_cast<long long>(blockIdx.y) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool ok = c < nc;
  const double sa = ok ? exp(mdl[c]) : 0.0;
  const double ar = ok ? area[c] : 0.0;
  // surveys list the readings of one source together: the source gradient t is reloaded
  // only when (a, b) changes (uniform across the block), halving the gradient loads
  int pa = -2, pb = -2;
  double tx = 0.0, tz = 0.0;
  for (int k = 0; k < 32; ++k) {
    const int i = blockIdx.x * 32 + k;
    if (i >= n_cfg) break;  // uniform across the block
    const ErtCfgDev cf = cfg[i];
    double term = 0.0;
    if (ok) {
      const long long mm = col_of_electrode[cf.m], nn = col_of_electrode[cf.n];
      if (cf.a != pa || cf.b != pb) {
        const long long a = col_of_electrode[cf.a];
        tx = gx[a * nc + c];
        tz = gz[a * nc + c];
        if (cf.b >= 0) {
          const long long bb = col_of_electrode[cf.b];
          tx = tx - gx[bb * nc + c];
          tz = tz - gz[bb * nc + c];
        }
        pa = cf.a;
        pb = cf.b;
      }
      const double rx = gx[mm * nc + c] - gx[nn * nc + c];
      const double rz = gz[mm * nc + c] - gz[nn * nc + c];
      term = cf.k * sa * ar * (tx * rx + tz * rz);
      J[static_cast<long long>(i) * ldj + c] = -term;  // J 1 = -g, term by term
    }
    double v[1] = {term};
    warp_reduce<1>(v);
    if (lane == 0) red[warp][k] = v[0];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int i = blockIdx.x * 32 + threadIdx.x;
    if (i < n_cfg) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
      gpart[static_cast<long long>(blockIdx.y) * n_cfg + i] = s;
    }
  }
}

// g_i = sum over cell chunks (fixed order), warp per config
__global__ void k_response_reduce(const double* __restrict__ gpart, int nchunks, int n_cfg, double* __restrict__ g) {
  griddep_wait();
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= n_cfg) return;
  double acc[1] = {0.0};
  for (int ch = lane; ch < nchunks; ch += 32) acc[0] = acc[0] + gpart[static_cast<long long>(ch) * n_cfg + i];
  warp_reduce<1>(acc);
  if (lane == 0) g[i] = acc[0];
}

// ------------------------------------------------------------------ launchers
__global__ void k_unit_columns(double* __restrict__ R, const int64_t* __restrict__ unit, int b) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < b) R[unit[q] * b + q] = 1.0;
}
void unit_columns(double* R, const int64_t* unit, long long nf, int b, cudaStream_t s) {
  const cudaError_t e = cudaMemsetAsync(R, 0, static_cast<size_t>(nf) * b * sizeof(double), s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("unit_columns: ") + cudaGetErrorString(e));
  k_unit_columns<<<cdiv(b, 64), 64, 0, s>>>(R, unit, b);
  note_launch("unit_columns");
}
void spmm(const DCsr& A, const double* X, double* Y, int b, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_spmm, dim3(cdiv(A.n_rows, 8), cdiv(b, 32)), dim3(32, 8), 0, s, A, X, Y, b));
  note_launch("spmm");
}
void col_dots(const double* X, const double* Y, long long n, int b, double* part, unsigned* counter, double* out,
              int with_xx, cudaStream_t s) {
  const int rows_per_chunk = 2048;
  GNW_LAUNCH(launch_k(k_col_dots, dim3(cdiv(n, rows_per_chunk), cdiv(b, 32)), dim3(32, 8), 0, s, X, Y, n, b,
                      rows_per_chunk, part, counter, out, with_xx));
  note_launch("col_dots");
}
int col_dots_chunks(long long n) { return static_cast<int>(cdiv(n, 2048)); }
void pcg_xr(double* x, double* r, const double* p, const double* Ap, const double* rz, const double* pap,
            const int* active, long long n, int b, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_pcg_xr, cdiv(n * b, kT), kT, 0, s, x, r, p, Ap, rz, pap, active, n, b));
  note_launch("pcg_xr");
}
void pcg_p(double* p, const double* z, const double* rz_new, const double* rz_old, const int* active, long long n,
           int b, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_pcg_p, cdiv(n * b, kT), kT, 0, s, p, z, rz_new, rz_old, active, n, b));
  note_launch("pcg_p");
}
void cell_grad(const int64_t* cells, const int64_t* node_to_free, const double* grad, const double* X, int b,
               long long nc, double* gx, double* gz, cudaStream_t s) {
  GNW_LAUNCH(launch_k(k_cell_grad, cdiv(nc, kT), kT, 0, s, cells, node_to_free, grad, X, b, nc, gx, gz));
  note_launch("cell_grad");
}
int jacobian_chunks(long long nc) { return static_cast<int>(cdiv(nc, kT)); }
void jacobian(const ErtCfgDev* cfg, int n_cfg, const int* col_of_electrode, const double* gx, const double* gz,
              const double* mdl, const double* area, long long nc, double* J, long long ldj, double* gpart, double* g,
              cudaStream_t s) {
  const int nch = jacobian_chunks(nc);
  GNW_LAUNCH(launch_k(k_jacobian, dim3(cdiv(n_cfg, 32), nch), kT, 0, s, cfg, n_cfg, col_of_electrode, gx, gz, mdl,
                      area, nc, J, ldj, gpart));
  note_launch("jacobian");
  GNW_LAUNCH(launch_k(k_response_reduce, cdiv(static_cast<long long>(n_cfg) * 32, kT), kT, 0, s, gpart, nch, n_cfg, g));
  note_launch("response_reduce");
}

}  // namespace gnw
