// ert_kernels.cuh -- launch interfaces of the ERT forward-model kernels (ert_kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace gnw {

struct ErtCfgDev {  // ElectrodeConfig, survey.hpp:15-21 (b < 0: pole at infinity)
  int a, b, m, n;
  double k;
};

// R = 0 except R[unit[q] * b + q] = 1 (the unit-pole right-hand sides, free x b interleaved)
void unit_columns(double* R, const int64_t* unit, long long nf, int b, cudaStream_t s);
void spmm(const DCsr& A, const double* X, double* Y, int b, cudaStream_t s);
int col_dots_chunks(long long n);
void col_dots(const double* X, const double* Y, long long n, int b, double* part, unsigned* counter, double* out,
              int with_xx, cudaStream_t s);
void pcg_xr(double* x, double* r, const double* p, const double* Ap, const double* rz, const double* pap,
            const int* active, long long n, int b, cudaStream_t s);
void pcg_p(double* p, const double* z, const double* rz_new, const double* rz_old, const int* active, long long n,
           int b, cudaStream_t s);
void cell_grad(const int64_t* cells, const int64_t* node_to_free, const double* grad, const double* X, int b,
               long long nc, double* gx, double* gz, cudaStream_t s);
int jacobian_chunks(long long nc);
void jacobian(const ErtCfgDev* cfg, int n_cfg, const int* col_of_electrode, const double* gx, const double* gz,
              const double* mdl, const double* area, long long nc, double* J, long long ldj, double* gpart, double* g,
              cudaStream_t s);

}  // namespace gnw
