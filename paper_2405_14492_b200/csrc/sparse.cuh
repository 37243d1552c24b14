// Sparse assembly (SDDMM) and SpMM launchers; see sparse.cu.
#pragma once

#include "common.cuh"
#include "pattern.cuh"

namespace fsa {

struct SddmmParams {
  int nu, family;
  double sigma2, sigma1_2, rho, gamma;
};

void sddmm_sigma_s(const double* U, long ldu, const Csr& pat, const double* lowrank_diag, const SddmmParams& P,
                   double* val, int* n_clamped_dev, cudaStream_t s);
void sddmm_drho(const double* U, const double* U1, const double* T, long ldu, const Csr& pat,
                const double* lowrank_diag, const SddmmParams& P, double* val, cudaStream_t s);
void sddmm_cross(const double* Rm, long ldr, const double* Cm, long ldc, const Csr& pat, const SddmmParams& P,
                 double* val, cudaStream_t s);
// out[i] = |U_i|^2 for i < n, 0 for padding
void colnorm2(const double* U, long ldu, long mpad, long n, long n_pad, double* out, cudaStream_t s);
// D[i] = val[diagpos[i]] (1 on padding), Dinv = 1/D, sqrtD = sqrt(D) (either may be null)
void extract_diag(const double* val, const long* diagpos, long n, long n_pad, double* D, double* Dinv,
                  double* sqrtD, cudaStream_t s);

}  // namespace fsa
