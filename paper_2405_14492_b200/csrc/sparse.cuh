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
// the same on the row groups (pat.gnnz > 0) through dense DMMA Gram blocks: mode 0 Sigma_s
// (also fills the SpMM value blocks gval when non-null), mode 1 d Sigma_s / d rho;
// gtmp holds kGroup * pat.gnnz doubles
void sddmm_block(int mode, const double* U, const double* U1, const double* T, long ldu, long mp, const Csr& pat,
                 const double* lowrank_diag, const SddmmParams& P, double* val, double* gval, int* n_clamped_dev,
                 double* gtmp, cudaStream_t s);
void sddmm_cross(const double* Rm, long ldr, const double* Cm, long ldc, const Csr& pat, const SddmmParams& P,
                 double* val, cudaStream_t s);
// Y = alpha S X + beta Y (first ncols <= 256 columns) fused with dot[c] = sum_r X[r][c] Y[r][c];
// partial must hold spmm_dot_blocks(nrows) * ncols doubles
long spmm_dot_blocks(long nrows);
// block variant on the row groups (pat.gnnz > 0, build_groups): Y = Y0 + S X and
// dot[c] = sum_r X[r][c] Y[r][c] for ncols <= 64 (multiple of 8, ldx == ldy == ncols);
// gval = group_values(pat, val); partial holds spmm_group_blocks(pat.ngrp) * ncols doubles
void group_values(const Csr& pat, const double* val, double* gval, cudaStream_t s);
long spmm_group_blocks(long ngrp);
bool spmm_block_supported(long ncols);
void spmm_block_dot(const Csr& pat, const double* gval, const double* X, long ldx, double* Y, long ldy, long ncols,
                    double* dot, double* partial, const double* Y0, cudaStream_t s);
// the same with the PCG direction update folded in (fused FITC sweep): X = Z (gathered), Y0 = Lw,
// and on the own rows H = Z + beta H, Y = (Lw + S Z) + beta Y (first sweep: H = Z, Y = Lw + S Z);
// dot[c] = sum_r H[r][c] Y[r][c]
void spmm_block_dot_h(const Csr& pat, const double* gval, const double* X, long ldx, double* Y, long ldy, long ncols,
                      double* dot, double* partial, const double* Y0, double* H, const double* beta, long kb,
                      bool first, cudaStream_t s, bool colsum = true);  // colsum = false: partials [ngrp][ncols] only
// (Y0, when given, replaces Y as the beta term: Y = alpha S X + beta Y0)
void spmm_dot(const long* rowptr, const int* col, const double* val, long nrows, const double* X, long ldx, double* Y,
              long ldy, long ncols, double alpha, double beta, double* dot, double* partial, cudaStream_t s,
              const double* Y0 = nullptr);
// out[i] = |U_i|^2 for i < n, 0 for padding
void colnorm2(const double* U, long ldu, long mpad, long n, long n_pad, double* out, cudaStream_t s);
// D[i] = val[diagpos[i]] (1 on padding), Dinv = 1/D, sqrtD = sqrt(D) (either may be null)
void extract_diag(const double* val, const long* diagpos, long n, long n_pad, double* D, double* Dinv,
                  double* sqrtD, cudaStream_t s);

}  // namespace fsa
