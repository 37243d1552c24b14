// TEST INFRASTRUCTURE ONLY — CPU oracle helper (see blas_lite.cpp).
#pragma once

namespace orc {
// C(MxN) = alpha * op(A) * op(B) + beta * C, column-major, op = 'N' or 'T'.
void dgemm(char ta, char tb, long M, long N, long K, double alpha, const double* A, long lda,
           const double* B, long ldb, double beta, double* C, long ldc);
}  // namespace orc
