// TEST INFRASTRUCTURE ONLY — part of the CPU oracle (see oracle/fsa_oracle.cpp).
// Nothing in the product path may link or call this file.
//
// A small cache-blocked, OpenMP-parallel dgemm standing in for the Eigen GEMM
// products the reference uses (fsa.cpp:33-34,62,67; preconditioners.cpp:49).
// Column-major; the summation order over k is fixed (blocks of KC in order,
// k ascending inside a block), and threads split only the M/N dimensions, so
// results are bitwise independent of the thread count.
#include <algorithm>
#include <cstring>
#include <vector>

#include "blas_lite.h"

namespace orc {

namespace {
constexpr long MR = 8, NR = 4, KC = 256, MC = 128;

inline double getA(char ta, const double* A, long lda, long i, long k) {
  return ta == 'N' ? A[i + k * lda] : A[k + i * lda];
}
inline double getB(char tb, const double* B, long ldb, long k, long j) {
  return tb == 'N' ? B[k + j * ldb] : B[j + k * ldb];
}

// acc(8x4) over kc steps from packed panels
inline void micro(long kc, const double* __restrict ap, const double* __restrict bp,
                  double* __restrict acc) {
  double c[NR][MR];
  for (int j = 0; j < NR; ++j)
    for (int i = 0; i < MR; ++i) c[j][i] = 0.0;
  for (long k = 0; k < kc; ++k) {
    const double* a = ap + k * MR;
    const double* b = bp + k * NR;
    for (int j = 0; j < NR; ++j) {
      const double bj = b[j];
      for (int i = 0; i < MR; ++i) c[j][i] += a[i] * bj;
    }
  }
  for (int j = 0; j < NR; ++j)
    for (int i = 0; i < MR; ++i) acc[j * MR + i] = c[j][i];
}
}  // namespace

void dgemm(char ta, char tb, long M, long N, long K, double alpha, const double* A, long lda,
           const double* B, long ldb, double beta, double* C, long ldc) {
  if (M <= 0 || N <= 0) return;
  // scale C by beta first (deterministic, elementwise)
#pragma omp parallel for schedule(static) if (M * N > 65536)
  for (long j = 0; j < N; ++j) {
    double* cj = C + j * ldc;
    if (beta == 0.0)
      for (long i = 0; i < M; ++i) cj[i] = 0.0;
    else if (beta != 1.0)
      for (long i = 0; i < M; ++i) cj[i] *= beta;
  }
  if (K <= 0 || alpha == 0.0) return;

  const long Np = (N + NR - 1) / NR * NR;
  std::vector<double> bpack(static_cast<size_t>(KC * Np));
  for (long pc = 0; pc < K; pc += KC) {
    const long kc = std::min(KC, K - pc);
    // pack B(kc x N) into NR-column strips, zero padded
#pragma omp parallel for schedule(static) if (kc * N > 65536)
    for (long js = 0; js < Np / NR; ++js) {
      double* dst = bpack.data() + js * NR * kc;
      for (long k = 0; k < kc; ++k)
        for (long jj = 0; jj < NR; ++jj) {
          const long j = js * NR + jj;
          dst[k * NR + jj] = j < N ? getB(tb, B, ldb, pc + k, j) : 0.0;
        }
    }
    const long nblk_m = (M + MC - 1) / MC;
    const long nstrip_n = Np / NR;
    // parallel over (m-block, n-strip group) tiles: each C element is owned by one thread
    const long NG = 16;  // n-strips per task
    const long ngroups = (nstrip_n + NG - 1) / NG;
#pragma omp parallel if (M * N * kc > 200000)
    {
      std::vector<double> apack(static_cast<size_t>(MC * KC));
      double acc[MR * NR];
      long last_ib = -1;
#pragma omp for schedule(static) collapse(2)
      for (long ib = 0; ib < nblk_m; ++ib) {
        for (long g = 0; g < ngroups; ++g) {
          const long i0 = ib * MC;
          const long mc = std::min(MC, M - i0);
          const long mstrips = (mc + MR - 1) / MR;
          if (ib != last_ib) {
            for (long is = 0; is < mstrips; ++is)
              for (long k = 0; k < kc; ++k)
                for (long ii = 0; ii < MR; ++ii) {
                  const long i = i0 + is * MR + ii;
                  apack[is * MR * kc + k * MR + ii] =
                      i < M ? getA(ta, A, lda, i, pc + k) : 0.0;
                }
            last_ib = ib;
          }
          const long s0 = g * NG, s1 = std::min(nstrip_n, s0 + NG);
          for (long js = s0; js < s1; ++js) {
            for (long is = 0; is < mstrips; ++is) {
              micro(kc, apack.data() + is * MR * kc, bpack.data() + js * NR * kc, acc);
              for (long jj = 0; jj < NR; ++jj) {
                const long j = js * NR + jj;
                if (j >= N) break;
                double* cj = C + j * ldc;
                for (long ii = 0; ii < MR; ++ii) {
                  const long i = i0 + is * MR + ii;
                  if (i >= M) break;
                  cj[i] += alpha * acc[jj * MR + ii];
                }
              }
            }
          }
        }
      }
    }
  }
}

}  // namespace orc
