// Device k-means++ / Lloyd inducing-point selection (inducing.cpp:48-139; kmeans.cu).
#pragma once
#include <cuda_runtime.h>

namespace fsa {
// coords: host, n x d column-major (original order); out: host, m x d column-major. Runs on
// stream s and synchronises it. Throws std::invalid_argument on the reference's shape errors.
void select_kmeanspp_device(cudaStream_t s, const double* coords, long n, int d, long m, unsigned long long seed,
                            int max_iter, double rel_tol, double* out);
}  // namespace fsa
