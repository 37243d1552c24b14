// Host-side input generators (see inputs.cpp).
#pragma once

namespace fsa {
void uniform_locations(long n, int d, unsigned long long seed, double* out);
void select_random(const double* c, long n, int d, long m, unsigned long long seed, double* out);
void select_kmeanspp(const double* c, long n, int d, long m, unsigned long long seed, int max_iter, double rel_tol,
                     double* out);
double gamma_for_avg_row_nnz(long n, double target);
void simulate_rff(const double* c, long n, int d, int nu_code, double sigma1_2, double rho, double nugget,
                  int features, unsigned long long seed, double* y);
void blob_locations(long n, int d, int blobs, double sd, unsigned long long seed, double* out);
}  // namespace fsa
