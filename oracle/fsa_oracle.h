// TEST INFRASTRUCTURE ONLY — C ABI of the CPU oracle (oracle/fsa_oracle.cpp),
// loaded by tests/ and bench.py's cpu_baseline leg through ctypes. Never linked
// by the product library.
#pragma once
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
struct orc_csr;
typedef struct orc_csr orc_csr;
const char* orc_last_error(void);
uint64_t orc_splitmix64(uint64_t x);
void orc_probe_gaussian(uint64_t seed, uint64_t i, long n1, double* e1, long n2, double* e2);
void orc_probe_rademacher(uint64_t seed, uint64_t i, long n, double* z);
uint64_t orc_mt19937_64_nth(uint64_t seed, long nth);
double orc_matern(double d, int nu, double s1, double rho);
double orc_matern_drho(double d, int nu, double s1, double rho);
double orc_taper_value(double d, int family, double gamma);
double orc_rho_for_correlation_at(double dist, double corr, int nu);
double orc_effective_range(double rho, int nu);
double orc_gamma_for_avg_row_nnz(long n, double target);
int orc_uniform_locations(long n, int d, uint64_t seed, double* out);
int orc_select_random(const double* c, long n, int d, long m, uint64_t seed, double* out);
int orc_select_kmeanspp(const double* c, long n, int d, long m, uint64_t seed, int max_iter, double rel_tol, double* out);
int orc_taper_pattern(const double* c, long n, int d, double gamma, const double* pc, long np, orc_csr** out, long* nnz);
void orc_csr_copy(const orc_csr* s, long* ptr, int* idx, double* val);
void orc_csr_free(orc_csr* s);
int orc_assemble(const double* c, long n, int d, const double* ind, long m, int nu, int fam, double gamma,
                 double s2, double s12, double rho, double jitter_rel, void** out);
void orc_model_free(void* md);
void orc_model_info(void* mdv, double* info);
int orc_model_csr(void* mdv, int which, long* ptr, int* idx, double* val);
int orc_model_dense(void* mdv, int which, double* out);
int orc_matmat(void* mdv, const double* V, long k, double* out);
int orc_deriv_matmat(void* mdv, int which, const double* V, long k, double* out);
int orc_make_preconditioner(void* mdv, int type, void** out);
int orc_fitc_plain(void* mdv, void** out);
int orc_jacobi(void* mdv, void** out);
void orc_precond_free(void* p);
double orc_precond_logdet(void* p);
int orc_precond_kind(void* p);
int orc_precond_solve_mat(void* p, const double* R, long k, double* out);
int orc_precond_solve_cols(void* p, const double* R, long k, double* out);
int orc_precond_sample_probes(void* p, int L, uint64_t seed, double* out);
int orc_precond_deriv_apply(void* p, int which, const double* v, double* out);
int orc_precond_deriv_trace(void* p, int which, double* out);
int orc_pcg(void* mdv, int op_kind, void* p, const double* B, long k, double tol, int max_iter, int batched,
            double* X, int* iters, int* conv, double* tdiag, double* toff, int* sweeps);
int orc_tridiag_log_quadrature(const double* diag, const double* off, long len, double* out);
int orc_iterative_nll_grad(void* mdv, void* p, const double* y, const double* X, long pcols, int L, uint64_t seed,
                           double tol, int max_iter, int cv, int want_grad, double* out, double* beta);
int orc_iterative_nll_grad_ex(void* mdv, void* p, const double* y, const double* X, long pcols, int L, uint64_t seed,
                              double tol, int max_iter, int cv, int want_grad, double* out, double* beta, int* iters,
                              double* rnorm, const long* rows, long nrows, double* xrows);
int orc_pcg_ex(void* mdv, int op_kind, void* p, const double* B, long k, double tol, int max_iter, int batched,
               double* X, int* iters, int* conv, double* tdiag, double* toff, double* rnorm, int* sweeps);
int orc_simulate_rff(const double* c, long n, int d, int nu_code, double sigma1_2, double rho, double nugget,
                     int features, uint64_t seed, double* y);
int orc_blob_locations(long n, int d, int blobs, double sd, uint64_t seed, double* out);
int orc_ste_grad_trace(void* mdv, void* p, const double* Z, const double* W, long L, int which, int mode, double* out);
int orc_pred_make(void* mdv, const double* pc, long np, void** out, long* nnz);
void orc_pred_free(void* p);
int orc_pred_csr(void* pv, long* ptr, int* idx, double* val);
int orc_cross_apply_t(void* mdv, void* pv, const double* u, double* out);
int orc_predict_mean_iterative(void* mdv, void* pv, const double* resid, void* p, double tol, int max_iter, double* out);
int orc_predict_var_sim(void* mdv, void* pv, int L, uint64_t seed, double tol, int maxit, double tol_s, int maxit_s,
                        int cv, double floor_rel, double* var, double* se, int* clamped, int* cg_iters);
int orc_pred_sample_timing(void* mdv, void* pv, long cols, int probes, uint64_t seed, double tol, int maxit,
                           double tol_s, int maxit_s, double* out);
int orc_pred_det_pieces(void* mdv, void* pv, double tol, int maxit, double tol_s, int maxit_s, double* d1, double* d2,
                        double* d3, int* cg_iters);
#ifdef __cplusplus
}
#endif
