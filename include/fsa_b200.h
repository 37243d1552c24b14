/*
 * fsa_b200.h — C ABI of the B200-native FSA iterative core.
 *
 * Drop-in boundary for the iterative path of the reference library `fsagp`
 * (/root/reference/proj). Every entry point names the reference interface it
 * replaces. Conventions follow the reference's Eigen types:
 *   - dense matrices are column-major doubles (den_mat_t, types.h:14), points
 *     in the caller's original order (LocationSet::coords is n x d);
 *   - sparse outputs are CSR with int64 row offsets and int32 column indices,
 *     columns sorted per row (sp_mat_t RowMajor, types.h:15-16);
 *   - parameter order is (sigma2 = nugget, sigma1_2 = marginal variance, rho)
 *     (types.h:72-102); gradients follow the same order.
 * The caller owns all host buffers; device state lives in the opaque handles. Handles are
 * reference counted: a geometry or model keeps its context alive and a preconditioner or
 * prediction set keeps its model alive, so the *_destroy calls may come in any order.
 * Return codes: FSA_OK, FSA_EINVAL (std::invalid_argument in the reference,
 * types.h:27-29), FSA_ENUMERIC (fsagp::NumericalError, types.h:22-25),
 * FSA_ECUDA (device failure). fsa_last_error() gives the message (thread-local).
 * There is no CPU fallback: every compute entry point needs a CUDA device.
 */
#ifndef FSA_B200_H
#define FSA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSA_OK 0
#define FSA_EINVAL 2
#define FSA_ENUMERIC 3
#define FSA_ECUDA 4

typedef struct fsa_ctx fsa_ctx;
typedef struct fsa_geometry fsa_geometry;
typedef struct fsa_model fsa_model;
typedef struct fsa_precond fsa_precond;
typedef struct fsa_pred fsa_pred;

/* MaternNu / TaperSpec / CovParams / AssembleOptions (types.h:32-102, fsa.h:15-18) */
typedef struct {
  int nu_code;       /* 0: nu = 1/2, 1: nu = 3/2, 2: nu = 5/2 */
  int taper_family;  /* 1: wendland1, 2: wendland2 */
  double gamma;      /* taper range */
  double sigma2;     /* nugget */
  double sigma1_2;   /* marginal variance */
  double rho;        /* range */
  double jitter_rel; /* AssembleOptions::jitter_rel, default 1e-10 */
} fsa_params;

/* CgOptions (krylov.h:28-32) */
typedef struct {
  double tol;
  int max_iter;
  int error_on_max_iter;
} fsa_cg_options;

/* IterativeNll (estimation.h:91-97) plus timing diagnostics */
typedef struct {
  double nll;
  double grad[3];
  double logdet;
  int cg_iterations;
  int sweeps;
  int64_t rhs_iterations; /* sum over columns of CG iterations */
  double pcg_ms;          /* device time of the PCG solve */
  double total_ms;        /* device time of the whole evaluation */
} fsa_nll_result;

/* PredVarResult (prediction.h:37-42) scalars */
typedef struct {
  int clamped;
  int cg_iterations;
  double det_ms;
  double sim_ms;
} fsa_predvar_info;

const char* fsa_last_error(void);
int fsa_version(void);

/* ---- context (one per device; one host thread per context) ---------------------- */
int fsa_ctx_create(int device, fsa_ctx** out);
void fsa_ctx_destroy(fsa_ctx* ctx);
int fsa_ctx_synchronize(fsa_ctx* ctx);
int fsa_ctx_stream(fsa_ctx* ctx, void** stream); /* cudaStream_t all kernels run on */
/* dense m x n passes with the low-rank factor: 0 auto (INT8 tensor-core Ozaki emulation of the fp64
 * product when the RHS block has <= 64 columns, DMMA fp64 otherwise), 1 DMMA fp64 always, 2 Ozaki */
int fsa_ctx_set_gemm_mode(fsa_ctx* ctx, int mode);
/* Diagnostics of the last PCG solve on this context (pcg_solve_multi, iterative_nll_grad, the
 * prediction solves): *k = its column count; for columns j < cap_k, iterations[j] and the
 * residual-norm history rnorm[j * cap_len + i] = ||r_j||_2 after iteration i + 1 (zero past the
 * column's count). No reference counterpart: CgMultiResult (krylov.h:52-75) keeps counts only;
 * the parity tests use the histories to tell an oracle tie from a divergence. */
int fsa_ctx_last_cg(fsa_ctx* ctx, int64_t* k, int64_t cap_k, int64_t cap_len, int* iterations, double* rnorm);
/* CUDA-event timers around kernel groups (name -> total ms, launches, algorithmic units) */
int fsa_ctx_set_profiling(fsa_ctx* ctx, int on);
int fsa_ctx_reset_timers(fsa_ctx* ctx);
int fsa_ctx_timer_names(fsa_ctx* ctx, char* buf, size_t len); /* newline separated */
int fsa_ctx_timer(fsa_ctx* ctx, const char* name, double* ms, int64_t* count, double* units);

/* ---- row-sharded contexts (multi-GPU fit path; no reference counterpart: the
 * reference is one process over OpenMP threads, fsa.cpp / krylov.cpp) ------------------
 * Rank r of W owns a contiguous block of the space-filling-curve-sorted points. Each PCG
 * sweep exchanges halo rows with the ranks whose points are within the taper range and
 * sums the m x t projections and per-column dots. Host inputs stay global (every rank
 * passes all n points, in the caller's order); results (nll, gradient, beta) are identical
 * on every rank. On a sharded context only the geometry / assemble / FITC preconditioner /
 * iterative_nll_grad path is available; the host-block entry points return FSA_EINVAL. */
/* 128-byte NCCL unique id (rank 0 creates it and broadcasts it, e.g. over torch.distributed) */
int fsa_nccl_unique_id(void* id_out);
/* one process per GPU: NCCL over NVLink/NVSwitch (libnccl.so.2 is loaded on first use) */
int fsa_ctx_create_nccl(int device, int rank, int world, const void* unique_id, fsa_ctx** out);
/* W contexts on one device whose collectives are host barriers + device copies; each context
 * must be driven by its own host thread, all making the same calls (test vehicle for the
 * sharded decomposition on a single GPU) */
int fsa_ctx_group_create(int device, int world, fsa_ctx** out /* array of world handles */);
int fsa_ctx_rank(fsa_ctx* ctx, int* rank, int* world);
/* replicated mode (on != 0, before creating geometries): every rank holds the whole model and
 * the communicator shards independent work instead of rows — fsa_predict_var_sim then splits
 * its probe batches over the ranks and sums the moment accumulators; all
 * single-GPU entry points are available. Default: row-sharded. */
int fsa_ctx_set_replicated(fsa_ctx* ctx, int on);

/* ---- input generators (host; same RNG streams as the reference) -------------------- */
/* uniform_locations (locations.cpp:9-17) */
int fsa_uniform_locations(int64_t n, int d, uint64_t seed, double* coords_out);
/* select_random (inducing.cpp:11-24) */
int fsa_select_random(const double* coords, int64_t n, int d, int64_t m, uint64_t seed, double* out);
/* select_kmeanspp (inducing.cpp:48-139), KmeansOptions{max_iter, rel_tol} */
int fsa_select_kmeanspp(const double* coords, int64_t n, int d, int64_t m, uint64_t seed, int max_iter,
                        double rel_tol, double* out);
/* select_kmeanspp on the device (inducing.cpp:48-139): same distinct pool,
 * RNG draws, Lloyd stop rule and greedy snapping as fsa_select_kmeanspp; the seeding rounds,
 * Lloyd assignments / centroids and snapping searches run as kernels on ctx's stream. */
int fsa_select_kmeanspp_device(fsa_ctx* ctx, const double* coords, int64_t n, int d, int64_t m, uint64_t seed,
                               int max_iter, double rel_tol, double* out);
/* gamma_for_avg_row_nnz (locations.cpp:192-195) */
double fsa_gamma_for_avg_row_nnz(int64_t n, double target_row_nnz);
/* synthetic response: random-Fourier-feature Matern draw + N(0, nugget) noise */
int fsa_simulate_rff(const double* coords, int64_t n, int d, int nu_code, double sigma1_2, double rho,
                     double nugget, int features, uint64_t seed, double* y_out);
/* clustered locations: mixture of Gaussian blobs on [0,1]^d */
int fsa_blob_locations(int64_t n, int d, int blobs, double sd, uint64_t seed, double* coords_out);
/* probe streams: probe_rng + gaussian_vector / rademacher_vector (types.h:104-129) */
int fsa_probe_gaussian(uint64_t seed, uint64_t index, int64_t n1, double* e1, int64_t n2, double* e2);
int fsa_probe_rademacher(uint64_t seed, uint64_t index, int64_t n, double* z);

/* ---- geometry: sorted points + taper pattern (GridIndex/taper_pattern, locations.cpp:19-163) */
int fsa_geometry_create(fsa_ctx* ctx, const double* coords, int64_t n, int d, double gamma, fsa_geometry** out);
void fsa_geometry_destroy(fsa_geometry* g);
int fsa_geometry_info(fsa_geometry* g, int64_t* n, int64_t* nnz); /* nnz of this rank's rows */
/* this rank's block [r0, r1) of the internal order and its halo size (0, n, 0 on one rank) */
int fsa_geometry_shard_info(fsa_geometry* g, int64_t* r0, int64_t* r1, int64_t* n_halo);
/* taper_pattern output in the caller's order: distances as values */
int fsa_geometry_pattern(fsa_geometry* g, int64_t* rowptr, int32_t* col, double* dist);
/* internal (space-filling-curve) order: perm[internal] = original index */
int fsa_geometry_permutation(fsa_geometry* g, int32_t* perm);
/* Fit-loop residency (the reference's fit_fsa objective, estimation.cpp:255-284, re-uploads
 * these every evaluation): keep [y | X] in HBM — fsa_iterative_nll_grad with y == NULL then
 * uses it — and cache the parameter-independent probe draws e1/e2 across evaluations. */
int fsa_geometry_set_response(fsa_geometry* g, const double* y, const double* X, int64_t pcols);
int fsa_geometry_cache_probes(fsa_geometry* g, int on);
/* kernels launched by this library so far (process wide) */
int64_t fsa_launch_count(void);

/* ---- FSA model (FsaModel, fsa.h:40-104) -------------------------------------------- */
/* FsaModel::assemble(locs, inducing, kern, taper, params, opts) (fsa.h:42-43); builds the geometry */
int fsa_model_assemble(fsa_ctx* ctx, const double* coords, int64_t n, int d, const double* inducing, int64_t m,
                       const fsa_params* params, fsa_model** out);
/* same on a cached geometry (the taper pattern is parameter independent) */
int fsa_model_assemble_geo(fsa_geometry* g, const double* inducing, int64_t m, const fsa_params* params,
                           fsa_model** out);
void fsa_model_destroy(fsa_model* md);
int fsa_model_info(fsa_model* md, int64_t* n, int64_t* m, int64_t* nnz, int64_t* n_clamped,
                   double* logdet_sigma_m);
/* sigma_s (which = 0) or deriv_sigma_s(2) (which = 1) in the caller's order */
int fsa_model_sigma_s(fsa_model* md, int which, int64_t* rowptr, int32_t* col, double* val);
/* FsaModel::matmat (fsa.cpp:65-68): out = Sigma V, V n x k */
int fsa_model_matmat(fsa_model* md, const double* V, int64_t k, double* out);
/* FsaModel::deriv_matmat (fsa.cpp:165-182) */
int fsa_model_deriv_matmat(fsa_model* md, int which, const double* V, int64_t k, double* out);
/* the low-rank factor U = L^{-1} Sigma_mn (L L^T = Sigma_m + jitter) of the assembled model, applied
 * through the context's GEMM path: out (m x k) = U V for V (n x k); out (n x k) = U^T W for W (m x k).
 * Diagnostics of the dense passes (the reference's A = Sigma_m^{-1} Sigma_mn, fsa.cpp:62-68, is L^{-T} U). */
int fsa_model_lowrank_project(fsa_model* md, const double* V, int64_t k, double* out);
int fsa_model_lowrank_expand(fsa_model* md, const double* W, int64_t k, double* out);
/* diag(Sigma_s) including the nugget (the FITC / Jacobi diagonal) and |U_i|^2 = lowrank diag */
int fsa_model_diagonals(fsa_model* md, double* sigma_s_diag, double* lowrank_diag);
/* Diagnostics (no reference counterpart): average device time of one launch group of a PCG
 * sweep kernel on synthetic k-column blocks — which 0: block SpMM + direction update
 * (k_spmm_v3), 1: Ozaki projection, 2: Ozaki expansion + Woodbury epilogue; flags must be 0
 * (the round-2 component switches were removed with the kernel they instrumented). */
int fsa_debug_kernel_bench(fsa_model* md, int which, int64_t k, int reps, int flags, double* ms_out);

/* ---- preconditioners (make_preconditioner, estimation.h:81-82; preconditioners.h) -- */
/* type: 0 none (IdentityPrecond), 1 diagonal (DiagPrecond), 2 fitc (FitcPrecond::from_fsa(model, true)) */
int fsa_make_preconditioner(fsa_model* md, int type, fsa_precond** out);
/* DiagPrecond(sigma_s.diagonal()) without derivatives (prediction.cpp:94) */
int fsa_make_jacobi(fsa_model* md, fsa_precond** out);
void fsa_precond_destroy(fsa_precond* p);
int fsa_precond_logdet(fsa_precond* p, double* out);
int fsa_precond_solve_mat(fsa_precond* p, const double* R, int64_t k, double* out);
/* Preconditioner::sample_probes (preconditioners.cpp:13-20) */
int fsa_precond_sample_probes(fsa_precond* p, int num_probes, uint64_t seed, double* Z);
/* Preconditioner::deriv_trace (preconditioners.cpp:106-115) */
int fsa_precond_deriv_trace(fsa_precond* p, int which, double* out);

/* ---- Krylov (krylov.h:49-142) -------------------------------------------------------- */
/* pcg_solve_multi (krylov.cpp:18-106), batched. op_kind: 0 FSA operator, 1 sigma_s only.
 * tdiag / toff: k x max_iter column-major (column j holds iterations[j] / iterations[j]-1 entries). */
int fsa_pcg_solve_multi(fsa_model* md, fsa_precond* p, int op_kind, const double* B, int64_t k,
                        const fsa_cg_options* cg, double* X, int* iterations, int* converged, double* tdiag,
                        double* toff, int* sweeps);
/* tridiag_log_quadrature (krylov.cpp:120-142) */
int fsa_tridiag_log_quadrature(const double* diag, const double* off, int64_t len, double* out);
/* iterative_nll_grad (estimation.cpp:178-227). X may be NULL when p = 0; beta has p entries.
 * cv_mode: 0 none, 1 one, 2 optimal (CvMode, krylov.h:87). */
int fsa_iterative_nll_grad(fsa_model* md, fsa_precond* p, const double* y, const double* X, int64_t pcols,
                           int num_probes, uint64_t seed, const fsa_cg_options* cg, int cv_mode, int want_grad,
                           fsa_nll_result* out, double* beta);

/* fisher_ste (fsa.cpp:284-301, FisherOptions fsa.h:107-111): stochastic expected Fisher
 * information of (sigma2, sigma1_2, rho) from num_probes keyed probes (Gaussian, or Rademacher
 * when rademacher != 0). The reference solves with its exact backend (FsaModel::solve); here the
 * L and 3L solves are batched PCG runs with preconditioner p and tolerance cg (pass a tight
 * tolerance for exact-solve agreement). F_out: 3 x 3 column-major, exactly symmetric.
 * cg_iterations (may be NULL): max over both solves. */
int fsa_fisher_ste(fsa_model* md, fsa_precond* p, int num_probes, uint64_t seed, int rademacher,
                   const fsa_cg_options* cg, double* F_out, int* cg_iterations);

/* ---- maximum-likelihood fit (fit_fsa, estimation.cpp:229-303) -------
 * L-BFGS over log(sigma2, sigma1_2, rho) (lbfgs_minimize, estimation.cpp:10-132: two-loop
 * recursion, Armijo + curvature bracketing, NumericalError = +inf), each evaluation
 * FsaModel::assemble + make_preconditioner + iterative_nll_grad on the device with fit-loop
 * residency (pattern, [y | X] and probe draws kept in HBM). Inducing points: kmeans++. */
typedef struct {
  int nu_code;
  int taper_family;
  int64_t num_inducing;
  double taper_range;    /* 0: gamma_for_avg_row_nnz(n, target_row_nnz) */
  double target_row_nnz;
  int precond;           /* 0 none, 1 diagonal, 2 fitc */
  int num_probes;
  int cv_mode;           /* 0 none, 1 one, 2 optimal */
  uint64_t seed;
  double cg_tol;
  int cg_max_iter;
  double jitter_rel;
  int max_evals;
  int lbfgs_memory;
  double armijo_c1;
  int max_backtracks;
  double f_rel_tol;
  double grad_tol_per_n; /* stopping tolerance = grad_tol_per_n * n (infinity norm, log space) */
} fsa_fit_options;
typedef struct {
  double sigma2, sigma1_2, rho, nll, gamma;
  double grad_log[3]; /* gradient at the returned point, log-parameter space */
  int evals;
  int converged;
  int64_t n_trace;    /* entries of the nll trace (one per evaluation) */
} fsa_fit_result;
/* the reference's FitOptions defaults */
void fsa_fit_options_default(fsa_fit_options* opts);
/* beta: pcols values; inducing: num_inducing x d (column-major); nll_trace: up to trace_cap values */
int fsa_fit(fsa_ctx* ctx, const double* coords, int64_t n, int d, const double* y, const double* X, int64_t pcols,
            const fsa_fit_options* opts, fsa_fit_result* out, double* beta, double* inducing, double* nll_trace,
            int64_t trace_cap);

/* ---- prediction (prediction.h:21-56) ------------------------------------------------- */
/* make_prediction_set (prediction.cpp:7-27) */
int fsa_pred_setup(fsa_model* md, const double* pcoords, int64_t np, fsa_pred** out);
void fsa_pred_destroy(fsa_pred* pr);
int fsa_pred_info(fsa_pred* pr, int64_t* np, int64_t* nnz);
/* cross_apply_t (prediction.cpp:29-31): out (np) = Sigma_np^T u */
int fsa_cross_apply_t(fsa_pred* pr, const double* u, double* out);
/* predict_mean_iterative (prediction.cpp:37-43) */
int fsa_predict_mean_iterative(fsa_pred* pr, const double* resid, fsa_precond* p, const fsa_cg_options* cg,
                               double* mean_out);
/* predict_var_sim (prediction.cpp:131-172); SimVarOptions (prediction.h:43-50) */
int fsa_predict_var_sim(fsa_pred* pr, int num_probes, uint64_t seed, const fsa_cg_options* cg,
                        const fsa_cg_options* cg_s, int control_variate, double floor_rel, double* var,
                        double* se, fsa_predvar_info* info);
/* the deterministic diagonals d1, d2, d3 of predict_var_sim (prediction.cpp:72-110) */
int fsa_pred_det_pieces(fsa_pred* pr, const fsa_cg_options* cg, const fsa_cg_options* cg_s, double* d1,
                        double* d2, double* d3, int* cg_iterations);

#ifdef __cplusplus
}
#endif

#endif /* FSA_B200_H */
