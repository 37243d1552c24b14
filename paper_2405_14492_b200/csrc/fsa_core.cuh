// Host side of the B200 FSA iterative core. Mirrors the reference's operator
// API (FsaModel::assemble, make_preconditioner, pcg_solve_multi,
// iterative_nll_grad, make_prediction_set, predict_mean_iterative,
// predict_var_sim) over device-resident state.
//
// Everything runs in the "U-form" of the FSA covariance:
//   Sigma = U^T U + Sigma_s,  U = L^{-1} Sigma_mn,  L L^T = Sigma_m (+ jitter)
// which is the reference's Sigma_mn^T Sigma_m^{-1} Sigma_mn low-rank part
// (fsa.cpp:62-68) without forming A = Sigma_m^{-1} Sigma_mn: one m x n matrix
// serves both the projection and the expansion, and the FITC Woodbury core
// becomes Q = I + U D^{-1} U^T = L^{-1} (Sigma_m + Sigma_mn D^{-1} Sigma_mn^T) L^{-T}.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "blas1.cuh"
#include "comm.cuh"
#include "common.cuh"
#include "ozaki.cuh"
#include "pattern.cuh"
#include "shard.cuh"

namespace fsa {

// PCG workspace (owned by the context so it is released before the stream)
struct CgWork {
  DBuf<double> R, H, V, Z, Lw, Vlr, dots, dbl, part;
  DBuf<double> part_rr;  // residual-update partials kept to the end of the sweep (fused control path)
  DBuf<int> ints;
  DBuf<double> tri;
  DBuf<unsigned int> tick;  // last-block counter of the fused control kernels
  DBuf<unsigned long long> wmax;  // column maxima of |w| from the core solve (fused control path)
};

struct PinnedBuf {
  double* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n) return;
    if (p) cudaFreeHost(p);
    FSA_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), count * sizeof(double)));
    n = count;
  }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};

// ---- context: device, stream, timers ----------------------------------------------------
struct Context {
  std::unique_ptr<CgWork> cgw{new CgWork()};
  PinnedBuf pin1, pin2;
  std::unique_ptr<Comm> comm{new SelfComm()};  // ranks of a multi-GPU job
  // true: geometries built on this context are row-sharded over `comm`; false (replicated):
  // every rank holds the whole model and `comm` shards independent work units (the
  // predictive-variance probe batches)
  bool shard_rows = true;
  SelfComm self_comm;
  bool row_sharded() const { return shard_rows && comm->size() > 1; }
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // second stream (rho-derivative build during the PCG), lazily created
  cudaStream_t side_stream();
  int* host_flags = nullptr;  // pinned, mapped
  int* host_flags_dev = nullptr;
  bool profile = false;
  struct Rec {
    std::string name;
    cudaEvent_t a, b;
    double units;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  struct Acc {
    double ms = 0.0;
    long count = 0;
    double units = 0.0;
  };
  std::map<std::string, Acc> totals;
  long launches = 0;  // kernels issued by the library (approximate: per host call site)
  // dense m x n passes with U: 0 auto (INT8 tensor-core Ozaki path when t_pad <= 64), 1 DMMA fp64, 2 Ozaki
  int gemm_mode = 0;
  // per-column iteration counts and residual-norm histories of the last PCG solve on this
  // context (fsa_ctx_last_cg: parity diagnostics)
  std::vector<int> last_cg_iterations;
  std::vector<std::vector<double>> last_cg_rnorm;

  explicit Context(int dev);
  ~Context();
  cudaEvent_t ev();
  void flush_timers();  // synchronises the stream
  void sync();
};

// RAII event pair around a kernel group when profiling is on
struct KTimer {
  Context* c;
  size_t idx = static_cast<size_t>(-1);
  KTimer(Context* ctx, const char* name, double units = 0.0);
  ~KTimer();
};

struct Params {
  int nu = 1;          // 0: 1/2, 1: 3/2, 2: 5/2
  int family = 1;      // 1: wendland1, 2: wendland2
  double gamma = 0.1;  // taper range
  double sigma2 = 1.0, sigma1_2 = 1.0, rho = 0.1;
  double jitter_rel = 1e-10;
};

// Parameter-independent geometry: sorted points and the taper pattern. The
// reference rebuilds it on every evaluation (fsa.cpp:37, estimation.cpp:260);
// here it is built once and shared by every Model assembled on it.
struct Geometry {
  SortedPoints pts;   // all points, global internal (Hilbert) order
  Csr pat;            // this rank's rows; columns in extended (local | halo) indexing
  ShardPlan shard;    // row block, halo and exchange plan (trivial for one rank)
  double gamma = 0.0;
  const double* coords_ext() const { return shard.world > 1 ? shard.coords_ext.get() : pts.coords.get(); }
  std::vector<double> coords_host;  // original order, n x d column-major
  // Fit-loop residency: the response [y | X] and the FITC probe
  // draws e1/e2 are parameter independent, so a fit keeps them in HBM.
  std::vector<double> resp_host;    // n x (1 + p), original order
  DBuf<double> resp_dev;            // same on the device
  long resp_p = -1;
  bool cache_probes = false;
  struct ProbeCache {
    bool valid = false;
    unsigned long long seed = 0;
    int L = 0;
    long tp = 0, m = 0;
    DBuf<double> E1, E2;
  } probes;
};
std::shared_ptr<Geometry> make_geometry(Context* ctx, const double* coords, long n, int d, double gamma);

class Model {
 public:
  Context* ctx = nullptr;
  std::shared_ptr<Geometry> geo;
  Params P;
  long n = 0, m = 0, n_pad = 0, m_pad = 0;  // n, n_pad: rows owned by this rank
  long n_ext_pad = 0;  // owned + halo points (U, U1, T and gathered RHS blocks have this many rows)
  long cols_hint = 0;  // real RHS columns of the running solve (timer units)
  int d = 2;
  std::vector<double> ind_host;  // m x d column-major
  DBuf<double> ind;              // same, device
  DBuf<double> Sm, L;            // Sigma_m (+jitter), its Cholesky factor (col-major, m_pad^2)
  double logdet_sigma_m = 0.0;
  DBuf<double> U;                // m_pad x n_pad, one column per point
  DBuf<double> lowrank;          // |U_i|^2
  DBuf<double> sval;             // Sigma_s values on geo->pat
  DBuf<double> gval;             // the same as the stored value tiles of the row groups (32 x Csr::ntiles)
  DBuf<double> D, Dinv, sqrtD;   // diag(Sigma_s) (FITC / Jacobi diagonal)
  long n_clamped = 0;
  // rho derivative blocks (lazy, fsa.cpp:101-124)
  bool have_rho = false;
  DBuf<double> U1, T, K2, dsval, dD;
  // scratch
  DBuf<double> red_scratch, dot_scratch, dinv_scratch, mt1, mt2;
  DBuf<int> info;

  static std::unique_ptr<Model> assemble(Context* ctx, std::shared_ptr<Geometry> geo, const double* inducing, long m,
                                         const Params& p);
  // rho-derivative blocks: built synchronously on first use, or started on the side stream by
  // start_rho_derivs and joined by the next ensure_rho_derivs
  void ensure_rho_derivs();
  void start_rho_derivs();
  void build_rho_derivs(cudaStream_t s, double* trsm_scratch, bool side);
  bool rho_pending = false;
  cudaEvent_t rho_done = nullptr;
  DBuf<double> rho_scratch;
  ~Model();
  // device, internal layout (row-major n_pad x tp)
  void matmat(const double* H, double* V, long tp);
  void sigma_s_mat(const double* H, double* V, long tp, double alpha = 1.0, double beta = 0.0);
  void deriv_matmat(int which, const double* V, double* out, long tp);
  // m_pad x tp projection U V (deterministic split-K), summed over ranks
  void project(const double* M, const double* V, long tp, double* out, const double* scale = nullptr);
  // n_pad x tp block U^T W for W m_pad x tp (ld tp)
  void expand(const double* W, long tp, double* Y);
  double* mt_buf(int which, long tp);
  // refresh the halo rows [n_pad, n_pad + n_halo) of an extended block (no-op on one rank)
  void halo_exchange(double* X, long tp);
  void cross_cov_ext(int mode, double* out, cudaStream_t s = nullptr);
  int world() const { return rcomm->size(); }
  Comm* rcomm = nullptr;  // sums over the row blocks: ctx->comm when row-sharded, else a no-op
  DBuf<double> halo_send;
  // INT8 digit planes of U for the tensor-core projection / expansion (built lazily)
  OzakiPlan oz;
  bool use_ozaki(long tp) const { return ctx->gemm_mode != 1 && ozaki_supported(tp); }
  void ensure_ozaki();
  void start_ozaki();
  bool oz_pending = false;
  cudaEvent_t oz_done = nullptr;
};

// ---- preconditioners (preconditioners.h:16-115) ------------------------------------------
class Precond {
 public:
  virtual ~Precond() = default;
  virtual int kind() const = 0;  // 0 none, 1 diagonal, 2 fitc
  virtual void solve(const double* R, double* Z, long tp) = 0;
  virtual double logdet() const = 0;
  // probes keyed by (seed, i): writes n_pad x tp internal-layout block, columns [0, L)
  virtual void sample_probes(int L, unsigned long long seed, double* Z, long tp) = 0;
  virtual bool has_derivs() const { return false; }
};

class IdentityPrecond final : public Precond {
 public:
  explicit IdentityPrecond(Model* m) : md(m) {}
  int kind() const override { return 0; }
  void solve(const double* R, double* Z, long tp) override;
  double logdet() const override { return 0.0; }
  void sample_probes(int L, unsigned long long seed, double* Z, long tp) override;
  Model* md;
};

class DiagPrecond final : public Precond {
 public:
  explicit DiagPrecond(Model* m, bool derivs);
  int kind() const override { return 1; }
  void solve(const double* R, double* Z, long tp) override;
  double logdet() const override { return ld; }
  void sample_probes(int L, unsigned long long seed, double* Z, long tp) override;
  bool has_derivs() const override { return derivs; }
  Model* md;
  double ld = 0.0;
  bool derivs = false;
};

class FitcPrecond final : public Precond {
 public:
  FitcPrecond(Model* m, bool with_derivs);
  int kind() const override { return 2; }
  void solve(const double* R, double* Z, long tp) override;
  double logdet() const override { return ld; }
  void sample_probes(int L, unsigned long long seed, double* Z, long tp) override;
  bool has_derivs() const override { return derivs; }
  // exact Tr(P^{-1} dP_k), k = 0, 1, 2 (preconditioners.cpp:106-115, U-form)
  double deriv_trace(int k);
  Model* md;
  DBuf<double> Q, LQ, Qinv;  // I + U D^{-1} U^T, its factor, its inverse
  double ld = 0.0, logdetQ = 0.0;
  bool derivs = false;
  bool have_traces = false;
  double trace[3] = {0, 0, 0};
  // the exact traces' device work, on the side stream after the rho-derivative build
  void start_traces();
  void finish_traces(const double* hs);
  bool traces_pending = false;
  cudaEvent_t traces_done = nullptr;
  double* traces_host = nullptr;  // pinned [8]
  DBuf<double> tr_q, tr_f, tr_pinv, tr_d1, tr_sums;
  ~FitcPrecond() override;
};

std::unique_ptr<Precond> make_preconditioner(Model* md, int type);

// ---- Krylov ---------------------------------------------------------------------------------
struct CgOptions {
  double tol = 1e-3;
  int max_iter = 1000;
  bool error_on_max_iter = false;
};
struct CgResult {
  std::vector<int> iterations;
  std::vector<int> converged;
  std::vector<std::vector<double>> tdiag, toff;
  std::vector<std::vector<double>> rnorm;  // ||r||_2 after each iteration, per column
  int sweeps = 0;
  bool all_converged() const;
  int max_iterations() const;
};
struct LinOp {
  virtual ~LinOp() = default;
  virtual void apply(const double* H, double* V, long tp) = 0;
};

// the full FSA operator (krylov.cpp:10-16) and the short-range block alone (prediction.cpp:90-93)
struct FsaOp final : LinOp {
  Model* md;
  explicit FsaOp(Model* m) : md(m) {}
  void apply(const double* H, double* V, long tp) override { md->matmat(H, V, tp); }
};
struct SigmaSOp final : LinOp {
  Model* md;
  explicit SigmaSOp(Model* m) : md(m) {}
  void apply(const double* H, double* V, long tp) override { md->sigma_s_mat(H, V, tp); }
};

// Lockstep multi-RHS PCG (krylov.cpp:18-106) on device blocks B, X (n_pad x tp, internal).
CgResult pcg_solve_multi(Model* md, LinOp& A, Precond& P, const double* B, long k, long tp, double* X,
                         const CgOptions& opts);
double tridiag_log_quadrature(const std::vector<double>& diag, const std::vector<double>& off);

struct NllResult {
  double nll = 0.0, grad[3] = {0, 0, 0}, logdet = 0.0;
  int cg_iterations = 0;
  std::vector<double> beta;
  // diagnostics
  double pcg_ms = 0.0, total_ms = 0.0;
  long rhs_iterations = 0;
  int sweeps = 0;
};
// iterative_nll_grad (estimation.cpp:178-227); y (n), X (n x p) host, original order
NllResult iterative_nll_grad(Model* md, Precond& P, const double* y, const double* X, long p, int num_probes,
                             unsigned long long seed, const CgOptions& cg, int cv_mode, bool want_grad);

// fisher_ste (fsa.cpp:284-301): F = sym( sum_i A_i^T T_i ) / (2 L) with, per probe z_i,
// A_i = [dSigma_k Sigma^{-1} z_i]_k and T_i = [Sigma^{-1} dSigma_k z_i]_k. The reference solves
// with its exact (sparse LDLT) backend; here every solve is one batched FITC-PCG run (L, then
// 3 L columns) to the caller's tolerance. F is 3 x 3 column-major.
struct FisherResult {
  double F[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  int cg_iterations = 0;  // max over both solves
  int sweeps = 0;         // sum over both solves
};
FisherResult fisher_ste(Model* md, Precond& P, int L, unsigned long long seed, bool rademacher, const CgOptions& cg);

// ---- host RNG identical to the reference (types.h:104-129) ------------------------------------
unsigned long long splitmix64(unsigned long long x);
void probe_gaussian(unsigned long long seed, unsigned long long i, long n1, double* e1, long n2, double* e2);
void probe_rademacher(unsigned long long seed, unsigned long long i, long n, double* z);

}  // namespace fsa
