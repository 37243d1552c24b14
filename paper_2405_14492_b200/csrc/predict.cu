// Prediction on the device; see predict.cuh.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "blas1.cuh"
#include "dgemm.cuh"
#include "kernels.cuh"
#include "predict.cuh"
#include "sparse.cuh"

namespace fsa {

namespace {

__global__ void k_rowdot(const double* __restrict__ A, const double* __restrict__ B, long ld, long len, long n,
                         long n_pad, double* __restrict__ out) {
  const long i = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_pad) return;
  double s = 0.0;
  if (i < n)
    for (long r = lane; r < len; r += 32) s = fma(A[i * ld + r], B[i * ld + r], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[i] = s;
}

// s[i] += sum_j z q ; s2[i] += sum_j (z q)^2   (krylov.cpp:210-213, one batch)
__global__ void k_moments(const double* __restrict__ Z, const double* __restrict__ Q, long np, long tp, long b,
                          double* __restrict__ s, double* __restrict__ s2) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= np) return;
  double a = 0.0, a2 = 0.0;
  for (long j = 0; j < b; ++j) {
    const double v = Z[i * tp + j] * Q[i * tp + j];
    a += v;
    a2 += v * v;
  }
  s[i] += a;
  s2[i] += a2;
}

__global__ void k_moments_cv(const double* __restrict__ Z, const double* __restrict__ Q,
                             const double* __restrict__ Qc, long np, long tp, long b, double* __restrict__ acc) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= np) return;
  double ra = 0, ra2 = 0, rb = 0, rb2 = 0, rab = 0;
  for (long j = 0; j < b; ++j) {
    const double z = Z[i * tp + j];
    const double va = z * Q[i * tp + j], vb = z * Qc[i * tp + j];
    ra += va;
    ra2 += va * va;
    rb += vb;
    rb2 += vb * vb;
    rab += va * vb;
  }
  acc[0 * np + i] += ra;
  acc[1 * np + i] += ra2;
  acc[2 * np + i] += rb;
  acc[3 * np + i] += rb2;
  acc[4 * np + i] += rab;
}

// control diagonal: sum_r S_np(r, j)^2 / ds(r)  over the transposed pattern rows j
__global__ void k_control_diag(const long* __restrict__ rowptr, const int* __restrict__ col,
                               const double* __restrict__ val, const double* __restrict__ Dinv, long np,
                               double* __restrict__ out) {
  const long j = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= np) return;
  double s = 0.0;
  for (long p = rowptr[j]; p < rowptr[j + 1]; ++p) s += val[p] * val[p] * Dinv[col[p]];
  out[j] = s;
}

__global__ void k_symmetrize(double* A, long m) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= m * m) return;
  const long r = idx % m, c = idx / m;
  if (r >= c) return;
  const double v = 0.5 * (A[c * m + r] + A[r * m + c]);
  A[c * m + r] = v;
  A[r * m + c] = v;
}

inline unsigned nb(long total, int th = 256) { return static_cast<unsigned>(cdiv(total, th)); }

void rowdot(const double* A, const double* B, long ld, long len, long n, long n_pad, double* out, cudaStream_t s) {
  k_rowdot<<<nb(n_pad * 32), 256, 0, s>>>(A, B, ld, len, n, n_pad, out);
  FSA_LAUNCH_CHECK();
}

// Sigma_mn^T as an n_pad x m_pad block: U^T L^T (W(k, c) = L(c, k), L column-major)
void sigma_mn_t(Model* md, double* B) {
  gemm_expand_store(md->U.get(), md->m_pad, md->n_pad, md->m_pad, md->L.get(), md->m_pad, md->m_pad, B, md->m_pad,
                    1.0, 0.0, md->ctx->stream);
}

// device vectors (internal order) -> host caller order
void pred_to_host(PredictionSet& pr, const double* dev, double* host) {
  cudaStream_t s = pr.md->ctx->stream;
  DBuf<double> raw(static_cast<size_t>(pr.np));
  unpack_cols(dev, pr.np, 1, pr.pts.perm_d.get(), 1, 0, raw.get(), s);
  FSA_CUDA(cudaMemcpyAsync(host, raw.get(), sizeof(double) * pr.np, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
}

struct DetDev {
  DBuf<double> d1, d2, d3;
  int cg_iterations = 0;
};

// deterministic_pieces (prediction.cpp:72-110) in U-form
DetDev deterministic_pieces(PredictionSet& pr, const CgOptions& cg, const CgOptions& cg_s) {
  Model* md = pr.md;
  Context* ctx = md->ctx;
  cudaStream_t s = ctx->stream;
  const long mp = md->m_pad, np_ = md->n_pad, npp = pr.np_pad, m = md->m;
  const long tp = mp;
  DetDev out;
  out.d1.alloc(npp);
  out.d2.alloc(npp);
  out.d3.alloc(npp);
  DBuf<double> B1(np_ * tp), X1(np_ * tp), X2(np_ * tp);
  sigma_mn_t(md, B1.get());
  // X1 = Sigma^{-1} Sigma_mn^T with FITC (no derivatives)
  FitcPrecond fitc(md, false);
  FsaOp op(md);
  CgResult r1 = pcg_solve_multi(md, op, fitc, B1.get(), m, tp, X1.get(), cg);
  if (!r1.all_converged()) throw NumericalError("prediction: cg did not converge");
  out.cg_iterations = r1.max_iterations();
  // d1_j = Up_j' E Up_j,  E = (U X1) L^{-T}
  DBuf<double> G(mp * mp), Et(mp * mp), Y(npp * mp);
  md->project(md->U.get(), X1.get(), tp, G.get());
  trsm_lower_cols(md->L.get(), mp, G.get(), mp, mp, md->dinv_scratch.get(), s);  // rows of G -> E rows
  launch_transpose(G.get(), mp, mp, mp, Et.get(), mp, s);
  gemm_expand_store(pr.Up.get(), mp, npp, mp, Et.get(), mp, mp, Y.get(), mp, 1.0, 0.0, s);
  rowdot(Y.get(), pr.Up.get(), mp, mp, pr.np, npp, out.d1.get(), s);
  // d2_j = (L^{-1} (Sigma_s_np^T X1)_j) . Up_j
  launch_spmm(pr.cols.rowptr.get(), pr.cols.col.get(), pr.vcol.get(), pr.np, X1.get(), tp, Y.get(), mp, tp, 1.0,
              0.0, s);
  trsm_lower_cols(md->L.get(), mp, Y.get(), mp, npp, md->dinv_scratch.get(), s);
  rowdot(Y.get(), pr.Up.get(), mp, mp, pr.np, npp, out.d2.get(), s);
  // X2 = Sigma_s^{-1} Sigma_mn^T with Jacobi
  DiagPrecond jac(md, false);
  SigmaSOp sop(md);
  CgResult r2 = pcg_solve_multi(md, sop, jac, B1.get(), m, tp, X2.get(), cg_s);
  if (!r2.all_converged()) throw NumericalError("prediction: cg did not converge");
  out.cg_iterations = std::max(out.cg_iterations, r2.max_iterations());
  // M' = sym(I + (U X2) L^{-T}) = L^{-1} sym(Sigma_m + Sigma_mn X2) L^{-T}
  md->project(md->U.get(), X2.get(), tp, G.get());
  trsm_lower_cols(md->L.get(), mp, G.get(), mp, mp, md->dinv_scratch.get(), s);
  add_identity(G.get(), mp, mp, s);
  k_symmetrize<<<nb(mp * mp), 256, 0, s>>>(G.get(), mp);
  FSA_LAUNCH_CHECK();
  potrf_lower(G.get(), mp, md->info.get(), md->dinv_scratch.get(), s);
  int hinfo = 0;
  FSA_CUDA(cudaMemcpyAsync(&hinfo, md->info.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  // d3_j = | L_M'^{-1} L^{-1} (Sigma_s_np^T X2)_j |^2
  launch_spmm(pr.cols.rowptr.get(), pr.cols.col.get(), pr.vcol.get(), pr.np, X2.get(), tp, Y.get(), mp, tp, 1.0,
              0.0, s);
  trsm_lower_cols(md->L.get(), mp, Y.get(), mp, npp, md->dinv_scratch.get(), s);
  FSA_CUDA(cudaStreamSynchronize(s));
  if (hinfo != 0) throw NumericalError("prediction: core matrix is not positive definite");
  trsm_lower_cols(G.get(), mp, Y.get(), mp, npp, md->dinv_scratch.get(), s);
  colnorm2(Y.get(), mp, mp, pr.np, npp, out.d3.get(), s);
  return out;
}

}  // namespace

std::unique_ptr<PredictionSet> make_prediction_set(Model* md, const double* pcoords, long np) {
  require(np > 0, "prediction: empty location set");
  Context* ctx = md->ctx;
  cudaStream_t s = ctx->stream;
  auto pr = std::make_unique<PredictionSet>();
  pr->md = md;
  pr->np = np;
  pr->np_pad = round_up(np, 128);
  const int d = md->d;
  const CellGrid g = make_grid(pcoords, np, d, md->P.gamma, nullptr, 0);
  sort_points(pcoords, np, d, g, pr->np_pad, pr->pts, s);
  const long mp = md->m_pad;
  pr->Up.alloc(mp * pr->np_pad);
  launch_cross_cov(md->ind.get(), md->m, md->m, pr->pts.coords.get(), pr->np_pad, np, pr->np_pad, d, md->P.nu,
                   md->P.sigma1_2, md->P.rho, 0, pr->Up.get(), mp, s);
  trsm_lower_cols(md->L.get(), mp, pr->Up.get(), mp, pr->np_pad, md->dinv_scratch.get(), s);
  build_pattern(md->geo->pts, pr->pts, md->P.gamma, false, pr->rows, s);
  build_pattern(pr->pts, md->geo->pts, md->P.gamma, false, pr->cols, s);
  SddmmParams sp{md->P.nu, md->P.family, md->P.sigma2, md->P.sigma1_2, md->P.rho, md->P.gamma};
  pr->vrow.alloc(pr->rows.nnz > 0 ? pr->rows.nnz : 1);
  pr->vcol.alloc(pr->cols.nnz > 0 ? pr->cols.nnz : 1);
  sddmm_cross(md->U.get(), mp, pr->Up.get(), mp, pr->rows, sp, pr->vrow.get(), s);
  sddmm_cross(pr->Up.get(), mp, md->U.get(), mp, pr->cols, sp, pr->vcol.get(), s);
  FSA_CUDA(cudaStreamSynchronize(s));
  return pr;
}

static void cross_apply_dev(PredictionSet& pr, const double* ub, long tp, double* out_blk) {
  Model* md = pr.md;
  cudaStream_t s = md->ctx->stream;
  double* W = md->mt_buf(0, tp);
  md->project(md->U.get(), ub, tp, W);
  gemm_expand_store(pr.Up.get(), md->m_pad, pr.np_pad, md->m_pad, W, tp, tp, out_blk, tp, 1.0, 0.0, s);
  launch_spmm(pr.cols.rowptr.get(), pr.cols.col.get(), pr.vcol.get(), pr.np, ub, tp, out_blk, tp, tp, 1.0, 1.0, s);
}

void cross_apply_t(PredictionSet& pr, const double* u, double* out) {
  Model* md = pr.md;
  cudaStream_t s = md->ctx->stream;
  const long tp = 8;
  DBuf<double> raw(md->n), ub(md->n_pad * tp), ob(pr.np_pad * tp), ro(pr.np);
  FSA_CUDA(cudaMemcpyAsync(raw.get(), u, sizeof(double) * md->n, cudaMemcpyHostToDevice, s));
  FSA_CUDA(cudaMemsetAsync(ub.get(), 0, sizeof(double) * md->n_pad * tp, s));
  pack_cols(raw.get(), md->n, 1, md->geo->pts.perm_d.get(), md->n_pad, tp, 0, ub.get(), s);
  cross_apply_dev(pr, ub.get(), tp, ob.get());
  unpack_cols(ob.get(), pr.np, 1, pr.pts.perm_d.get(), tp, 0, ro.get(), s);
  FSA_CUDA(cudaMemcpyAsync(out, ro.get(), sizeof(double) * pr.np, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
}

void predict_mean_iterative(PredictionSet& pr, const double* resid, Precond& P, const CgOptions& cg, double* mean) {
  Model* md = pr.md;
  cudaStream_t s = md->ctx->stream;
  const long tp = 8;
  DBuf<double> raw(md->n), B(md->n_pad * tp), X(md->n_pad * tp), ob(pr.np_pad * tp), ro(pr.np);
  FSA_CUDA(cudaMemcpyAsync(raw.get(), resid, sizeof(double) * md->n, cudaMemcpyHostToDevice, s));
  FSA_CUDA(cudaMemsetAsync(B.get(), 0, sizeof(double) * md->n_pad * tp, s));
  pack_cols(raw.get(), md->n, 1, md->geo->pts.perm_d.get(), md->n_pad, tp, 0, B.get(), s);
  FsaOp op(md);
  CgResult r = pcg_solve_multi(md, op, P, B.get(), 1, tp, X.get(), cg);
  if (!r.all_converged()) throw NumericalError("prediction: cg did not converge");
  cross_apply_dev(pr, X.get(), tp, ob.get());
  unpack_cols(ob.get(), pr.np, 1, pr.pts.perm_d.get(), tp, 0, ro.get(), s);
  FSA_CUDA(cudaMemcpyAsync(mean, ro.get(), sizeof(double) * pr.np, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
}

void deterministic_pieces_host(PredictionSet& pr, const CgOptions& cg, const CgOptions& cg_s, double* d1, double* d2,
                               double* d3, int* cg_iterations) {
  DetDev det = deterministic_pieces(pr, cg, cg_s);
  pred_to_host(pr, det.d1.get(), d1);
  pred_to_host(pr, det.d2.get(), d2);
  pred_to_host(pr, det.d3.get(), d3);
  *cg_iterations = det.cg_iterations;
}

// predict_var_sim (prediction.cpp:131-172) with stochastic_diag(_cv) (krylov.cpp:230-291)
PredVarInfo predict_var_sim(PredictionSet& pr, int L, unsigned long long seed, const CgOptions& cg,
                            const CgOptions& cg_s, bool cv, double floor_rel, double* var, double* se) {
  NvtxRange nvtx_("fsa::predict_var_sim");
  Model* md = pr.md;
  Context* ctx = md->ctx;
  cudaStream_t s = ctx->stream;
  require(L > 0, "stochastic_diag: invalid options");
  if (cv) require(L > 1, "stochastic_diag_cv: needs at least two probes");
  PredVarInfo info;
  cudaEvent_t e0 = ctx->ev(), e1 = ctx->ev(), e2 = ctx->ev();
  FSA_CUDA(cudaEventRecord(e0, s));
  DetDev det = deterministic_pieces(pr, cg, cg_s);
  FSA_CUDA(cudaEventRecord(e1, s));
  int max_it = det.cg_iterations;
  const long np = pr.np, npp = pr.np_pad, n = md->n, nP = md->n_pad;
  const int batch = 256;
  const long tpb = pad_cols(batch);
  DBuf<double> acc(static_cast<size_t>(5 * np)), Zb(npp * tpb), G(nP * tpb), Xs(nP * tpb), Q(npp * tpb),
      Qc(npp * tpb), raw(static_cast<size_t>(np) * batch), cdiag(np);
  FSA_CUDA(cudaMemsetAsync(acc.get(), 0, sizeof(double) * 5 * np, s));
  DiagPrecond jac(md, false);
  SigmaSOp sop(md);
  std::vector<double> zh(static_cast<size_t>(np) * batch);
  if (cv) {
    k_control_diag<<<nb(np), 256, 0, s>>>(pr.cols.rowptr.get(), pr.cols.col.get(), pr.vcol.get(), md->Dinv.get(), np,
                                          cdiag.get());
    FSA_LAUNCH_CHECK();
  }
  // replicated multi-GPU mode: probe batch bi runs on rank bi % world; the moment
  // sums are added over ranks below
  Comm& comm = *ctx->comm;
  const bool shard_batches = !ctx->shard_rows && comm.size() > 1;
  const int rank = shard_batches ? comm.rank() : 0, nranks = shard_batches ? comm.size() : 1;
  int done = 0;
  for (int bi = 0; done < L; ++bi) {
    const int b = std::min(batch, L - done);
    if (bi % nranks != rank) {
      done += b;
      continue;
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int j = 0; j < b; ++j)
      probe_rademacher(seed, static_cast<unsigned long long>(done + j), np, zh.data() + static_cast<long>(j) * np);
    FSA_CUDA(cudaMemcpyAsync(raw.get(), zh.data(), sizeof(double) * np * b, cudaMemcpyHostToDevice, s));
    FSA_CUDA(cudaMemsetAsync(Zb.get(), 0, sizeof(double) * npp * tpb, s));
    pack_cols(raw.get(), np, b, pr.pts.perm_d.get(), npp, tpb, 0, Zb.get(), s);
    // quad_mat: Sigma_s_np^T Sigma_s^{-1} Sigma_s_np Z  (prediction.cpp:142-148)
    FSA_CUDA(cudaMemsetAsync(G.get(), 0, sizeof(double) * nP * tpb, s));
    launch_spmm(pr.rows.rowptr.get(), pr.rows.col.get(), pr.vrow.get(), n, Zb.get(), tpb, G.get(), tpb, tpb, 1.0,
                0.0, s);
    CgResult r = pcg_solve_multi(md, sop, jac, G.get(), b, tpb, Xs.get(), cg_s);
    if (!r.all_converged()) throw NumericalError("prediction: cg did not converge");
    max_it = std::max(max_it, r.max_iterations());
    launch_spmm(pr.cols.rowptr.get(), pr.cols.col.get(), pr.vcol.get(), np, Xs.get(), tpb, Q.get(), tpb, tpb, 1.0,
                0.0, s);
    if (!cv) {
      k_moments<<<nb(np), 256, 0, s>>>(Zb.get(), Q.get(), np, tpb, b, acc.get(), acc.get() + np);
      FSA_LAUNCH_CHECK();
    } else {  // control: Sigma_s_np^T D^{-1} Sigma_s_np Z (prediction.cpp:153-157)
      scale_rows(G.get(), G.get(), md->Dinv.get(), nP, tpb, s);
      launch_spmm(pr.cols.rowptr.get(), pr.cols.col.get(), pr.vcol.get(), np, G.get(), tpb, Qc.get(), tpb, tpb, 1.0,
                  0.0, s);
      k_moments_cv<<<nb(np), 256, 0, s>>>(Zb.get(), Q.get(), Qc.get(), np, tpb, b, acc.get());
      FSA_LAUNCH_CHECK();
    }
    done += b;
  }
  if (shard_batches) {
    comm.allreduce(acc.get(), 5 * np, s);
    std::vector<double> its(static_cast<size_t>(nranks), 0.0);
    its[static_cast<size_t>(rank)] = max_it;
    comm.allreduce_host(its.data(), nranks, s);
    for (double v : its) max_it = std::max(max_it, static_cast<int>(v));
  }
  FSA_CUDA(cudaEventRecord(e2, s));
  // finish moments + combine_pieces (krylov.cpp:215-226,273-290; prediction.cpp:112-127), internal order
  std::vector<double> ha(static_cast<size_t>(5 * np)), hd1(static_cast<size_t>(np)), hd2(hd1), hd3(hd1), hcd(hd1);
  FSA_CUDA(cudaMemcpyAsync(ha.data(), acc.get(), sizeof(double) * 5 * np, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaMemcpyAsync(hd1.data(), det.d1.get(), sizeof(double) * np, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaMemcpyAsync(hd2.data(), det.d2.get(), sizeof(double) * np, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaMemcpyAsync(hd3.data(), det.d3.get(), sizeof(double) * np, cudaMemcpyDeviceToHost, s));
  if (cv) FSA_CUDA(cudaMemcpyAsync(hcd.data(), cdiag.get(), sizeof(double) * np, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  const double l = static_cast<double>(L);
  const double prior = md->P.sigma1_2 + md->P.sigma2;
  const double floor = md->P.sigma2 * floor_rel;
  for (long i = 0; i < np; ++i) {
    const long o = pr.pts.perm[static_cast<size_t>(i)];
    double dg, sev;
    if (!cv) {
      const double sm = ha[static_cast<size_t>(i)], sm2 = ha[static_cast<size_t>(np + i)];
      dg = sm / l;
      sev = 0.0;
      if (L > 1) {
        const double v = (sm2 - l * dg * dg) / (l - 1.0);
        sev = std::sqrt(std::max(v, 0.0) / l);
      }
    } else {
      const double sa = ha[static_cast<size_t>(i)], sa2 = ha[static_cast<size_t>(np + i)],
                   sb = ha[static_cast<size_t>(2 * np + i)], sb2 = ha[static_cast<size_t>(3 * np + i)],
                   sab = ha[static_cast<size_t>(4 * np + i)];
      const double ab = sa / l, bb = sb / l;
      const double va = std::max((sa2 - l * ab * ab) / (l - 1.0), 0.0);
      const double vb = std::max((sb2 - l * bb * bb) / (l - 1.0), 0.0);
      const double cab = (sab - l * (ab * bb)) / (l - 1.0);
      const double scale = std::max(std::fabs(bb), 1.0);
      const double c = vb > 1e-28 * scale * scale ? cab / vb : 0.0;
      dg = ab - c * (bb - hcd[static_cast<size_t>(i)]);
      sev = std::sqrt(std::max(va - 2.0 * c * cab + c * c * vb, 0.0) / l);
    }
    double v = prior - hd1[static_cast<size_t>(i)] - 2.0 * hd2[static_cast<size_t>(i)] + hd3[static_cast<size_t>(i)] - dg;
    if (v < floor) {
      v = floor;
      ++info.clamped;
    }
    var[o] = v;
    se[o] = sev;
  }
  info.cg_iterations = max_it;
  float a = 0.f, b2 = 0.f;
  FSA_CUDA(cudaEventElapsedTime(&a, e0, e1));
  FSA_CUDA(cudaEventElapsedTime(&b2, e1, e2));
  info.det_ms = a;
  info.sim_ms = b2;
  ctx->pool.push_back(e0);
  ctx->pool.push_back(e1);
  ctx->pool.push_back(e2);
  return info;
}

}  // namespace fsa
