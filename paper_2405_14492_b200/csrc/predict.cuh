// Prediction on the device (reference prediction.cpp:7-172), U-form:
//   C = Sigma_m^{-1} Sigma_mnp = L^{-T} Up,  Up = L^{-1} Sigma_mnp
//   Sigma_np^T u = Sigma_s_np^T u + C^T Sigma_mn u = Sigma_s_np^T u + Up^T (U u)
#pragma once

#include <memory>

#include "fsa_core.cuh"
#include "pattern.cuh"

namespace fsa {

struct PredictionSet {
  Model* md = nullptr;
  long np = 0, np_pad = 0;
  SortedPoints pts;      // prediction points, own internal order
  DBuf<double> Up;       // m_pad x np_pad, one column per prediction point
  Csr rows;              // training (rows) x prediction (cols): Sigma_s_np
  Csr cols;              // prediction (rows) x training (cols): Sigma_s_np^T
  DBuf<double> vrow, vcol;
};

struct PredVarInfo {
  int clamped = 0, cg_iterations = 0;
  double det_ms = 0.0, sim_ms = 0.0;
};

std::unique_ptr<PredictionSet> make_prediction_set(Model* md, const double* pcoords, long np);
// host in/out, caller order
void cross_apply_t(PredictionSet& pr, const double* u, double* out);
void predict_mean_iterative(PredictionSet& pr, const double* resid, Precond& P, const CgOptions& cg, double* mean);
PredVarInfo predict_var_sim(PredictionSet& pr, int num_probes, unsigned long long seed, const CgOptions& cg,
                            const CgOptions& cg_s, bool control_variate, double floor_rel, double* var, double* se);
void deterministic_pieces_host(PredictionSet& pr, const CgOptions& cg, const CgOptions& cg_s, double* d1, double* d2,
                               double* d3, int* cg_iterations);

}  // namespace fsa
