"""B200-native (sm_100a, fp64) FSA iterative core — arXiv 2405.14492.

The hot path of the reference's iterative backend (FITC-preconditioned lockstep
PCG, SLQ log-determinant, STE gradient traces, simulated predictive variances)
as hand-written CUDA behind a C ABI (include/fsa_b200.h); this package is the
Python mirror of the reference's operator API over that ABI.
"""
from .fsa import (  # noqa: F401
    Context, CudaError, FsaModel, Geometry, NumericalError, Preconditioner, PredictionSet, blob_locations,
    default_context, gamma_for_avg_row_nnz, iterative_nll_grad, lib, make_prediction_set, make_preconditioner,
    pcg_solve_multi, probe_gaussian, select_kmeanspp, select_random, simulate_rff, tridiag_log_quadrature,
    uniform_locations,
)
