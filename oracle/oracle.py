"""TEST INFRASTRUCTURE ONLY — ctypes front-end of the CPU oracle.

The oracle (oracle/fsa_oracle.cpp) restates the reference's FSA iterative path
(/root/reference/proj) in plain C++. Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module; the
product package never does.

Arrays follow the reference's Eigen conventions: dense matrices column-major
(numpy order="F"), CSR with int32 column indices and sorted columns per row.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libfsa_oracle.so")
_lib = None

dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="F_CONTIGUOUS")
ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
vp = C.c_void_p

NU_CODE = {0.5: 0, 1.5: 1, 2.5: 2}
CV_CODE = {"none": 0, "one": 1, "optimal": 2}
PRECOND_CODE = {"none": 0, "diagonal": 1, "fitc": 2}


class NumericalError(RuntimeError):
    """Mirror of fsagp::NumericalError (types.h:22-25)."""


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_splitmix64": (C.c_uint64, [C.c_uint64]),
            "orc_probe_gaussian": (None, [C.c_uint64, C.c_uint64, C.c_long, dp, C.c_long, dp]),
            "orc_probe_rademacher": (None, [C.c_uint64, C.c_uint64, C.c_long, dp]),
            "orc_mt19937_64_nth": (C.c_uint64, [C.c_uint64, C.c_long]),
            "orc_matern": (C.c_double, [C.c_double, C.c_int, C.c_double, C.c_double]),
            "orc_matern_drho": (C.c_double, [C.c_double, C.c_int, C.c_double, C.c_double]),
            "orc_taper_value": (C.c_double, [C.c_double, C.c_int, C.c_double]),
            "orc_rho_for_correlation_at": (C.c_double, [C.c_double, C.c_double, C.c_int]),
            "orc_effective_range": (C.c_double, [C.c_double, C.c_int]),
            "orc_gamma_for_avg_row_nnz": (C.c_double, [C.c_long, C.c_double]),
            "orc_uniform_locations": (C.c_int, [C.c_long, C.c_int, C.c_uint64, dp]),
            "orc_select_random": (C.c_int, [dp, C.c_long, C.c_int, C.c_long, C.c_uint64, dp]),
            "orc_select_kmeanspp": (C.c_int, [dp, C.c_long, C.c_int, C.c_long, C.c_uint64, C.c_int, C.c_double, dp]),
            "orc_taper_pattern": (C.c_int, [dp, C.c_long, C.c_int, C.c_double, vp, C.c_long, C.POINTER(vp), C.POINTER(C.c_long)]),
            "orc_csr_copy": (None, [vp, lp, ip, dp]),
            "orc_csr_free": (None, [vp]),
            "orc_assemble": (C.c_int, [dp, C.c_long, C.c_int, dp, C.c_long, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_double, C.POINTER(vp)]),
            "orc_model_free": (None, [vp]),
            "orc_model_info": (None, [vp, dp]),
            "orc_model_csr": (C.c_int, [vp, C.c_int, lp, ip, dp]),
            "orc_model_dense": (C.c_int, [vp, C.c_int, dp]),
            "orc_matmat": (C.c_int, [vp, dp, C.c_long, dp]),
            "orc_deriv_matmat": (C.c_int, [vp, C.c_int, dp, C.c_long, dp]),
            "orc_make_preconditioner": (C.c_int, [vp, C.c_int, C.POINTER(vp)]),
            "orc_fitc_plain": (C.c_int, [vp, C.POINTER(vp)]),
            "orc_jacobi": (C.c_int, [vp, C.POINTER(vp)]),
            "orc_precond_free": (None, [vp]),
            "orc_precond_logdet": (C.c_double, [vp]),
            "orc_precond_kind": (C.c_int, [vp]),
            "orc_precond_solve_mat": (C.c_int, [vp, dp, C.c_long, dp]),
            "orc_precond_solve_cols": (C.c_int, [vp, dp, C.c_long, dp]),
            "orc_precond_sample_probes": (C.c_int, [vp, C.c_int, C.c_uint64, dp]),
            "orc_precond_deriv_apply": (C.c_int, [vp, C.c_int, dp, dp]),
            "orc_precond_deriv_trace": (C.c_int, [vp, C.c_int, C.POINTER(C.c_double)]),
            "orc_pcg": (C.c_int, [vp, C.c_int, vp, dp, C.c_long, C.c_double, C.c_int, C.c_int, dp, ip, ip, dp, dp,
                                  C.POINTER(C.c_int)]),
            "orc_tridiag_log_quadrature": (C.c_int, [dp, dp, C.c_long, C.POINTER(C.c_double)]),
            "orc_iterative_nll_grad": (C.c_int, [vp, vp, dp, dp, C.c_long, C.c_int, C.c_uint64, C.c_double, C.c_int,
                                                 C.c_int, C.c_int, dp, dp]),
            "orc_iterative_nll_grad_ex": (C.c_int, [vp, vp, dp, dp, C.c_long, C.c_int, C.c_uint64, C.c_double,
                                                    C.c_int, C.c_int, C.c_int, dp, dp, ip, dp, lp, C.c_long, dp]),
            "orc_pcg_ex": (C.c_int, [vp, C.c_int, vp, dp, C.c_long, C.c_double, C.c_int, C.c_int, dp, ip, ip, dp,
                                     dp, dp, C.POINTER(C.c_int)]),
            "orc_simulate_rff": (C.c_int, [dp, C.c_long, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                           C.c_int, C.c_uint64, dp]),
            "orc_blob_locations": (C.c_int, [C.c_long, C.c_int, C.c_int, C.c_double, C.c_uint64, dp]),
            "orc_ste_grad_trace": (C.c_int, [vp, vp, dp, dp, C.c_long, C.c_int, C.c_int, dp]),
            "orc_pred_make": (C.c_int, [vp, dp, C.c_long, C.POINTER(vp), C.POINTER(C.c_long)]),
            "orc_pred_free": (None, [vp]),
            "orc_pred_csr": (C.c_int, [vp, lp, ip, dp]),
            "orc_cross_apply_t": (C.c_int, [vp, vp, dp, dp]),
            "orc_predict_mean_iterative": (C.c_int, [vp, vp, dp, vp, C.c_double, C.c_int, dp]),
            "orc_predict_var_sim": (C.c_int, [vp, vp, C.c_int, C.c_uint64, C.c_double, C.c_int, C.c_double, C.c_int,
                                              C.c_int, C.c_double, dp, dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "orc_pred_sample_timing": (C.c_int, [vp, vp, C.c_long, C.c_int, C.c_uint64, C.c_double, C.c_int,
                                                 C.c_double, C.c_int, dp]),
            "orc_pred_det_pieces": (C.c_int, [vp, vp, C.c_double, C.c_int, C.c_double, C.c_int, dp, dp, dp,
                                              C.POINTER(C.c_int)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 2:
        raise ValueError(msg)
    if rc == 3:
        raise NumericalError(msg)
    raise RuntimeError(msg)


def F(a, dtype=np.float64):
    return np.asfortranarray(np.asarray(a, dtype=dtype))


# ---- scalar kernels / RNG -------------------------------------------------------
def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(x))


def matern(d, nu, s1, rho):
    return lib().orc_matern(d, NU_CODE[nu], s1, rho)


def matern_drho(d, nu, s1, rho):
    return lib().orc_matern_drho(d, NU_CODE[nu], s1, rho)


def taper_value(d, family, gamma):
    return lib().orc_taper_value(d, family, gamma)


def rho_for_correlation_at(dist, corr, nu):
    return lib().orc_rho_for_correlation_at(dist, corr, NU_CODE[nu])


def effective_range(rho, nu):
    return lib().orc_effective_range(rho, NU_CODE[nu])


def gamma_for_avg_row_nnz(n, target):
    return lib().orc_gamma_for_avg_row_nnz(n, target)


def probe_gaussian(seed, i, n1, n2):
    e1 = F(np.zeros(max(n1, 1)))
    e2 = F(np.zeros(max(n2, 1)))
    lib().orc_probe_gaussian(seed, i, n1, e1, n2, e2)
    return e1[:n1], e2[:n2]


def probe_rademacher(seed, i, n):
    z = F(np.zeros(n))
    lib().orc_probe_rademacher(seed, i, n, z)
    return z


def uniform_locations(n, d, seed):
    out = F(np.zeros((n, d)))
    _check(lib().orc_uniform_locations(n, d, seed, out))
    return out


def select_random(coords, m, seed):
    c = F(coords)
    out = F(np.zeros((m, c.shape[1])))
    _check(lib().orc_select_random(c, c.shape[0], c.shape[1], m, seed, out))
    return out


def select_kmeanspp(coords, m, seed, max_iter=20, rel_tol=1e-4):
    c = F(coords)
    out = F(np.zeros((m, c.shape[1])))
    _check(lib().orc_select_kmeanspp(c, c.shape[0], c.shape[1], m, seed, max_iter, rel_tol, out))
    return out


def _csr_from(handle, nnz, rows):
    ptr = np.zeros(rows + 1, np.int64)
    idx = np.zeros(max(nnz, 1), np.int32)
    val = F(np.zeros(max(nnz, 1)))
    lib().orc_csr_copy(handle, ptr, idx, val)
    lib().orc_csr_free(handle)
    return ptr, idx[:nnz], val[:nnz]


def taper_pattern(coords, gamma):
    c = F(coords)
    h = vp()
    nnz = C.c_long()
    _check(lib().orc_taper_pattern(c, c.shape[0], c.shape[1], gamma, None, 0, C.byref(h), C.byref(nnz)))
    return _csr_from(h, nnz.value, c.shape[0])


def cross_taper_pattern(rows, cols, gamma):
    r, c = F(rows), F(cols)
    h = vp()
    nnz = C.c_long()
    _check(lib().orc_taper_pattern(r, r.shape[0], r.shape[1], gamma, c.ctypes.data_as(vp), c.shape[0],
                                   C.byref(h), C.byref(nnz)))
    return _csr_from(h, nnz.value, r.shape[0])


def tridiag_log_quadrature(diag, off):
    d = F(diag)
    o = F(off) if len(off) else F(np.zeros(1))
    out = C.c_double()
    _check(lib().orc_tridiag_log_quadrature(d, o, len(d), C.byref(out)))
    return out.value


# ---- model / preconditioner / solvers ---------------------------------------------
class Model:
    """Oracle mirror of fsagp::FsaModel (fsa.h:40-104)."""

    def __init__(self, coords, inducing, nu=1.5, taper_family=1, gamma=0.1, sigma2=1.0, sigma1_2=1.0,
                 rho=0.1, jitter_rel=1e-10):
        self.coords = F(coords)
        self.inducing = F(inducing)
        self.n, self.d = self.coords.shape
        self.m = self.inducing.shape[0]
        self.nu, self.taper_family, self.gamma = nu, taper_family, gamma
        self.sigma2, self.sigma1_2, self.rho = sigma2, sigma1_2, rho
        h = vp()
        _check(lib().orc_assemble(self.coords, self.n, self.d, self.inducing, self.m, NU_CODE[nu], taper_family,
                                  gamma, sigma2, sigma1_2, rho, jitter_rel, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_model_free(self.h)
            self.h = None

    def info(self):
        out = F(np.zeros(5))
        lib().orc_model_info(self.h, out)
        return {"n": int(out[0]), "m": int(out[1]), "nnz": int(out[2]), "n_clamped": int(out[3]),
                "logdet_sigma_m": float(out[4])}

    def csr(self, which=1):
        nnz = self.info()["nnz"]
        ptr = np.zeros(self.n + 1, np.int64)
        idx = np.zeros(nnz, np.int32)
        val = F(np.zeros(nnz))
        _check(lib().orc_model_csr(self.h, which, ptr, idx, val))
        return ptr, idx, val

    def dense(self, which):
        shapes = {0: (self.m, self.m), 1: (self.m, self.n), 2: (self.m, self.n), 3: (self.m, self.n),
                  4: (self.m, self.n), 5: (self.m, self.n), 6: (self.n,), 7: (self.m, self.m), 8: (self.m, self.m)}
        out = F(np.zeros(shapes[which]))
        _check(lib().orc_model_dense(self.h, which, out))
        return out

    def matmat(self, V):
        V = F(V).reshape(self.n, -1, order="F")
        out = F(np.zeros_like(V))
        _check(lib().orc_matmat(self.h, V, V.shape[1], out))
        return out

    def deriv_matmat(self, which, V):
        V = F(V).reshape(self.n, -1, order="F")
        out = F(np.zeros_like(V))
        _check(lib().orc_deriv_matmat(self.h, which, V, V.shape[1], out))
        return out


class Precond:
    def __init__(self, model: Model, kind="fitc", plain=False):
        self.model = model
        h = vp()
        if kind == "jacobi":
            _check(lib().orc_jacobi(model.h, C.byref(h)))
        elif plain and kind == "fitc":
            _check(lib().orc_fitc_plain(model.h, C.byref(h)))
        else:
            _check(lib().orc_make_preconditioner(model.h, PRECOND_CODE[kind], C.byref(h)))
        self.h = h
        self.n = model.n

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_precond_free(self.h)
            self.h = None

    def logdet(self):
        return lib().orc_precond_logdet(self.h)

    def solve_mat(self, R):
        R = F(R).reshape(self.n, -1, order="F")
        out = F(np.zeros_like(R))
        _check(lib().orc_precond_solve_mat(self.h, R, R.shape[1], out))
        return out

    def solve_cols(self, R):
        R = F(R).reshape(self.n, -1, order="F")
        out = F(np.zeros_like(R))
        _check(lib().orc_precond_solve_cols(self.h, R, R.shape[1], out))
        return out

    def sample_probes(self, L, seed):
        out = F(np.zeros((self.n, L)))
        _check(lib().orc_precond_sample_probes(self.h, L, seed, out))
        return out

    def deriv_apply(self, which, v):
        v = F(v)
        out = F(np.zeros_like(v))
        _check(lib().orc_precond_deriv_apply(self.h, which, v, out))
        return out

    def deriv_trace(self, which):
        out = C.c_double()
        _check(lib().orc_precond_deriv_trace(self.h, which, C.byref(out)))
        return out.value


def pcg_solve_multi(model: Model, P: Precond, B, tol=1e-3, max_iter=1000, batched=True, op="fsa"):
    """Mirror of pcg_solve_multi (krylov.cpp:18-106); op='sigma_s' solves with Sigma_s only."""
    B = F(B).reshape(model.n, -1, order="F")
    k = B.shape[1]
    X = F(np.zeros_like(B))
    it = np.zeros(k, np.int32)
    cv = np.zeros(k, np.int32)
    td = F(np.zeros((max_iter, k)))
    to = F(np.zeros((max_iter, k)))
    sw = C.c_int()
    _check(lib().orc_pcg(model.h, 0 if op == "fsa" else 1, P.h, B, k, tol, max_iter, 1 if batched else 0, X, it, cv,
                         td, to, C.byref(sw)))
    tri = [(td[: it[j], j].copy(), to[: max(it[j] - 1, 0), j].copy()) for j in range(k)]
    return {"X": X, "iterations": it, "converged": cv.astype(bool), "tridiags": tri, "sweeps": sw.value}


def iterative_nll_grad(model: Model, P: Precond, y, X=None, num_probes=50, seed=0, tol=1e-3, max_iter=1000,
                       cv="optimal", want_grad=True):
    """Mirror of iterative_nll_grad (estimation.cpp:178-227)."""
    y = F(y)
    p = 0 if X is None else np.asarray(X).reshape(model.n, -1).shape[1]
    Xf = F(np.zeros((model.n, 1))) if p == 0 else F(np.asarray(X).reshape(model.n, p))
    out = F(np.zeros(6))
    beta = F(np.zeros(max(p, 1)))
    _check(lib().orc_iterative_nll_grad(model.h, P.h, y, Xf, p, num_probes, seed, tol, max_iter, CV_CODE[cv],
                                        1 if want_grad else 0, out, beta))
    return {"nll": out[0], "grad": out[1:4].copy(), "logdet": out[4], "cg_iterations": int(out[5]),
            "beta": beta[:p].copy()}


def iterative_nll_grad_ex(model: Model, P: Precond, y, X=None, num_probes=50, seed=0, tol=1e-3, max_iter=1000,
                          cv="optimal", want_grad=True, rows=None):
    """iterative_nll_grad plus the solve's diagnostics (tests only): per-column CG iterations,
    residual-norm histories ``rnorm[j]`` (||r||_2 after each iteration) and X at ``rows``."""
    y = F(y)
    p = 0 if X is None else np.asarray(X).reshape(model.n, -1).shape[1]
    Xf = F(np.zeros((model.n, 1))) if p == 0 else F(np.asarray(X).reshape(model.n, p))
    k = num_probes + 1 + p
    rows = np.zeros(0, np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    out = F(np.zeros(6))
    beta = F(np.zeros(max(p, 1)))
    it = np.zeros(k, np.int32)
    rn = F(np.zeros((max_iter, k)))
    xr = F(np.zeros((max(len(rows), 1), k)))
    _check(lib().orc_iterative_nll_grad_ex(model.h, P.h, y, Xf, p, num_probes, seed, tol, max_iter, CV_CODE[cv],
                                           1 if want_grad else 0, out, beta, it, rn, rows, len(rows), xr))
    return {"nll": out[0], "grad": out[1:4].copy(), "logdet": out[4], "cg_iterations": int(out[5]),
            "beta": beta[:p].copy(), "iterations": it, "rnorm": [rn[: it[j], j].copy() for j in range(k)],
            "xrows": xr[: len(rows)].copy()}


def pcg_solve_multi_ex(model: Model, P: Precond, B, tol=1e-3, max_iter=1000, op="fsa"):
    """pcg_solve_multi plus the per-column residual-norm histories (tests only)."""
    B = F(B).reshape(model.n, -1, order="F")
    k = B.shape[1]
    X = F(np.zeros_like(B))
    it = np.zeros(k, np.int32)
    cv = np.zeros(k, np.int32)
    td, to, rn = (F(np.zeros((max_iter, k))) for _ in range(3))
    sw = C.c_int()
    _check(lib().orc_pcg_ex(model.h, 0 if op == "fsa" else 1, P.h, B, k, tol, max_iter, 1, X, it, cv, td, to, rn,
                            C.byref(sw)))
    tri = [(td[: it[j], j].copy(), to[: max(it[j] - 1, 0), j].copy()) for j in range(k)]
    return {"X": X, "iterations": it, "converged": cv.astype(bool), "tridiags": tri, "sweeps": sw.value,
            "rnorm": [rn[: it[j], j].copy() for j in range(k)]}


def simulate_rff(coords, nu, sigma1_2, rho, nugget, features=1024, seed=0):
    """Synthetic response of the BASELINE configs: RFF Matern draw + N(0, nugget) noise."""
    c = F(coords)
    n, d = c.shape
    y = F(np.zeros(n))
    _check(lib().orc_simulate_rff(c, n, d, NU_CODE[nu], sigma1_2, rho, nugget, features, seed, y))
    return y


def blob_locations(n, d, blobs, sd, seed):
    """Config-5 locations: mixture of seeded Gaussian blobs on [0,1]^d (points outside rejected)."""
    out = F(np.zeros((n, d)))
    _check(lib().orc_blob_locations(n, d, blobs, sd, seed, out))
    return out


def ste_grad_trace(model, P, Z, W, which, mode="optimal"):
    Z, W = F(Z), F(W)
    out = F(np.zeros(3))
    _check(lib().orc_ste_grad_trace(model.h, P.h, Z, W, Z.shape[1], which, CV_CODE[mode], out))
    return {"value": out[0], "c_hat": out[1], "variance_of_mean": out[2]}


class PredictionSet:
    """Oracle mirror of make_prediction_set (prediction.cpp:7-27)."""

    def __init__(self, model: Model, pcoords):
        self.model = model
        self.pcoords = F(pcoords)
        self.np = self.pcoords.shape[0]
        h = vp()
        nnz = C.c_long()
        _check(lib().orc_pred_make(model.h, self.pcoords, self.np, C.byref(h), C.byref(nnz)))
        self.h, self.nnz = h, nnz.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_pred_free(self.h)
            self.h = None

    def csr(self):
        ptr = np.zeros(self.model.n + 1, np.int64)
        idx = np.zeros(self.nnz, np.int32)
        val = F(np.zeros(self.nnz))
        _check(lib().orc_pred_csr(self.h, ptr, idx, val))
        return ptr, idx, val

    def cross_apply_t(self, u):
        out = F(np.zeros(self.np))
        _check(lib().orc_cross_apply_t(self.model.h, self.h, F(u), out))
        return out

    def predict_mean_iterative(self, resid, P: Precond, tol=1e-3, max_iter=1000):
        out = F(np.zeros(self.np))
        _check(lib().orc_predict_mean_iterative(self.model.h, self.h, F(resid), P.h, tol, max_iter, out))
        return out

    def det_pieces(self, tol=1e-3, max_iter=1000, tol_s=1e-3, max_iter_s=1000):
        d1, d2, d3 = (F(np.zeros(self.np)) for _ in range(3))
        it = C.c_int()
        _check(lib().orc_pred_det_pieces(self.model.h, self.h, tol, max_iter, tol_s, max_iter_s, d1, d2, d3,
                                         C.byref(it)))
        return d1, d2, d3, it.value

    def sample_timing(self, cols=16, probes=256, seed=0, tol=1e-3, max_iter=1000, tol_s=1e-3, max_iter_s=1000):
        """Seconds for cols columns of the two m-RHS solves and for one simulation batch."""
        out = F(np.zeros(3))
        _check(lib().orc_pred_sample_timing(self.model.h, self.h, cols, probes, seed, tol, max_iter, tol_s, max_iter_s,
                                            out))
        return {"x1": out[0], "x2": out[1], "batch": out[2]}

    def predict_var_sim(self, num_probes=1000, seed=0, tol=1e-3, max_iter=1000, tol_s=1e-3, max_iter_s=1000,
                        control_variate=False, floor_rel=1e-6):
        var, se = F(np.zeros(self.np)), F(np.zeros(self.np))
        cl, it = C.c_int(), C.c_int()
        _check(lib().orc_predict_var_sim(self.model.h, self.h, num_probes, seed, tol, max_iter, tol_s, max_iter_s,
                                         1 if control_variate else 0, floor_rel, var, se, C.byref(cl), C.byref(it)))
        return {"var": var, "se": se, "clamped": cl.value, "cg_iterations": it.value}


def fisher_ste(model: Model, num_probes=50, seed=0, rademacher=False):
    """fisher_ste (fsa.cpp:284-301) restated in numpy. FsaModel::solve is the reference's exact
    backend (sparse LDLT of Sigma_s + Woodbury, fsa.cpp:196-223); for the small sizes the oracle
    serves, a dense Cholesky of the same Sigma (= matmat of the identity) is that solve."""
    import scipy.linalg as sla

    if num_probes <= 0:
        raise ValueError("need at least one probe")  # fsa.cpp:285
    n = model.n
    S = model.matmat(np.eye(n))
    cf = sla.cho_factor(0.5 * (S + S.T), lower=True)
    F_ = np.zeros((3, 3))
    for i in range(num_probes):
        z = probe_rademacher(seed, i, n) if rademacher else probe_gaussian(seed, i, 0, n)[1]
        w = sla.cho_solve(cf, z)
        a = np.column_stack([model.deriv_matmat(k, w)[:, 0] for k in range(3)])
        t = np.column_stack([sla.cho_solve(cf, model.deriv_matmat(k, z)[:, 0]) for k in range(3)])
        F_ += a.T @ t
    F_ /= 2.0 * num_probes
    return 0.5 * (F_ + F_.T)
