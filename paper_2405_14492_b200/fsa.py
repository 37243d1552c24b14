"""Python front-end of the B200 FSA iterative core (ctypes over include/fsa_b200.h).

Names and argument meanings mirror the reference's C++ API
(/root/reference/proj/include/fsagp): ``FsaModel.assemble`` (fsa.h:42-43),
``make_preconditioner`` (estimation.h:81-82), ``pcg_solve_multi`` (krylov.h:73-75),
``iterative_nll_grad`` (estimation.h:101-103), ``make_prediction_set`` /
``predict_mean_iterative`` / ``predict_var_sim`` (prediction.h:21-60). Errors
map to ``ValueError`` (std::invalid_argument) and ``NumericalError``
(fsagp::NumericalError). There is no CPU fallback: every compute call runs the
sm_100a kernels in libfsa_b200.so and raises if the library or the GPU is absent.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FSA_LIB selects another build of the same library (the bounds-checked one: make -C csrc checked)
LIB_PATH = os.environ.get("FSA_LIB") or os.path.join(_HERE, "libfsa_b200.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="F_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_i64 = C.c_int64
_u64 = C.c_uint64

NU_CODE = {0.5: 0, 1.5: 1, 2.5: 2}
PRECOND_CODE = {"none": 0, "diagonal": 1, "fitc": 2}
CV_CODE = {"none": 0, "one": 1, "optimal": 2}
FAMILY_CODE = {"wendland1": 1, "wendland2": 2, 1: 1, 2: 2}


class NumericalError(RuntimeError):
    """fsagp::NumericalError (types.h:22-25)."""


class CudaError(RuntimeError):
    """Device-side failure."""


class Params(C.Structure):
    _fields_ = [("nu_code", C.c_int), ("taper_family", C.c_int), ("gamma", C.c_double), ("sigma2", C.c_double),
                ("sigma1_2", C.c_double), ("rho", C.c_double), ("jitter_rel", C.c_double)]


class CgOptions(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("error_on_max_iter", C.c_int)]


class NllResult(C.Structure):
    _fields_ = [("nll", C.c_double), ("grad", C.c_double * 3), ("logdet", C.c_double), ("cg_iterations", C.c_int),
                ("sweeps", C.c_int), ("rhs_iterations", C.c_int64), ("pcg_ms", C.c_double),
                ("total_ms", C.c_double)]


class FitOptions(C.Structure):
    _fields_ = [("nu_code", C.c_int), ("taper_family", C.c_int), ("num_inducing", C.c_int64),
                ("taper_range", C.c_double), ("target_row_nnz", C.c_double), ("precond", C.c_int),
                ("num_probes", C.c_int), ("cv_mode", C.c_int), ("seed", C.c_uint64), ("cg_tol", C.c_double),
                ("cg_max_iter", C.c_int), ("jitter_rel", C.c_double), ("max_evals", C.c_int),
                ("lbfgs_memory", C.c_int), ("armijo_c1", C.c_double), ("max_backtracks", C.c_int),
                ("f_rel_tol", C.c_double), ("grad_tol_per_n", C.c_double)]


class FitResult(C.Structure):
    _fields_ = [("sigma2", C.c_double), ("sigma1_2", C.c_double), ("rho", C.c_double), ("nll", C.c_double),
                ("gamma", C.c_double), ("grad_log", C.c_double * 3), ("evals", C.c_int), ("converged", C.c_int),
                ("n_trace", C.c_int64)]


class PredVarInfo(C.Structure):
    _fields_ = [("clamped", C.c_int), ("cg_iterations", C.c_int), ("det_ms", C.c_double), ("sim_ms", C.c_double)]


_SIGS = {
    "fsa_last_error": (C.c_char_p, []),
    "fsa_version": (C.c_int, []),
    "fsa_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "fsa_ctx_destroy": (None, [_vp]),
    "fsa_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "fsa_ctx_create_nccl": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(_vp)]),
    "fsa_ctx_group_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(_vp)]),
    "fsa_ctx_rank": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "fsa_ctx_set_replicated": (C.c_int, [_vp, C.c_int]),
    "fsa_ctx_synchronize": (C.c_int, [_vp]),
    "fsa_ctx_set_gemm_mode": (C.c_int, [_vp, C.c_int]),
    "fsa_ctx_last_cg": (C.c_int, [_vp, C.POINTER(C.c_int64), C.c_int64, C.c_int64, _vp, _vp]),
    "fsa_debug_kernel_bench": (C.c_int, [_vp, C.c_int, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "fsa_ctx_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "fsa_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "fsa_ctx_reset_timers": (C.c_int, [_vp]),
    "fsa_ctx_timer_names": (C.c_int, [_vp, C.c_char_p, C.c_size_t]),
    "fsa_ctx_timer": (C.c_int, [_vp, C.c_char_p, C.POINTER(C.c_double), C.POINTER(_i64), C.POINTER(C.c_double)]),
    "fsa_uniform_locations": (C.c_int, [_i64, C.c_int, _u64, _dp]),
    "fsa_select_random": (C.c_int, [_dp, _i64, C.c_int, _i64, _u64, _dp]),
    "fsa_select_kmeanspp": (C.c_int, [_dp, _i64, C.c_int, _i64, _u64, C.c_int, C.c_double, _dp]),
    "fsa_select_kmeanspp_device": (C.c_int, [_vp, _dp, _i64, C.c_int, _i64, _u64, C.c_int, C.c_double, _dp]),
    "fsa_gamma_for_avg_row_nnz": (C.c_double, [_i64, C.c_double]),
    "fsa_simulate_rff": (C.c_int, [_dp, _i64, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, _u64,
                                   _dp]),
    "fsa_blob_locations": (C.c_int, [_i64, C.c_int, C.c_int, C.c_double, _u64, _dp]),
    "fsa_probe_gaussian": (C.c_int, [_u64, _u64, _i64, _dp, _i64, _dp]),
    "fsa_probe_rademacher": (C.c_int, [_u64, _u64, _i64, _dp]),
    "fsa_geometry_create": (C.c_int, [_vp, _dp, _i64, C.c_int, C.c_double, C.POINTER(_vp)]),
    "fsa_geometry_destroy": (None, [_vp]),
    "fsa_geometry_info": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64)]),
    "fsa_geometry_pattern": (C.c_int, [_vp, _lp, _ip, _dp]),
    "fsa_geometry_shard_info": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]),
    "fsa_geometry_permutation": (C.c_int, [_vp, _ip]),
    "fsa_geometry_set_response": (C.c_int, [_vp, _dp, _vp, _i64]),
    "fsa_geometry_cache_probes": (C.c_int, [_vp, C.c_int]),
    "fsa_launch_count": (C.c_int64, []),
    "fsa_model_assemble": (C.c_int, [_vp, _dp, _i64, C.c_int, _dp, _i64, C.POINTER(Params), C.POINTER(_vp)]),
    "fsa_model_assemble_geo": (C.c_int, [_vp, _dp, _i64, C.POINTER(Params), C.POINTER(_vp)]),
    "fsa_model_destroy": (None, [_vp]),
    "fsa_model_info": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64),
                                 C.POINTER(C.c_double)]),
    "fsa_model_sigma_s": (C.c_int, [_vp, C.c_int, _lp, _ip, _dp]),
    "fsa_model_matmat": (C.c_int, [_vp, _dp, _i64, _dp]),
    "fsa_model_deriv_matmat": (C.c_int, [_vp, C.c_int, _dp, _i64, _dp]),
    "fsa_model_diagonals": (C.c_int, [_vp, _dp, _dp]),
    "fsa_model_lowrank_project": (C.c_int, [_vp, _dp, _i64, _dp]),
    "fsa_model_lowrank_expand": (C.c_int, [_vp, _dp, _i64, _dp]),
    "fsa_make_preconditioner": (C.c_int, [_vp, C.c_int, C.POINTER(_vp)]),
    "fsa_make_jacobi": (C.c_int, [_vp, C.POINTER(_vp)]),
    "fsa_precond_destroy": (None, [_vp]),
    "fsa_precond_logdet": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "fsa_precond_solve_mat": (C.c_int, [_vp, _dp, _i64, _dp]),
    "fsa_precond_sample_probes": (C.c_int, [_vp, C.c_int, _u64, _dp]),
    "fsa_precond_deriv_trace": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_double)]),
    "fsa_pcg_solve_multi": (C.c_int, [_vp, _vp, C.c_int, _dp, _i64, C.POINTER(CgOptions), _dp, _ip, _ip, _dp, _dp,
                                      C.POINTER(C.c_int)]),
    "fsa_tridiag_log_quadrature": (C.c_int, [_dp, _dp, _i64, C.POINTER(C.c_double)]),
    "fsa_iterative_nll_grad": (C.c_int, [_vp, _vp, _vp, _vp, _i64, C.c_int, _u64, C.POINTER(CgOptions), C.c_int,
                                         C.c_int, C.POINTER(NllResult), _vp]),
    "fsa_fisher_ste": (C.c_int, [_vp, _vp, C.c_int, _u64, C.c_int, C.POINTER(CgOptions), _dp,
                                 C.POINTER(C.c_int)]),
    "fsa_pred_setup": (C.c_int, [_vp, _dp, _i64, C.POINTER(_vp)]),
    "fsa_fit_options_default": (None, [C.POINTER(FitOptions)]),
    "fsa_fit": (C.c_int, [_vp, _dp, _i64, C.c_int, _dp, _vp, _i64, C.POINTER(FitOptions), C.POINTER(FitResult),
                          _vp, _dp, _dp, _i64]),
    "fsa_pred_destroy": (None, [_vp]),
    "fsa_pred_info": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64)]),
    "fsa_cross_apply_t": (C.c_int, [_vp, _dp, _dp]),
    "fsa_predict_mean_iterative": (C.c_int, [_vp, _dp, _vp, C.POINTER(CgOptions), _dp]),
    "fsa_predict_var_sim": (C.c_int, [_vp, C.c_int, _u64, C.POINTER(CgOptions), C.POINTER(CgOptions), C.c_int,
                                      C.c_double, _dp, _dp, C.POINTER(PredVarInfo)]),
    "fsa_pred_det_pieces": (C.c_int, [_vp, C.POINTER(CgOptions), C.POINTER(CgOptions), _dp, _dp, _dp,
                                      C.POINTER(C.c_int)]),
}


def _destroy(fn, h):
    """Handle release from __del__: skipped at interpreter shutdown, when the module globals are
    already torn down (the process exit releases the device state)."""
    if _lib is None or _SIGS is None:
        return
    getattr(_lib, fn)(h)


def lib():
    """Load libfsa_b200.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = lib().fsa_last_error().decode()
    if rc == 2:
        raise ValueError(msg)
    if rc == 3:
        raise NumericalError(msg)
    raise CudaError(msg)


def _F(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _cg(tol, max_iter, error_on_max_iter=False):
    return CgOptions(float(tol), int(max_iter), 1 if error_on_max_iter else 0)


# ---- generators (host) -------------------------------------------------------------------
def uniform_locations(n, d, seed):
    out = _F(np.zeros((n, d)))
    _check(lib().fsa_uniform_locations(n, d, seed, out))
    return out


def select_random(coords, m, seed):
    c = _F(coords)
    out = _F(np.zeros((m, c.shape[1])))
    _check(lib().fsa_select_random(c, c.shape[0], c.shape[1], m, seed, out))
    return out


def select_kmeanspp(coords, m, seed, max_iter=20, rel_tol=1e-4, device=False, ctx=None):
    """select_kmeanspp (inducing.cpp:48-139). device=True runs the seeding, Lloyd and snapping
    kernels on ``ctx`` (default context) instead of the host restatement."""
    c = _F(coords)
    out = _F(np.zeros((m, c.shape[1])))
    if device or ctx is not None:
        ctx = ctx or default_context()
        _check(lib().fsa_select_kmeanspp_device(ctx.h, c, c.shape[0], c.shape[1], m, seed, max_iter, rel_tol, out))
    else:
        _check(lib().fsa_select_kmeanspp(c, c.shape[0], c.shape[1], m, seed, max_iter, rel_tol, out))
    return out


def gamma_for_avg_row_nnz(n, target):
    g = lib().fsa_gamma_for_avg_row_nnz(n, target)
    if g < 0:
        _check(2)
    return g


def simulate_rff(coords, nu, sigma1_2, rho, nugget, features=1024, seed=0):
    c = _F(coords)
    y = _F(np.zeros(c.shape[0]))
    _check(lib().fsa_simulate_rff(c, c.shape[0], c.shape[1], NU_CODE[nu], sigma1_2, rho, nugget, features, seed, y))
    return y


def blob_locations(n, d, blobs, sd, seed):
    out = _F(np.zeros((n, d)))
    _check(lib().fsa_blob_locations(n, d, blobs, sd, seed, out))
    return out


def probe_gaussian(seed, index, n1, n2):
    e1, e2 = _F(np.zeros(max(n1, 1))), _F(np.zeros(max(n2, 1)))
    _check(lib().fsa_probe_gaussian(seed, index, n1, e1, n2, e2))
    return e1[:n1], e2[:n2]


def launch_count() -> int:
    """Kernels launched by libfsa_b200.so so far in this process."""
    return int(lib().fsa_launch_count())


def tridiag_log_quadrature(diag, off):
    d = _F(diag)
    o = _F(off) if len(off) else _F(np.zeros(1))
    out = C.c_double()
    _check(lib().fsa_tridiag_log_quadrature(d, o, len(d), C.byref(out)))
    return out.value


# ---- device objects -------------------------------------------------------------------------
def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id; rank 0 creates it and broadcasts it to the other ranks."""
    buf = C.create_string_buffer(128)
    _check(lib().fsa_nccl_unique_id(buf))
    return buf.raw


class Context:
    """One CUDA device + stream (one host thread per context).

    ``Context.nccl(device, rank, world, uid)`` makes rank ``rank`` of a row-sharded
    multi-GPU job (one process per GPU); ``Context.group(device, world)`` makes ``world``
    sharded ranks on one device, each to be driven by its own host thread.
    """

    def __init__(self, device=0, _handle=None):
        if _handle is None:
            h = _vp()
            _check(lib().fsa_ctx_create(device, C.byref(h)))
        else:
            h = _handle
        self.h = h

    @classmethod
    def nccl(cls, device, rank, world, unique_id: bytes):
        h = _vp()
        _check(lib().fsa_ctx_create_nccl(device, rank, world, bytes(unique_id), C.byref(h)))
        return cls(_handle=h)

    @classmethod
    def group(cls, device, world):
        hs = (_vp * world)()
        _check(lib().fsa_ctx_group_create(device, world, hs))
        return [cls(_handle=_vp(hs[r])) for r in range(world)]

    def set_replicated(self, on=True):
        """Replicated mode: whole model per rank; predict_var_sim shards its probe batches."""
        _check(lib().fsa_ctx_set_replicated(self.h, 1 if on else 0))

    def rank_world(self):
        r, w = C.c_int(), C.c_int()
        _check(lib().fsa_ctx_rank(self.h, C.byref(r), C.byref(w)))
        return r.value, w.value

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _destroy("fsa_ctx_destroy", self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    def synchronize(self):
        _check(lib().fsa_ctx_synchronize(self.h))

    GEMM_MODES = {"auto": 0, "dmma": 1, "ozaki": 2}

    def set_gemm_mode(self, mode="auto"):
        """Dense U passes: 'auto' (INT8 tensor-core Ozaki path for <= 64 RHS columns), 'dmma', 'ozaki'."""
        _check(lib().fsa_ctx_set_gemm_mode(self.h, self.GEMM_MODES[mode]))

    def last_cg(self):
        """Per-column iteration counts and residual-norm histories of the last PCG solve."""
        k = C.c_int64()
        _check(lib().fsa_ctx_last_cg(self.h, C.byref(k), 0, 0, None, None))
        it = np.zeros(k.value, np.int32)
        _check(lib().fsa_ctx_last_cg(self.h, C.byref(k), k.value, 0, it.ctypes.data, None))
        cap = max(int(it.max()) if len(it) else 0, 1)
        rn = np.zeros((k.value, cap))
        _check(lib().fsa_ctx_last_cg(self.h, C.byref(k), k.value, cap, it.ctypes.data, rn.ctypes.data))
        return {"iterations": it, "rnorm": [rn[j, : it[j]].copy() for j in range(k.value)]}

    def stream(self) -> int:
        s = _vp()
        _check(lib().fsa_ctx_stream(self.h, C.byref(s)))
        return s.value or 0

    def set_profiling(self, on=True):
        _check(lib().fsa_ctx_set_profiling(self.h, 1 if on else 0))

    def reset_timers(self):
        _check(lib().fsa_ctx_reset_timers(self.h))

    def timers(self):
        buf = C.create_string_buffer(1 << 16)
        _check(lib().fsa_ctx_timer_names(self.h, buf, len(buf)))
        out = {}
        for name in buf.value.decode().split():
            ms, cnt, units = C.c_double(), _i64(), C.c_double()
            _check(lib().fsa_ctx_timer(self.h, name.encode(), C.byref(ms), C.byref(cnt), C.byref(units)))
            out[name] = {"ms": ms.value, "count": cnt.value, "units": units.value}
        return out


_default_ctx = None


def default_context():
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class Geometry:
    """Sorted points + taper pattern (parameter independent; locations.cpp:19-163)."""

    def __init__(self, coords, gamma, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.coords = _F(coords)
        self.n, self.d = self.coords.shape
        self.gamma = float(gamma)
        h = _vp()
        _check(lib().fsa_geometry_create(self.ctx.h, self.coords, self.n, self.d, self.gamma, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _destroy("fsa_geometry_destroy", self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    def nnz(self):
        n, nnz = _i64(), _i64()
        _check(lib().fsa_geometry_info(self.h, C.byref(n), C.byref(nnz)))
        return nnz.value

    def pattern(self):
        nnz = self.nnz()
        ptr = np.zeros(self.n + 1, np.int64)
        idx = np.zeros(max(nnz, 1), np.int32)
        val = _F(np.zeros(max(nnz, 1)))
        _check(lib().fsa_geometry_pattern(self.h, ptr, idx, val))
        return ptr, idx[:nnz], val[:nnz]

    def shard_info(self):
        """(r0, r1, n_halo): this rank's block of the internal order and its halo size."""
        a, b, c = _i64(), _i64(), _i64()
        _check(lib().fsa_geometry_shard_info(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def permutation(self):
        p = np.zeros(self.n, np.int32)
        _check(lib().fsa_geometry_permutation(self.h, p))
        return p

    def set_response(self, y, X=None):
        """Keep [y | X] resident in HBM; iterative_nll_grad(..., y=None) then uses it."""
        self._y = _F(y)
        p = 0 if X is None else np.asarray(X).reshape(self.n, -1).shape[1]
        self._X = None if p == 0 else _F(np.asarray(X).reshape(self.n, p))
        _check(lib().fsa_geometry_set_response(self.h, self._y, None if p == 0 else self._X.ctypes.data, p))

    def cache_probes(self, on=True):
        _check(lib().fsa_geometry_cache_probes(self.h, 1 if on else 0))


class FsaModel:
    """Device mirror of fsagp::FsaModel (fsa.h:40-104)."""

    def __init__(self):
        self.h = None

    @staticmethod
    def assemble(coords, inducing, nu=1.5, taper_family=1, gamma=0.1, sigma2=1.0, sigma1_2=1.0, rho=0.1,
                 jitter_rel=1e-10, ctx: Context | None = None, geometry: Geometry | None = None):
        self = FsaModel()
        self.inducing = _F(inducing)
        self.params = Params(NU_CODE[nu], FAMILY_CODE[taper_family], float(gamma), float(sigma2), float(sigma1_2),
                             float(rho), float(jitter_rel))
        h = _vp()
        if geometry is not None:
            self.ctx = geometry.ctx
            self.geometry = geometry
            _check(lib().fsa_model_assemble_geo(geometry.h, self.inducing, self.inducing.shape[0],
                                                C.byref(self.params), C.byref(h)))
            self.n = geometry.n
        else:
            self.ctx = ctx or default_context()
            c = _F(coords)
            self.n = c.shape[0]
            _check(lib().fsa_model_assemble(self.ctx.h, c, c.shape[0], c.shape[1], self.inducing,
                                            self.inducing.shape[0], C.byref(self.params), C.byref(h)))
        self.h = h
        self.m = self.inducing.shape[0]
        self.sigma2, self.sigma1_2, self.rho = sigma2, sigma1_2, rho
        return self

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _destroy("fsa_model_destroy", self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    def info(self):
        n, m, nnz, cl = _i64(), _i64(), _i64(), _i64()
        ld = C.c_double()
        _check(lib().fsa_model_info(self.h, C.byref(n), C.byref(m), C.byref(nnz), C.byref(cl), C.byref(ld)))
        return {"n": n.value, "m": m.value, "nnz": nnz.value, "n_clamped": cl.value, "logdet_sigma_m": ld.value}

    def sigma_s(self, which=0):
        nnz = self.info()["nnz"]
        ptr = np.zeros(self.n + 1, np.int64)
        idx = np.zeros(max(nnz, 1), np.int32)
        val = _F(np.zeros(max(nnz, 1)))
        _check(lib().fsa_model_sigma_s(self.h, which, ptr, idx, val))
        return ptr, idx[:nnz], val[:nnz]

    def diagonals(self):
        a, b = _F(np.zeros(self.n)), _F(np.zeros(self.n))
        _check(lib().fsa_model_diagonals(self.h, a, b))
        return a, b

    def lowrank_project(self, V):
        """U V with U = L^{-1} Sigma_mn (m x n), V n x k, through the context's GEMM path."""
        V = _F(V).reshape(self.n, -1, order="F")
        out = _F(np.zeros((self.m, V.shape[1])))
        _check(lib().fsa_model_lowrank_project(self.h, V, V.shape[1], out))
        return out

    def lowrank_expand(self, W):
        """U^T W for W m x k."""
        W = _F(W).reshape(self.m, -1, order="F")
        out = _F(np.zeros((self.n, W.shape[1])))
        _check(lib().fsa_model_lowrank_expand(self.h, W, W.shape[1], out))
        return out

    def debug_kernel_bench(self, which=0, k=51, reps=20, flags=0):
        """Average ms of one sweep-kernel launch group on synthetic blocks (diagnostics)."""
        ms = C.c_double()
        _check(lib().fsa_debug_kernel_bench(self.h, int(which), int(k), int(reps), int(flags), C.byref(ms)))
        return ms.value

    def matmat(self, V):
        V = _F(V).reshape(self.n, -1, order="F")
        out = _F(np.zeros_like(V))
        _check(lib().fsa_model_matmat(self.h, V, V.shape[1], out))
        return out

    def deriv_matmat(self, which, V):
        V = _F(V).reshape(self.n, -1, order="F")
        out = _F(np.zeros_like(V))
        _check(lib().fsa_model_deriv_matmat(self.h, which, V, V.shape[1], out))
        return out


class Preconditioner:
    def __init__(self, model: FsaModel, kind="fitc"):
        self.model = model
        self.kind = kind
        h = _vp()
        if kind == "jacobi":
            _check(lib().fsa_make_jacobi(model.h, C.byref(h)))
        else:
            _check(lib().fsa_make_preconditioner(model.h, PRECOND_CODE[kind], C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _destroy("fsa_precond_destroy", self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    def name(self):
        return self.kind

    def logdet(self):
        out = C.c_double()
        _check(lib().fsa_precond_logdet(self.h, C.byref(out)))
        return out.value

    def solve_mat(self, R):
        R = _F(R).reshape(self.model.n, -1, order="F")
        out = _F(np.zeros_like(R))
        _check(lib().fsa_precond_solve_mat(self.h, R, R.shape[1], out))
        return out

    def sample_probes(self, num_probes, seed):
        out = _F(np.zeros((self.model.n, num_probes)))
        _check(lib().fsa_precond_sample_probes(self.h, num_probes, seed, out))
        return out

    def deriv_trace(self, which):
        out = C.c_double()
        _check(lib().fsa_precond_deriv_trace(self.h, which, C.byref(out)))
        return out.value


def make_preconditioner(model: FsaModel, kind="fitc") -> Preconditioner:
    """make_preconditioner (estimation.cpp:160-176): 'none' | 'diagonal' | 'fitc'."""
    return Preconditioner(model, kind)


def pcg_solve_multi(model: FsaModel, P: Preconditioner, B, tol=1e-3, max_iter=1000, op="fsa",
                    error_on_max_iter=False):
    """pcg_solve_multi (krylov.cpp:18-106); op='sigma_s' solves with Sigma_s alone."""
    B = _F(B).reshape(model.n, -1, order="F")
    k = B.shape[1]
    X = _F(np.zeros_like(B))
    it = np.zeros(k, np.int32)
    cv = np.zeros(k, np.int32)
    td = _F(np.zeros((max_iter, k)))
    to = _F(np.zeros((max_iter, k)))
    sw = C.c_int()
    cg = _cg(tol, max_iter, error_on_max_iter)
    _check(lib().fsa_pcg_solve_multi(model.h, P.h, 0 if op == "fsa" else 1, B, k, C.byref(cg), X, it, cv, td, to,
                                     C.byref(sw)))
    tri = [(td[: it[j], j].copy(), to[: max(it[j] - 1, 0), j].copy()) for j in range(k)]
    return {"X": X, "iterations": it, "converged": cv.astype(bool), "tridiags": tri, "sweeps": sw.value}


def iterative_nll_grad(model: FsaModel, P: Preconditioner, y, X=None, num_probes=50, seed=0, tol=1e-3,
                       max_iter=1000, cv="optimal", want_grad=True):
    """iterative_nll_grad (estimation.cpp:178-227)."""
    y = None if y is None else _F(y)
    p = 0 if X is None else np.asarray(X).reshape(model.n, -1).shape[1]
    Xf = None if p == 0 else _F(np.asarray(X).reshape(model.n, p))
    if y is None:  # resident response (Geometry.set_response)
        p = model.geometry._X.shape[1] if getattr(model.geometry, "_X", None) is not None else 0
    beta = _F(np.zeros(max(p, 1)))
    res = NllResult()
    cg = _cg(tol, max_iter)
    beta = _F(np.zeros(max(p, 1)))
    _check(lib().fsa_iterative_nll_grad(model.h, P.h, None if y is None else y.ctypes.data,
                                        None if Xf is None else Xf.ctypes.data, 0 if y is None else p,
                                        num_probes, seed,
                                        C.byref(cg), CV_CODE[cv], 1 if want_grad else 0, C.byref(res),
                                        beta.ctypes.data))
    return {"nll": res.nll, "grad": np.array(res.grad[:]), "logdet": res.logdet, "cg_iterations": res.cg_iterations,
            "beta": beta[:p].copy(), "sweeps": res.sweeps, "rhs_iterations": res.rhs_iterations,
            "pcg_ms": res.pcg_ms, "total_ms": res.total_ms}


def fisher_ste(model: FsaModel, num_probes=50, seed=0, rademacher=False, P: Preconditioner = None, tol=1e-8,
               max_iter=1000):
    """fisher_ste (fsa.cpp:284-301; FisherOptions fsa.h:107-111). The reference's exact solves
    are batched PCG runs here (preconditioner P, FITC by default) to tolerance ``tol``."""
    if P is None:
        P = make_preconditioner(model, "fitc")
    F = _F(np.zeros((3, 3)))
    it = C.c_int()
    cg = _cg(tol, max_iter)
    _check(lib().fsa_fisher_ste(model.h, P.h, num_probes, seed, 1 if rademacher else 0, C.byref(cg), F,
                                C.byref(it)))
    return F


class PredictionSet:
    """make_prediction_set (prediction.cpp:7-27) on the device."""

    def __init__(self, model: FsaModel, pcoords):
        self.model = model
        self.pcoords = _F(pcoords)
        self.np = self.pcoords.shape[0]
        h = _vp()
        _check(lib().fsa_pred_setup(model.h, self.pcoords, self.np, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _destroy("fsa_pred_destroy", self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    def nnz(self):
        a, b = _i64(), _i64()
        _check(lib().fsa_pred_info(self.h, C.byref(a), C.byref(b)))
        return b.value

    def cross_apply_t(self, u):
        out = _F(np.zeros(self.np))
        _check(lib().fsa_cross_apply_t(self.h, _F(u), out))
        return out

    def predict_mean_iterative(self, resid, P: Preconditioner, tol=1e-3, max_iter=1000):
        out = _F(np.zeros(self.np))
        cg = _cg(tol, max_iter)
        _check(lib().fsa_predict_mean_iterative(self.h, _F(resid), P.h, C.byref(cg), out))
        return out

    def det_pieces(self, tol=1e-3, max_iter=1000, tol_s=1e-3, max_iter_s=1000):
        d1, d2, d3 = (_F(np.zeros(self.np)) for _ in range(3))
        it = C.c_int()
        cg, cgs = _cg(tol, max_iter), _cg(tol_s, max_iter_s)
        _check(lib().fsa_pred_det_pieces(self.h, C.byref(cg), C.byref(cgs), d1, d2, d3, C.byref(it)))
        return d1, d2, d3, it.value

    def predict_var_sim(self, num_probes=1000, seed=0, tol=1e-3, max_iter=1000, tol_s=1e-3, max_iter_s=1000,
                        control_variate=False, floor_rel=1e-6):
        var, se = _F(np.zeros(self.np)), _F(np.zeros(self.np))
        info = PredVarInfo()
        cg, cgs = _cg(tol, max_iter), _cg(tol_s, max_iter_s)
        _check(lib().fsa_predict_var_sim(self.h, num_probes, seed, C.byref(cg), C.byref(cgs),
                                         1 if control_variate else 0, floor_rel, var, se, C.byref(info)))
        return {"var": var, "se": se, "clamped": info.clamped, "cg_iterations": info.cg_iterations,
                "det_ms": info.det_ms, "sim_ms": info.sim_ms}


def make_prediction_set(model: FsaModel, pcoords) -> PredictionSet:
    return PredictionSet(model, pcoords)


def fit_fsa(coords, y, X=None, nu=1.5, taper_family=1, num_inducing=200, taper_range=0.0, target_row_nnz=40.0,
            precond="fitc", num_probes=50, cv="optimal", seed=0, cg_tol=1e-3, cg_max_iter=1000, max_evals=200,
            grad_tol_per_n=1e-3, ctx: Context | None = None, **lbfgs):
    """fit_fsa (estimation.cpp:229-303), iterative backend, with fit-loop residency on the device."""
    ctx = ctx or default_context()
    c = _F(coords)
    n, d = c.shape
    y = _F(y)
    p = 0 if X is None else np.asarray(X).reshape(n, -1).shape[1]
    Xf = None if p == 0 else _F(np.asarray(X).reshape(n, p))
    o = FitOptions()
    lib().fsa_fit_options_default(C.byref(o))
    o.nu_code, o.taper_family, o.num_inducing = NU_CODE[nu], FAMILY_CODE[taper_family], int(num_inducing)
    o.taper_range, o.target_row_nnz = float(taper_range), float(target_row_nnz)
    o.precond, o.num_probes, o.cv_mode, o.seed = PRECOND_CODE[precond], int(num_probes), CV_CODE[cv], int(seed)
    o.cg_tol, o.cg_max_iter, o.max_evals, o.grad_tol_per_n = float(cg_tol), int(cg_max_iter), int(max_evals), float(grad_tol_per_n)
    for k, v in lbfgs.items():
        setattr(o, k, v)
    res = FitResult()
    beta = _F(np.zeros(max(p, 1)))
    ind = _F(np.zeros((int(num_inducing), d)))
    cap = int(max_evals) + 8
    trace = _F(np.zeros(cap))
    _check(lib().fsa_fit(ctx.h, c, n, d, y, None if Xf is None else Xf.ctypes.data, p, C.byref(o), C.byref(res),
                         beta.ctypes.data, ind, trace, cap))
    return {"sigma2": res.sigma2, "sigma1_2": res.sigma1_2, "rho": res.rho, "nll": res.nll, "gamma": res.gamma,
            "beta": beta[:p].copy(), "evals": res.evals, "converged": bool(res.converged),
            "grad_log": np.array(res.grad_log[:]), "inducing": ind,
            "nll_trace": trace[:min(cap, res.n_trace)].copy()}
