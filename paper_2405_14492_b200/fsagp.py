"""Drop-in mirror of the reference's Python module ``fsagp`` (proj/python/src/bindings.cpp:40-141)
for the path this build accelerates: the iterative log-likelihood and the simulation-based
predictive distribution, on the B200 library through its C ABI.

Same names, argument names, defaults and return shapes as the pybind module:

  Model(coords, inducing, nu=1.5, taper_family="wendland1", gamma=0.1, sigma2=1.0, sigma1_2=1.0,
        rho=0.1)                                              (bindings.cpp:78-81)
    .n, .m, .matvec(v)                                         (:82-84)
    .nll_iterative(y, probes=50, seed=0, precond="fitc", cg_tol=1e-3, cg_max_iter=1000)
        -> (nll, cg_iterations)                                (:101-117)
    .predict(pred_coords, resid, var_method="sim", probes=500, rank=50, seed=0) -> (mean, var)
                                                               (:118-141)
  select_inducing(coords, m, seed=0, method="kmeanspp"), taper_range_for_row_nnz(n, target_row_nnz),
  matern(d, nu, sigma1_2, rho), fit(coords, y, X, backend="iterative", ...) (:43-72, :143-176)

Outside the hot path (and outside this build): the exact backend (Model.solve / logdet / nll /
nll_grad, predict var_method="exact" / "lanczos", fit backend="cholesky"), Vecchia and scores.
Those raise ValueError naming the missing backend, as the reference raises invalid_argument for
an unknown method. Two documented differences: predict's mean is the FITC-PCG solve
(predict_mean_iterative, prediction.cpp:37-43, at tol 1e-8) where the pybind binding calls the
exact solve, and the default var_method is "sim" (the reference defaults to "exact").
"""
from __future__ import annotations

import numpy as np

from . import fsa

NumericalError = fsa.NumericalError

_FAMILIES = {"wendland1": 1, "wendland2": 2}
_OUT_OF_SCOPE = "needs the reference's exact (Cholesky) backend, which is outside this build's scope"


def _family(taper_family):
    if isinstance(taper_family, str):
        if taper_family not in _FAMILIES:
            raise ValueError("taper family must be wendland1 or wendland2")
        return _FAMILIES[taper_family]
    return int(taper_family)


def matern(d, nu, sigma1_2, rho):
    """Matern covariance, parameterised with sqrt(2 nu) d / rho (kernels.cpp:7-22)."""
    d, nu = float(d), float(nu)
    if nu == 0.5:
        return sigma1_2 * np.exp(-d / rho)
    if nu == 1.5:
        x = np.sqrt(3.0) * d / rho
        return sigma1_2 * (1.0 + x) * np.exp(-x)
    if nu == 2.5:
        x = np.sqrt(5.0) * d / rho
        return sigma1_2 * (1.0 + x + x * x / 3.0) * np.exp(-x)
    raise ValueError("nu must be 0.5, 1.5 or 2.5")


def select_inducing(coords, m, seed=0, method="kmeanspp"):
    if method == "kmeanspp":
        return fsa.select_kmeanspp(np.asarray(coords, float), int(m), int(seed))
    if method == "random":
        return fsa.select_random(np.asarray(coords, float), int(m), int(seed))
    raise ValueError("method must be kmeanspp or random")


def taper_range_for_row_nnz(n, target_row_nnz):
    return fsa.gamma_for_avg_row_nnz(int(n), float(target_row_nnz))


class Model:
    """FsaModel (fsa.h:40-104) assembled on the device."""

    def __init__(self, coords, inducing, nu=1.5, taper_family="wendland1", gamma=0.1, sigma2=1.0, sigma1_2=1.0,
                 rho=0.1):
        self._kw = dict(nu=float(nu), taper_family=_family(taper_family), gamma=float(gamma), sigma2=float(sigma2),
                        sigma1_2=float(sigma1_2), rho=float(rho))
        self._coords = np.asarray(coords, float)
        self._md = fsa.FsaModel.assemble(self._coords, np.asarray(inducing, float), **self._kw)

    @property
    def n(self):
        return self._md.n

    @property
    def m(self):
        return self._md.m

    def matvec(self, v):
        return self._md.matmat(np.asarray(v, float).reshape(self.n, 1))[:, 0]

    def nll_iterative(self, y, probes=50, seed=0, precond="fitc", cg_tol=1e-3, cg_max_iter=1000):
        if precond not in ("none", "diagonal", "fitc"):
            raise ValueError("preconditioner must be none, diagonal or fitc")
        P = fsa.make_preconditioner(self._md, precond)
        r = fsa.iterative_nll_grad(self._md, P, np.asarray(y, float), num_probes=int(probes), seed=int(seed),
                                   tol=float(cg_tol), max_iter=int(cg_max_iter), want_grad=False)
        return r["nll"], r["cg_iterations"]

    def nll_grad_iterative(self, y, probes=50, seed=0, precond="fitc", cg_tol=1e-3, cg_max_iter=1000,
                           cv="optimal"):
        """iterative_nll_grad with the gradient (estimation.cpp:178-227): (nll, grad[3], cg_iterations)."""
        P = fsa.make_preconditioner(self._md, precond)
        r = fsa.iterative_nll_grad(self._md, P, np.asarray(y, float), num_probes=int(probes), seed=int(seed),
                                   tol=float(cg_tol), max_iter=int(cg_max_iter), cv=cv)
        return r["nll"], r["grad"], r["cg_iterations"]

    def predict(self, pred_coords, resid, var_method="sim", probes=500, rank=50, seed=0):
        if var_method not in ("sim", "none"):
            if var_method in ("exact", "lanczos"):
                raise ValueError(f"var_method {var_method!r} {_OUT_OF_SCOPE}")
            raise ValueError("var_method must be exact, sim, lanczos, or none")
        pr = fsa.make_prediction_set(self._md, np.asarray(pred_coords, float))
        P = fsa.make_preconditioner(self._md, "fitc")
        mean = pr.predict_mean_iterative(np.asarray(resid, float), P, tol=1e-8)
        var = np.zeros(0)
        if var_method == "sim":
            var = pr.predict_var_sim(num_probes=int(probes), seed=int(seed))["var"]
        return mean, var

    def solve(self, b):
        raise ValueError(f"Model.solve {_OUT_OF_SCOPE}")

    def logdet(self):
        raise ValueError(f"Model.logdet {_OUT_OF_SCOPE}")

    def nll(self, y):
        raise ValueError(f"Model.nll {_OUT_OF_SCOPE}; use nll_iterative")

    def nll_grad(self, y):
        raise ValueError(f"Model.nll_grad {_OUT_OF_SCOPE}; use nll_grad_iterative")


def fit(coords, y, X, backend="iterative", m=200, target_row_nnz=40.0, gamma=0.0, nu=1.5, precond="fitc", probes=50,
        seed=0, max_evals=200):
    """fit_fsa (estimation.cpp:229-303), iterative backend; the same result keys as bindings.cpp:158-170."""
    if backend != "iterative":
        raise ValueError(f"backend {backend!r} {_OUT_OF_SCOPE}")
    X = np.asarray(X, float)
    r = fsa.fit_fsa(np.asarray(coords, float), np.asarray(y, float), X if X.size else None, nu=nu,
                    num_inducing=m, taper_range=gamma, target_row_nnz=target_row_nnz, precond=precond,
                    num_probes=probes, seed=seed, max_evals=max_evals)
    return {k: r[k] for k in ("sigma2", "sigma1_2", "rho", "beta", "nll", "evals", "converged", "gamma", "inducing")
            if k in r}
