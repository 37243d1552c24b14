"""Dense NumPy mirror of the reference's test oracles (tests/oracles.h:19-82).

Written from the scalar definitions, sharing no code with either the CPU oracle
or the product — the same independence rule the reference states
(oracles.h:3-4). Used to pin the oracle and, on the GPU, the product.
"""
import numpy as np


def matern_ref(d, nu, s1, rho):  # oracles.h:19-27
    d = np.asarray(d, dtype=np.float64)
    if nu == 0.5:
        return s1 * np.exp(-d / rho)
    if nu == 1.5:
        x = np.sqrt(3.0) * d / rho
        return s1 * (1.0 + x) * np.exp(-x)
    x = np.sqrt(5.0) * d / rho
    return s1 * (1.0 + x + x * x / 3.0) * np.exp(-x)


def wendland_ref(d, gamma, family):  # oracles.h:29-34
    r = np.asarray(d, dtype=np.float64) / gamma
    out = np.where(family == 1, (1.0 - r) ** 4 * (1.0 + 4.0 * r),
                   (1.0 - r) ** 6 * (1.0 + 6.0 * r + 35.0 * r * r / 3.0))
    return np.where(r >= 1.0, 0.0, out)


def pairwise(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    diff = a[:, None, :] - b[None, :, :]
    return np.sqrt((diff * diff).sum(-1))


def dense_cov(a, b, nu, s1, rho):  # oracles.h:36-45
    return matern_ref(pairwise(a, b), nu, s1, rho)


def dense_fsa_cov(locs, inducing, nu, family, gamma, sigma2, sigma1_2, rho, jitter_rel=1e-10):
    """oracles.h:49-70: low-rank part + tapered residual (diag clamped) + nugget."""
    sm = dense_cov(inducing, inducing, nu, sigma1_2, rho)
    sm[np.diag_indices_from(sm)] += jitter_rel * sigma1_2
    smn = dense_cov(inducing, locs, nu, sigma1_2, rho)
    low = smn.T @ np.linalg.solve(sm, smn)
    d = pairwise(locs, locs)
    full = matern_ref(d, nu, sigma1_2, rho)
    out = low + (full - low) * wendland_ref(d, gamma, family)
    n = len(locs)
    out[np.arange(n), np.arange(n)] = low.diagonal() + np.maximum(sigma1_2 - low.diagonal(), 0.0) + sigma2
    return out


def dense_cross(locs, plocs, inducing, nu, family, gamma, sigma1_2, rho):
    """n x n_p approximated cross covariance (test_prediction.cpp:32-47)."""
    sm = dense_cov(inducing, inducing, nu, sigma1_2, rho)
    sm[np.diag_indices_from(sm)] += 1e-10 * sigma1_2
    smn = dense_cov(inducing, locs, nu, sigma1_2, rho)
    smp = dense_cov(inducing, plocs, nu, sigma1_2, rho)
    cross = smn.T @ np.linalg.solve(sm, smp)
    d = pairwise(locs, plocs)
    mask = d < gamma
    cross = np.where(mask, cross + (matern_ref(d, nu, sigma1_2, rho) - cross) * wendland_ref(d, gamma, family), cross)
    return cross


def dense_logdet(cov):  # oracles.h:72-75
    return 2.0 * np.log(np.diag(np.linalg.cholesky(cov))).sum()


def dense_nll(cov, resid):  # oracles.h:77-82
    u = np.linalg.solve(cov, resid)
    return 0.5 * (dense_logdet(cov) + resid @ u + len(resid) * 1.8378770664093454836)


def dense_fitc(low_plus_diag_low, diag):
    return low_plus_diag_low + np.diag(diag)
