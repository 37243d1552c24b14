"""Pin the oracle's iterative_nll_grad and predict_var_sim, mirroring reference
tests/test_estimation.cpp:132-194 and tests/test_prediction.cpp:66-143,174-184."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import dense_mirror as DM


def exact_nll_grad(model, dense, y, X):
    Si = np.linalg.inv(dense)
    SX = Si @ X
    beta = np.linalg.solve(X.T @ SX, SX.T @ y)
    r = y - X @ beta
    u = Si @ r
    nll = DM.dense_nll(dense, r)
    g = []
    for k in range(3):
        dS = model.deriv_matmat(k, np.eye(model.n))
        g.append(0.5 * (np.trace(Si @ dS) - u @ dS @ u))
    return nll, np.array(g), beta


def test_iterative_nll_tracks_exact():  # test_estimation.cpp:132-174
    n = 220
    locs = O.uniform_locations(n, 2, 107)
    ind = O.select_kmeanspp(locs, 25, 108)
    model = O.Model(locs, ind, gamma=0.25, sigma2=0.5, sigma1_2=1.0, rho=0.1)
    dense = DM.dense_fsa_cov(locs, ind, 1.5, 1, 0.25, 0.5, 1.0, 0.1)
    rng = np.random.default_rng(7)
    X = np.column_stack([np.ones(n), rng.standard_normal(n)])
    gen = DM.dense_fsa_cov(locs, ind, 1.5, 1, 0.25, 0.9, 1.8, 0.15)
    y = np.linalg.cholesky(gen) @ rng.standard_normal(n) + X @ np.array([0.5, -1.0])
    P = O.Precond(model, "fitc")
    it = O.iterative_nll_grad(model, P, y, X, num_probes=400, seed=11, tol=1e-10, max_iter=2000)
    nll, g, beta = exact_nll_grad(model, dense, y, X)
    assert np.linalg.norm(it["beta"] - beta) < 1e-7
    assert abs(it["nll"] - nll) / abs(nll) < 0.02
    for k in range(3):
        assert abs(it["grad"][k] - g[k]) / max(abs(g[k]), 5.0) < 0.25
    assert it["cg_iterations"] > 0


def test_iterative_nll_deterministic():  # test_estimation.cpp:176-194
    n = 120
    locs = O.uniform_locations(n, 2, 109)
    ind = O.select_kmeanspp(locs, 15, 110)
    model = O.Model(locs, ind, gamma=0.3, sigma2=0.5, sigma1_2=1.0, rho=0.1)
    y = np.random.default_rng(13).standard_normal(n)
    P = O.Precond(model, "fitc")
    a = O.iterative_nll_grad(model, P, y, num_probes=30, seed=17)
    b = O.iterative_nll_grad(model, P, y, num_probes=30, seed=17)
    assert a["nll"] == b["nll"] and np.array_equal(a["grad"], b["grad"]) and a["logdet"] == b["logdet"]


def pred_setup(n, np_, m, gamma, seed, s2=0.3, s12=1.0, rho=0.1):
    locs = O.uniform_locations(n, 2, seed)
    plocs = O.uniform_locations(np_, 2, seed + 100)
    ind = O.select_kmeanspp(locs, m, seed + 1)
    model = O.Model(locs, ind, gamma=gamma, sigma2=s2, sigma1_2=s12, rho=rho)
    pred = O.PredictionSet(model, plocs)
    dense = DM.dense_fsa_cov(locs, ind, 1.5, 1, gamma, s2, s12, rho)
    cross = DM.dense_cross(locs, plocs, ind, 1.5, 1, gamma, s12, rho)
    return model, pred, dense, cross


def test_prediction_set_matches_dense_cross():  # test_prediction.cpp:66-73
    model, pred, dense, cross = pred_setup(150, 40, 12, 0.2, 3)
    u = np.random.default_rng(5).standard_normal(150)
    assert np.abs(pred.cross_apply_t(u) - cross.T @ u).max() < 1e-10


def test_iterative_mean_matches_exact():  # test_prediction.cpp:82-90
    model, pred, dense, cross = pred_setup(150, 40, 12, 0.2, 11)
    resid = np.random.default_rng(18).standard_normal(150)
    P = O.Precond(model, "fitc", plain=True)
    it = pred.predict_mean_iterative(resid, P, tol=1e-9)
    ex = cross.T @ np.linalg.solve(dense, resid)
    assert np.abs(it - ex).max() < 1e-7


def exact_var(dense, cross, s2, s12):
    G = np.linalg.solve(dense, cross)
    return s12 + s2 - (cross * G).sum(0)


def test_deterministic_pieces_exact_when_ell_exact():
    # d1 + 2 d2 - d3 + d_exact reproduces the dense predictive variance
    model, pred, dense, cross = pred_setup(120, 30, 10, 0.2, 7)
    d1, d2, d3, _ = pred.det_pieces(tol=1e-11, tol_s=1e-11, max_iter=3000, max_iter_s=3000)
    ptr, idx, val = model.csr(1)
    Ss = np.zeros((120, 120))
    for i in range(120):
        Ss[i, idx[ptr[i]:ptr[i + 1]]] = val[ptr[i]:ptr[i + 1]]
    pp, pi, pv = pred.csr()
    Snp = np.zeros((120, 30))
    for i in range(120):
        Snp[i, pi[pp[i]:pp[i + 1]]] = pv[pp[i]:pp[i + 1]]
    d_ell = (Snp * np.linalg.solve(Ss, Snp)).sum(0)
    var = 1.0 + 0.3 - d1 - 2 * d2 + d3 - d_ell
    np.testing.assert_allclose(var, exact_var(dense, cross, 0.3, 1.0), atol=1e-7)


def test_sim_variances_converge():  # test_prediction.cpp:105-125
    model, pred, dense, cross = pred_setup(200, 50, 12, 0.18, 17)
    ex = exact_var(dense, cross, 0.3, 1.0)
    sim = pred.predict_var_sim(num_probes=3000, seed=19, tol=1e-8, tol_s=1e-8)
    inside = int((np.abs(sim["var"] - ex) <= 4 * sim["se"] + 1e-8).sum())
    assert inside >= 47
    assert np.sqrt(((sim["var"] - ex) ** 2).mean()) < 0.05


def test_sim_variances_cv():  # test_prediction.cpp:127-143
    model, pred, dense, cross = pred_setup(150, 30, 10, 0.2, 23)
    ex = exact_var(dense, cross, 0.3, 1.0)
    sim = pred.predict_var_sim(num_probes=2000, seed=29, tol=1e-8, tol_s=1e-8, control_variate=True)
    assert int((np.abs(sim["var"] - ex) <= 4 * sim["se"] + 1e-8).sum()) >= 28


def test_variance_floor():  # test_prediction.cpp:174-184
    model, pred, _, _ = pred_setup(80, 20, 8, 0.25, 41)
    sim = pred.predict_var_sim(num_probes=5, seed=43, floor_rel=1e6)
    assert sim["clamped"] == 20
    assert sim["var"].min() >= 1e6 * 0.3 - 1e-9
