"""The fsagp-shaped facade (paper_2405_14492_b200/fsagp.py) mirrors the reference's pybind module
(proj/python/src/bindings.cpp:40-176; its tests: proj/python/tests/test_smoke.py)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2405_14492_b200 import fsagp


def grid(n_side):
    xs = np.linspace(0.0, 1.0, n_side)
    xx, yy = np.meshgrid(xs, xs)
    return np.column_stack([xx.ravel(), yy.ravel()])


def test_matern_value():  # test_smoke.py:14-17
    val = fsagp.matern(0.5, 1.5, 2.0, 0.5)
    s3 = np.sqrt(3.0)
    assert val == pytest.approx(2.0 * (1.0 + s3) * np.exp(-s3), rel=1e-12)
    for nu in (0.5, 1.5, 2.5):
        assert fsagp.matern(0.03, nu, 1.3, 0.1) == pytest.approx(O.matern(0.03, nu, 1.3, 0.1), rel=1e-14)


def test_host_helpers_match_oracle():
    c = grid(12)
    assert np.array_equal(fsagp.select_inducing(c, 10, seed=3, method="random"), O.select_random(c, 10, 3))
    assert np.array_equal(fsagp.select_inducing(c, 10, seed=3), O.select_kmeanspp(c, 10, 3))
    assert fsagp.taper_range_for_row_nnz(144, 10.0) == O.gamma_for_avg_row_nnz(144, 10.0)
    with pytest.raises(ValueError):
        fsagp.select_inducing(c, 10, method="grid")


@pytest.mark.gpu
def test_model_nll_iterative_and_predict_match_oracle():
    c = O.uniform_locations(3000, 2, 5)
    ind = fsagp.select_inducing(c, 60, seed=3)
    gamma = fsagp.taper_range_for_row_nnz(c.shape[0], 25.0)
    kw = dict(nu=1.5, gamma=gamma, sigma2=0.1, sigma1_2=1.0, rho=0.08)
    y = O.simulate_rff(c, 1.5, 1.0, 0.08, 0.1, 256, 7)
    model = fsagp.Model(c, ind, **kw)
    assert (model.n, model.m) == (3000, 60)
    nll, its = model.nll_iterative(y, probes=20, seed=5, cg_tol=1e-6)
    om = O.Model(c, ind, taper_family=1, **kw)
    want = O.iterative_nll_grad(om, O.Precond(om, "fitc"), y, num_probes=20, seed=5, tol=1e-6, want_grad=False)
    assert its == want["cg_iterations"]
    assert nll == pytest.approx(want["nll"], rel=1e-8)
    v = np.random.default_rng(1).standard_normal(3000)
    np.testing.assert_allclose(model.matvec(v), om.matmat(v.reshape(-1, 1))[:, 0], rtol=1e-10, atol=1e-10)
    pc = O.uniform_locations(400, 2, 9)
    mean, var = model.predict(pc, y, var_method="sim", probes=256, seed=2)
    opr = O.PredictionSet(om, pc)
    wm = opr.predict_mean_iterative(y, O.Precond(om, "fitc"), tol=1e-8)
    wv = opr.predict_var_sim(num_probes=256, seed=2)["var"]
    np.testing.assert_allclose(mean, wm, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(var, wv, rtol=1e-6)
    for bad in ("exact", "lanczos", "bogus"):
        with pytest.raises(ValueError):
            model.predict(pc, y, var_method=bad)
    with pytest.raises(ValueError):
        model.solve(v)
