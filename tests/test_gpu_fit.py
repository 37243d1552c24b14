"""Maximum-likelihood fit: L-BFGS over the device nll/gradient with
fit-loop residency, checked against the oracle at the returned point."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

fsa = pytest.importorskip("paper_2405_14492_b200.fsa")


def test_fit_converges_to_a_stationary_point_of_the_oracle_objective():
    n = 3000
    locs = O.uniform_locations(n, 2, 5)
    y = fsa.simulate_rff(locs, 1.5, 1.0, 0.08, 0.1, 512, 6)
    X = np.column_stack([np.ones(n), locs[:, 0]])
    y = y + X @ np.array([0.5, -1.0])
    r = fsa.fit_fsa(locs, y, X, nu=1.5, num_inducing=60, target_row_nnz=40, num_probes=20, seed=3, cg_tol=1e-6,
                    max_evals=60)
    assert r["converged"]
    assert r["nll"] <= r["nll_trace"][0]
    assert 0.02 < r["sigma2"] < 0.5 and 0.3 < r["sigma1_2"] < 3.0 and 0.02 < r["rho"] < 0.3
    tol = 1e-3 * n
    assert np.abs(r["grad_log"]).max() <= tol
    # the oracle's objective at the returned point: same nll, stationary gradient
    kw = dict(nu=1.5, taper_family=1, gamma=r["gamma"], sigma2=r["sigma2"], sigma1_2=r["sigma1_2"], rho=r["rho"])
    om = O.Model(locs, r["inducing"], **kw)
    ref = O.iterative_nll_grad(om, O.Precond(om, "fitc"), y, X, num_probes=20, seed=3, tol=1e-6, cv="optimal")
    assert r["nll"] == pytest.approx(ref["nll"], rel=1e-6)
    g_log = ref["grad"] * np.array([r["sigma2"], r["sigma1_2"], r["rho"]])
    assert np.abs(g_log).max() <= 2 * tol
    np.testing.assert_allclose(r["beta"], ref["beta"], rtol=1e-6)


def test_fit_infeasible_start_is_an_error():
    n = 200
    locs = O.uniform_locations(n, 2, 7)
    y = np.zeros(n)  # zero residual variance: sigma2 = sigma1_2 = 0 at the start point
    with pytest.raises((fsa.NumericalError, ValueError)):
        fsa.fit_fsa(locs, y, num_inducing=20, max_evals=5)
