"""Pin the oracle's FSA operator, preconditioners and Krylov layer against the
dense mirror, mirroring reference tests/test_fsa.cpp, test_preconditioners.cpp
and test_krylov.cpp (same sizes and tolerances)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import dense_mirror as DM


def small_model(n, m, gamma, s2, s12, rho, seed, family=1, nu=1.5):
    locs = O.uniform_locations(n, 2, seed)
    ind = O.select_kmeanspp(locs, m, seed + 1)
    model = O.Model(locs, ind, nu=nu, taper_family=family, gamma=gamma, sigma2=s2, sigma1_2=s12, rho=rho)
    dense = DM.dense_fsa_cov(locs, ind, nu, family, gamma, s2, s12, rho)
    return model, dense, locs, ind


def test_operator_matches_dense():  # test_fsa.cpp:36-60
    model, dense, _, _ = small_model(150, 12, 0.2, 0.4, 1.3, 0.12, 3)
    V = np.random.default_rng(9).standard_normal((150, 3))
    assert np.abs(model.matmat(V) - dense @ V).max() < 1e-10
    for fam, nu in ((2, 0.5), (1, 2.5)):
        m2, d2, _, _ = small_model(120, 10, 0.25, 0.3, 1.0, 0.1, 5, family=fam, nu=nu)
        assert np.abs(m2.matmat(V[:120]) - d2 @ V[:120]).max() < 1e-10


def test_operator_positive_definite():  # test_fsa.cpp:62-70
    _, dense, _, _ = small_model(120, 10, 0.25, 0.05, 1.0, 0.2, 13)
    assert np.linalg.eigvalsh(dense).min() >= 0.05 * (1 - 1e-10)


def test_derivative_operator_matches_fd():  # test_fsa.cpp:111-136
    theta = np.array([0.4, 1.2, 0.15])
    locs = O.uniform_locations(90, 2, 43)
    ind = O.select_kmeanspp(locs, 9, 44)
    v = np.random.default_rng(8).standard_normal(90)
    mk = lambda t: O.Model(locs, ind, nu=1.5, taper_family=1, gamma=0.22, sigma2=t[0], sigma1_2=t[1], rho=t[2])
    base = mk(theta)
    for k in range(3):
        h = 1e-5 * theta[k]
        tp, tm = theta.copy(), theta.copy()
        tp[k] += h
        tm[k] -= h
        fd = (mk(tp).matmat(v)[:, 0] - mk(tm).matmat(v)[:, 0]) / (2 * h)
        got = base.deriv_matmat(k, v)[:, 0]
        assert np.linalg.norm(got - fd) / max(np.linalg.norm(fd), 1e-8) < 1e-5


def fitc_dense(model):
    smn = model.dense(1)
    sm = model.dense(0)
    low = smn.T @ np.linalg.solve(sm, smn)
    ptr, idx, val = model.csr(1)
    diag = np.array([val[ptr[i]:ptr[i + 1]][idx[ptr[i]:ptr[i + 1]] == i][0] for i in range(model.n)])
    return low + np.diag(diag)


def test_fitc_matches_dense():  # test_preconditioners.cpp:71-100
    locs = O.uniform_locations(120, 2, 7)
    ind = O.select_kmeanspp(locs, 10, 8)
    model = O.Model(locs, ind, gamma=0.2, sigma2=0.5, sigma1_2=1.0, rho=0.1)
    P = O.Precond(model, "fitc")
    dense = fitc_dense(model)
    rng = np.random.default_rng(9)
    r = rng.standard_normal(120)
    assert np.linalg.norm(P.solve_cols(r)[:, 0] - np.linalg.solve(dense, r)) / np.linalg.norm(r) < 1e-9
    assert P.logdet() == pytest.approx(DM.dense_logdet(dense), rel=1e-9)
    R = rng.standard_normal((120, 3))
    assert np.abs(P.solve_mat(R) - np.linalg.solve(dense, R)).max() < 1e-8
    inv = np.linalg.inv(dense)
    for k in range(3):
        dP = np.column_stack([P.deriv_apply(k, e) for e in np.eye(120)])
        assert P.deriv_trace(k) == pytest.approx(np.trace(inv @ dP), rel=1e-8)


def test_fitc_derivative_matches_fd():  # test_preconditioners.cpp:102-143
    theta = np.array([0.4, 1.1, 0.13])
    locs = O.uniform_locations(90, 2, 11)
    ind = O.select_kmeanspp(locs, 8, 12)
    mk = lambda t: O.Model(locs, ind, gamma=0.22, sigma2=t[0], sigma1_2=t[1], rho=t[2])
    P = O.Precond(mk(theta), "fitc")
    v = np.random.default_rng(13).standard_normal(90)
    for k in range(3):
        h = 1e-5 * theta[k]
        tp, tm = theta.copy(), theta.copy()
        tp[k] += h
        tm[k] -= h
        Pp = O.Precond(mk(tp), "fitc", plain=True)
        Pm = O.Precond(mk(tm), "fitc", plain=True)
        Dp = np.linalg.inv(Pp.solve_mat(np.eye(90)))
        Dm = np.linalg.inv(Pm.solve_mat(np.eye(90)))
        fd = (Dp @ v - Dm @ v) / (2 * h)
        got = P.deriv_apply(k, v)
        assert np.linalg.norm(got - fd) / max(np.linalg.norm(fd), 1e-8) < 1e-4


def test_vanishing_taper_makes_fitc_exact():  # test_preconditioners.cpp:145-158
    locs = O.uniform_locations(150, 2, 17)
    ind = O.select_kmeanspp(locs, 15, 18)
    model = O.Model(locs, ind, gamma=1e-6, sigma2=0.5, sigma1_2=1.0, rho=0.1)
    assert model.info()["nnz"] == 150
    P = O.Precond(model, "fitc", plain=True)
    b = np.random.default_rng(19).standard_normal(150)
    r = O.pcg_solve_multi(model, P, b, tol=1e-8, batched=False)
    assert r["converged"][0] and r["iterations"][0] <= 2


def test_preconditioned_solves_agree():  # test_preconditioners.cpp:184-205
    model, dense, _, _ = small_model(200, 15, 0.15, 0.5, 1.0, 0.1, 37)
    b = np.random.default_rng(41).standard_normal(200)
    want = np.linalg.solve(dense, b)
    for kind in ("none", "diagonal", "fitc"):
        P = O.Precond(model, kind)
        r = O.pcg_solve_multi(model, P, b, tol=1e-9, max_iter=3000, batched=False)
        assert r["converged"][0]
        assert np.linalg.norm(r["X"][:, 0] - want) / np.linalg.norm(want) < 1e-7


def test_identity_probes_are_signs():  # test_preconditioners.cpp:27-36
    model, _, _, _ = small_model(20, 4, 0.3, 0.5, 1.0, 0.1, 1)
    Z = O.Precond(model, "none").sample_probes(6, 3)
    assert np.all(np.abs(Z) == 1.0)


def test_cg_against_factorised():  # test_krylov.cpp:36-52
    model, dense, _, _ = small_model(200, 15, 0.15, 0.5, 1.0, 0.1, 3)
    b = np.random.default_rng(7).standard_normal(200)
    r = O.pcg_solve_multi(model, O.Precond(model, "none"), b, tol=1e-10, max_iter=2000, batched=False)
    x = r["X"][:, 0]
    assert r["converged"][0]
    assert np.linalg.norm(dense @ x - b) < 1e-9
    want = np.linalg.solve(dense, b)
    assert np.linalg.norm(x - want) / np.linalg.norm(want) < 1e-8
    d, o = r["tridiags"][0]
    assert len(d) == r["iterations"][0] and len(o) == r["iterations"][0] - 1


def test_cg_zero_rhs():  # test_krylov.cpp:54-61
    model, _, _, _ = small_model(50, 6, 0.2, 0.5, 1.0, 0.1, 5)
    r = O.pcg_solve_multi(model, O.Precond(model, "none"), np.zeros(50), batched=False)
    assert r["converged"][0] and r["iterations"][0] == 0 and np.all(r["X"] == 0.0)


def test_strict_multi_equals_single_bitwise():  # test_krylov.cpp:73-92
    model, _, _, _ = small_model(150, 12, 0.18, 0.5, 1.0, 0.1, 11)
    P = O.Precond(model, "fitc", plain=True)
    B = np.random.default_rng(13).standard_normal((150, 4))
    multi = O.pcg_solve_multi(model, P, B, tol=1e-6, batched=False)
    assert multi["converged"].all()
    for j in range(4):
        single = O.pcg_solve_multi(model, P, B[:, j], tol=1e-6, batched=False)
        assert np.array_equal(multi["X"][:, j], single["X"][:, 0])
        assert multi["iterations"][j] == single["iterations"][0]
        assert np.array_equal(multi["tridiags"][j][0], single["tridiags"][0][0])
        assert np.array_equal(multi["tridiags"][j][1], single["tridiags"][0][1])


def test_batched_matches_strict():  # test_krylov.cpp:94-111
    model, _, _, _ = small_model(150, 12, 0.18, 0.5, 1.0, 0.1, 17)
    P = O.Precond(model, "fitc", plain=True)
    B = np.random.default_rng(19).standard_normal((150, 5))
    s = O.pcg_solve_multi(model, P, B, tol=1e-8, batched=False)
    b = O.pcg_solve_multi(model, P, B, tol=1e-8, batched=True)
    assert b["converged"].all()
    assert np.abs(s["X"] - b["X"]).max() < 1e-7
    assert np.array_equal(s["iterations"], b["iterations"])


def test_slq_brackets_exact_logdet():  # test_krylov.cpp:141-168
    model, dense, _, _ = small_model(250, 15, 0.15, 0.5, 1.0, 0.1, 23)
    exact = DM.dense_logdet(dense)
    P = O.Precond(model, "fitc", plain=True)
    Z = P.sample_probes(150, 29)
    r = O.pcg_solve_multi(model, P, Z, tol=1e-8)
    assert r["converged"].all()
    q = np.array([O.tridiag_log_quadrature(d, o) for d, o in r["tridiags"]])
    est = 250 / 150 * q.sum() + P.logdet()
    se = 250 * np.sqrt(q.var(ddof=1) / 150)
    assert abs(est - exact) < 4 * se + 1e-6
    assert abs(est - exact) / abs(exact) < 0.05


def test_probes_keyed_per_column():  # test_krylov.cpp:170-176
    model, _, _, _ = small_model(60, 6, 0.2, 0.5, 1.0, 0.1, 31)
    P = O.Precond(model, "fitc", plain=True)
    assert np.array_equal(P.sample_probes(5, 77)[:, :3], P.sample_probes(3, 77))


def test_ste_unbiased_and_cv_shrinks():  # test_krylov.cpp:178-205
    model, dense, _, _ = small_model(200, 12, 0.15, 0.5, 1.0, 0.1, 37)
    P = O.Precond(model, "fitc")
    inv = np.linalg.inv(dense)
    Z = P.sample_probes(400, 41)
    sol = O.pcg_solve_multi(model, P, Z, tol=1e-8)
    assert sol["converged"].all()
    for k in range(3):
        dA = model.deriv_matmat(k, np.eye(200))
        exact = np.trace(inv @ dA)
        plain = O.ste_grad_trace(model, P, Z, sol["X"], k, "none")
        cv = O.ste_grad_trace(model, P, Z, sol["X"], k, "optimal")
        assert abs(plain["value"] - exact) < 4 * np.sqrt(plain["variance_of_mean"]) + 1e-8
        assert abs(cv["value"] - exact) < 4 * np.sqrt(cv["variance_of_mean"]) + 1e-8
        assert cv["variance_of_mean"] <= plain["variance_of_mean"] + 1e-12


def test_fisher_ste_approximates_dense():  # test_fsa.cpp:182-215
    model, dense, _, _ = small_model(100, 10, 0.2, 0.5, 1.0, 0.12, 73)
    n = 100
    inv = np.linalg.inv(dense)
    dS = [model.deriv_matmat(k, np.eye(n)) for k in range(3)]
    want = np.array([[0.5 * np.trace(inv @ dS[k] @ inv @ dS[l]) for l in range(3)] for k in range(3)])
    got = O.fisher_ste(model, num_probes=600, seed=5)
    assert np.abs(got - got.T).max() < 1e-10
    assert (np.abs(got - want) / np.maximum(np.abs(want), 1.0)).max() < 0.2
    # Rademacher probes estimate the same matrix
    got_r = O.fisher_ste(model, num_probes=600, seed=5, rademacher=True)
    assert (np.abs(got_r - want) / np.maximum(np.abs(want), 1.0)).max() < 0.2
