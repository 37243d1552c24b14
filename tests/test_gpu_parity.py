"""GPU parity: the sm_100a library (through its C ABI) against the CPU oracle.

Mirrors the reference's hot-path tests (tests/test_fsa.cpp, test_krylov.cpp,
test_preconditioners.cpp, test_estimation.cpp, test_prediction.cpp) with the
north-star tolerances: solves to relative 1e-8, scalars to relative 1e-6.
The GPU evaluates the covariance in U-form (U = L^{-1} Sigma_mn) while the
oracle follows the reference's Sigma_mn^T (A V) sequence, so agreement is to
rounding, not bitwise.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests import dense_mirror as DM

pytestmark = pytest.mark.gpu

fsa = pytest.importorskip("paper_2405_14492_b200.fsa")


def setup(n=1500, m=60, gamma=0.08, s2=0.3, s12=1.0, rho=0.1, seed=3, nu=1.5, family=1, kmeans=True, d=2):
    locs = O.uniform_locations(n, d, seed)
    ind = O.select_kmeanspp(locs, m, seed + 1) if kmeans else O.select_random(locs, m, seed + 1)
    kw = dict(nu=nu, taper_family=family, gamma=gamma, sigma2=s2, sigma1_2=s12, rho=rho)
    return locs, ind, kw, fsa.FsaModel.assemble(locs, ind, **kw), O.Model(locs, ind, **kw)


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def test_native_library_is_loaded():
    import os

    assert os.path.exists(fsa.LIB_PATH)
    assert fsa.lib().fsa_version() == 1


@pytest.mark.parametrize("d", [1, 2, 3])
def test_taper_pattern_exact(d):
    n = 700
    locs = O.uniform_locations(n, d, 21)
    gamma = {1: 0.01, 2: 0.06, 3: 0.15}[d]
    g = fsa.Geometry(locs, gamma)
    ptr, idx, val = g.pattern()
    optr, oidx, oval = O.taper_pattern(locs, gamma)
    assert np.array_equal(ptr, optr)
    assert np.array_equal(idx, oidx)
    np.testing.assert_array_equal(val, oval)
    perm = g.permutation()
    assert sorted(perm.tolist()) == list(range(n))


def test_assembly_matches_oracle():
    locs, ind, kw, md, om = setup()
    info, oinfo = md.info(), om.info()
    assert info["nnz"] == oinfo["nnz"] and info["n_clamped"] == oinfo["n_clamped"]
    assert info["logdet_sigma_m"] == pytest.approx(oinfo["logdet_sigma_m"], rel=1e-10)
    ptr, idx, val = md.sigma_s(0)
    optr, oidx, oval = om.csr(1)
    assert np.array_equal(ptr, optr) and np.array_equal(idx, oidx)
    assert rel(val, oval) < 1e-10
    sdiag, lowrank = md.diagonals()
    np.testing.assert_allclose(lowrank, om.dense(6), rtol=1e-11, atol=1e-13)


@pytest.mark.parametrize("nu,family,kmeans", [(0.5, 1, False), (1.5, 1, True), (2.5, 2, True)])
def test_matmat_matches_oracle_and_dense(nu, family, kmeans):
    locs, ind, kw, md, om = setup(n=900, m=40, nu=nu, family=family, kmeans=kmeans, seed=5)
    V = np.random.default_rng(9).standard_normal((900, 5))
    got = md.matmat(V)
    assert rel(got, om.matmat(V)) < 1e-12
    dense = DM.dense_fsa_cov(locs, ind, nu, family, kw["gamma"], kw["sigma2"], kw["sigma1_2"], kw["rho"])
    assert np.abs(got - dense @ V).max() < 1e-10


def test_deriv_matmat_matches_oracle():
    locs, ind, kw, md, om = setup(n=800, m=48, seed=7)
    V = np.random.default_rng(1).standard_normal((800, 3))
    for k in range(3):
        assert rel(md.deriv_matmat(k, V), om.deriv_matmat(k, V)) < 1e-9, k
    ptr, idx, val = md.sigma_s(1)
    optr, oidx, oval = om.csr(2)
    assert np.array_equal(idx, oidx) and rel(val, oval) < 1e-9


def test_fitc_matches_oracle():
    locs, ind, kw, md, om = setup(n=1200, m=50, seed=11)
    P, OP = fsa.make_preconditioner(md, "fitc"), O.Precond(om, "fitc")
    assert P.logdet() == pytest.approx(OP.logdet(), rel=1e-10)
    R = np.random.default_rng(2).standard_normal((1200, 4))
    assert rel(P.solve_mat(R), OP.solve_mat(R)) < 1e-10
    Z, OZ = P.sample_probes(6, 77), OP.sample_probes(6, 77)
    assert rel(Z, OZ) < 1e-12
    for k in range(3):
        assert P.deriv_trace(k) == pytest.approx(OP.deriv_trace(k), rel=1e-9), k


@pytest.mark.parametrize("n,m,L,seed", [(3001, 77, 20, 5), (1200, 50, 1, 0), (800, 33, 33, 12345)])
def test_device_probe_streams_match_oracle(n, m, L, seed):
    """k_probe_gaussian draws the reference's per-probe MT19937-64 / polar normal streams on the
    device (odd m and n exercise the discarded saved value between e1 and e2): the probes
    z = U^T e1 + sqrt(D) e2 agree with the oracle's host draws to fp64 rounding."""
    locs, ind, kw, md, om = setup(n=n, m=m, seed=seed % 7 + 1)
    Z = fsa.make_preconditioner(md, "fitc").sample_probes(L, seed)
    OZ = O.Precond(om, "fitc").sample_probes(L, seed)
    assert rel(Z, OZ) < 1e-13


def test_pcg_matches_oracle():
    locs, ind, kw, md, om = setup(n=2000, m=64, seed=13, s2=0.1)
    P, OP = fsa.make_preconditioner(md, "fitc"), O.Precond(om, "fitc")
    B = P.sample_probes(8, 3)
    got = fsa.pcg_solve_multi(md, P, B, tol=1e-3)
    want = O.pcg_solve_multi(om, OP, B, tol=1e-3)
    assert np.array_equal(got["iterations"], want["iterations"])
    assert got["converged"].all()
    for j in range(8):
        x, ox = got["X"][:, j], want["X"][:, j]
        assert np.linalg.norm(x - ox) / np.linalg.norm(ox) < 1e-8
        np.testing.assert_allclose(got["tridiags"][j][0], want["tridiags"][j][0], rtol=1e-8)
        np.testing.assert_allclose(got["tridiags"][j][1], want["tridiags"][j][1], rtol=1e-8)
    # tight tolerance against the dense solve
    dense = DM.dense_fsa_cov(locs, ind, 1.5, 1, kw["gamma"], kw["sigma2"], kw["sigma1_2"], kw["rho"])
    tight = fsa.pcg_solve_multi(md, P, B[:, :2], tol=1e-10, max_iter=2000)
    want_x = np.linalg.solve(dense, B[:, :2])
    assert np.linalg.norm(tight["X"] - want_x) / np.linalg.norm(want_x) < 1e-8


def test_pcg_edge_cases():
    locs, ind, kw, md, om = setup(n=600, m=32, seed=17)
    P = fsa.make_preconditioner(md, "fitc")
    B = np.zeros((600, 3))
    B[:, 1] = 1.0
    r = fsa.pcg_solve_multi(md, P, B, tol=1e-6)
    assert r["iterations"][0] == 0 and r["converged"][0] and np.all(r["X"][:, 0] == 0)
    assert r["iterations"][1] > 0
    # unpreconditioned and Jacobi arms against the oracle
    # (plain CG over ~65 iterations loses orthogonality, so a rounding-level change of
    # the operator can move the stopping sweep by one or two: compare to the
    # reference's own re-association tolerance, test_krylov.cpp:94-111)
    for kind in ("none", "diagonal"):
        g = fsa.pcg_solve_multi(md, fsa.make_preconditioner(md, kind), B[:, 1:2], tol=1e-8, max_iter=3000)
        w = O.pcg_solve_multi(om, O.Precond(om, kind), B[:, 1:2], tol=1e-8, max_iter=3000)
        assert abs(int(g["iterations"][0]) - int(w["iterations"][0])) <= 2, kind
        assert rel(g["X"], w["X"]) < 1e-7
    # sigma_s-only solves with Jacobi (prediction.cpp:90-98)
    g = fsa.pcg_solve_multi(md, fsa.Preconditioner(md, "jacobi"), B[:, 1:2], tol=1e-8, op="sigma_s")
    w = O.pcg_solve_multi(om, O.Precond(om, "jacobi"), B[:, 1:2], tol=1e-8, op="sigma_s")
    assert g["iterations"][0] == w["iterations"][0]
    assert rel(g["X"], w["X"]) < 1e-9


def test_vanishing_taper_fitc_exact():  # test_preconditioners.cpp:145-158
    locs = O.uniform_locations(500, 2, 17)
    ind = O.select_kmeanspp(locs, 15, 18)
    md = fsa.FsaModel.assemble(locs, ind, gamma=1e-6, sigma2=0.5, sigma1_2=1.0, rho=0.1)
    assert md.info()["nnz"] == 500
    P = fsa.make_preconditioner(md, "fitc")
    r = fsa.pcg_solve_multi(md, P, np.random.default_rng(19).standard_normal(500), tol=1e-8)
    assert r["converged"][0] and r["iterations"][0] <= 2


@pytest.mark.parametrize("cv", ["optimal", "none", "one"])
def test_iterative_nll_grad_matches_oracle(cv):
    locs, ind, kw, md, om = setup(n=2500, m=80, seed=23, s2=0.1, rho=0.08)
    y = fsa.simulate_rff(locs, 1.5, 1.0, 0.08, 0.1, 256, 5)
    X = np.column_stack([np.ones(2500), locs[:, 0]])
    P, OP = fsa.make_preconditioner(md, "fitc"), O.Precond(om, "fitc")
    got = fsa.iterative_nll_grad(md, P, y, X, num_probes=20, seed=9, cv=cv)
    want = O.iterative_nll_grad(om, OP, y, X, num_probes=20, seed=9, cv=cv)
    assert got["cg_iterations"] == want["cg_iterations"]
    assert got["nll"] == pytest.approx(want["nll"], rel=1e-6)
    assert got["logdet"] == pytest.approx(want["logdet"], rel=1e-6)
    np.testing.assert_allclose(got["beta"], want["beta"], rtol=1e-6)
    np.testing.assert_allclose(got["grad"], want["grad"], rtol=1e-6, atol=1e-6 * np.abs(want["grad"]).max())


def test_iterative_nll_other_preconditioners():
    locs, ind, kw, md, om = setup(n=1000, m=40, seed=29, s2=0.3)
    y = np.random.default_rng(4).standard_normal(1000)
    for kind in ("none", "diagonal"):
        got = fsa.iterative_nll_grad(md, fsa.make_preconditioner(md, kind), y, num_probes=12, seed=3, tol=1e-6)
        want = O.iterative_nll_grad(om, O.Precond(om, kind), y, num_probes=12, seed=3, tol=1e-6)
        assert got["nll"] == pytest.approx(want["nll"], rel=1e-6), kind
        np.testing.assert_allclose(got["grad"], want["grad"], rtol=1e-6, atol=1e-6 * np.abs(want["grad"]).max())


def test_nll_deterministic_in_seed():  # test_estimation.cpp:176-194
    locs, ind, kw, md, om = setup(n=900, m=30, seed=31)
    y = np.random.default_rng(13).standard_normal(900)
    P = fsa.make_preconditioner(md, "fitc")
    a = fsa.iterative_nll_grad(md, P, y, num_probes=10, seed=17)
    b = fsa.iterative_nll_grad(md, P, y, num_probes=10, seed=17)
    assert a["nll"] == b["nll"] and np.array_equal(a["grad"], b["grad"]) and a["logdet"] == b["logdet"]


def test_errors_surface():
    locs = O.uniform_locations(200, 2, 1)
    ind = np.vstack([locs[:10], locs[:10]])  # duplicated inducing points, no jitter: singular
    with pytest.raises(fsa.NumericalError):
        fsa.FsaModel.assemble(locs, ind, gamma=0.1, jitter_rel=0.0)
    with pytest.raises(ValueError):
        fsa.FsaModel.assemble(locs, locs[:10], gamma=0.1, sigma2=-1.0)
    with pytest.raises(ValueError):
        fsa.FsaModel.assemble(locs, locs[:10], gamma=0.0)


def test_prediction_matches_oracle():
    locs, ind, kw, md, om = setup(n=1500, m=50, seed=41)
    plocs = O.uniform_locations(700, 2, 141)
    pr, opr = fsa.make_prediction_set(md, plocs), O.PredictionSet(om, plocs)
    assert pr.nnz() == opr.nnz
    u = np.random.default_rng(5).standard_normal(1500)
    assert rel(pr.cross_apply_t(u), opr.cross_apply_t(u)) < 1e-11
    P, OP = fsa.make_preconditioner(md, "fitc"), O.Precond(om, "fitc", plain=True)
    mean = pr.predict_mean_iterative(u, P, tol=1e-9)
    assert rel(mean, opr.predict_mean_iterative(u, OP, tol=1e-9)) < 1e-8
    d = pr.det_pieces(tol=1e-3, tol_s=1e-3)
    od = opr.det_pieces(tol=1e-3, tol_s=1e-3)
    assert d[3] == od[3]
    for a, b in zip(d[:3], od[:3]):
        assert np.abs(a - b).max() < 1e-8 * max(1.0, np.abs(b).max())
    sim = pr.predict_var_sim(num_probes=300, seed=7)
    osim = opr.predict_var_sim(num_probes=300, seed=7)
    assert np.abs(sim["var"] - osim["var"]).max() < 1e-6
    assert np.abs(sim["se"] - osim["se"]).max() < 1e-6
    assert sim["clamped"] == osim["clamped"]
    cvs = pr.predict_var_sim(num_probes=300, seed=7, control_variate=True)
    ocv = opr.predict_var_sim(num_probes=300, seed=7, control_variate=True)
    assert np.abs(cvs["var"] - ocv["var"]).max() < 1e-6


def test_prediction_many_inducing_matches_oracle():
    """m = 300 inducing points: the deterministic pieces solve with m_pad = 384 right-hand
    sides (column slabs in the SpMM, N-tiled GEMMs)."""
    locs, ind, kw, md, om = setup(n=3000, m=300, seed=43, gamma=0.05, rho=0.08)
    plocs = O.uniform_locations(500, 2, 143)
    pr, opr = fsa.make_prediction_set(md, plocs), O.PredictionSet(om, plocs)
    d = pr.det_pieces(tol=1e-3, tol_s=1e-3)
    od = opr.det_pieces(tol=1e-3, tol_s=1e-3)
    assert d[3] == od[3]
    for a, b in zip(d[:3], od[:3]):
        assert np.abs(a - b).max() < 1e-8 * max(1.0, np.abs(b).max())
    sim = pr.predict_var_sim(num_probes=260, seed=3)  # two probe batches (256 + 4)
    osim = opr.predict_var_sim(num_probes=260, seed=3)
    assert np.abs(sim["var"] - osim["var"]).max() < 1e-6


def test_sim_variance_converges_to_exact():  # test_prediction.cpp:105-125
    locs = O.uniform_locations(200, 2, 17)
    plocs = O.uniform_locations(50, 2, 117)
    ind = O.select_kmeanspp(locs, 12, 18)
    md = fsa.FsaModel.assemble(locs, ind, gamma=0.18, sigma2=0.3, sigma1_2=1.0, rho=0.1)
    pr = fsa.make_prediction_set(md, plocs)
    dense = DM.dense_fsa_cov(locs, ind, 1.5, 1, 0.18, 0.3, 1.0, 0.1)
    cross = DM.dense_cross(locs, plocs, ind, 1.5, 1, 0.18, 1.0, 0.1)
    ex = 1.3 - (cross * np.linalg.solve(dense, cross)).sum(0)
    sim = pr.predict_var_sim(num_probes=3000, seed=19, tol=1e-8, tol_s=1e-8)
    assert int((np.abs(sim["var"] - ex) <= 4 * sim["se"] + 1e-8).sum()) >= 47
    assert np.sqrt(((sim["var"] - ex) ** 2).mean()) < 0.05


def test_config1_scale_matches_oracle():
    """BASELINE config 1 shape (n=1e4, m=200 random, Matern-1/2, ~30 nnz/row, t=51)."""
    n, m = 10000, 200
    locs = fsa.uniform_locations(n, 2, 1)
    ind = fsa.select_random(locs, m, 2)
    gamma = fsa.gamma_for_avg_row_nnz(n, 30.0)
    y = fsa.simulate_rff(locs, 0.5, 1.0, 0.1, 0.1, 1024, 3)
    kw = dict(nu=0.5, taper_family=1, gamma=gamma, sigma2=0.1, sigma1_2=1.0, rho=0.1)
    md = fsa.FsaModel.assemble(locs, ind, **kw)
    om = O.Model(locs, ind, **kw)
    got = fsa.iterative_nll_grad(md, fsa.make_preconditioner(md, "fitc"), y, num_probes=50, seed=0)
    want = O.iterative_nll_grad(om, O.Precond(om, "fitc"), y, num_probes=50, seed=0)
    assert got["cg_iterations"] == want["cg_iterations"]
    assert got["nll"] == pytest.approx(want["nll"], rel=1e-6)
    np.testing.assert_allclose(got["grad"], want["grad"], rtol=1e-6, atol=1e-6 * np.abs(want["grad"]).max())


@pytest.mark.parametrize("d,n,m,L", [(1, 3000, 40, 20), (3, 3000, 80, 30), (2, 4000, 100, 64), (2, 2000, 130, 5)])
def test_nll_dimensions_and_widths_match_oracle(d, n, m, L):
    """d = 1 and 3 geometries, t_pad = 72 (DMMA dense passes, 64 + 8 column SpMM tiles),
    m_pad = 256 with a ragged m, tiny t."""
    locs = O.uniform_locations(n, d, 41 + d)
    ind = O.select_kmeanspp(locs, m, 42 + d)
    gamma = {1: 0.01, 2: 0.06, 3: 0.15}[d]
    kw = dict(nu=1.5, taper_family=1, gamma=gamma, sigma2=0.1, sigma1_2=1.0, rho=0.1)
    y = np.random.default_rng(d).standard_normal(n)
    md = fsa.FsaModel.assemble(locs, ind, **kw)
    om = O.Model(locs, ind, **kw)
    got = fsa.iterative_nll_grad(md, fsa.make_preconditioner(md, "fitc"), y, num_probes=L, seed=2, tol=1e-3)
    want = O.iterative_nll_grad(om, O.Precond(om, "fitc"), y, num_probes=L, seed=2, tol=1e-3)
    assert got["cg_iterations"] == want["cg_iterations"]
    assert got["nll"] == pytest.approx(want["nll"], rel=1e-6)
    np.testing.assert_allclose(got["grad"], want["grad"], rtol=1e-6, atol=1e-6 * np.abs(want["grad"]).max())


@pytest.mark.parametrize("rademacher,L", [(False, 24), (True, 9)])
def test_fisher_ste_matches_oracle(rademacher, L):  # fsa.cpp:284-301 (test_fsa.cpp:182-215)
    locs, ind, kw, md, om = setup(n=1200, m=50, seed=11)
    want = O.fisher_ste(om, num_probes=L, seed=5, rademacher=rademacher)  # exact dense solves
    got = fsa.fisher_ste(md, num_probes=L, seed=5, rademacher=rademacher, tol=1e-11)  # FITC-PCG solves
    assert np.abs(got - got.T).max() <= 1e-12 * np.abs(got).max()
    # same probes, solves to 1e-11: agreement to the north-star scalar tolerance
    assert rel(got, want) < 1e-6, (got, want)


def test_handles_outlive_their_context():
    # handles are reference counted: destroying the context (then the model) before the
    # preconditioner, prediction set and geometry must neither crash nor break those handles
    locs = O.uniform_locations(2000, 2, 31)
    ind = O.select_random(locs, 40, 32)
    ctx = fsa.Context(0)
    g = fsa.Geometry(locs, 0.05, ctx=ctx)
    md = fsa.FsaModel.assemble(None, ind, geometry=g, nu=1.5, taper_family=1, gamma=0.05, sigma2=0.2,
                               sigma1_2=1.0, rho=0.1)
    P = fsa.make_preconditioner(md, "fitc")
    pr = fsa.PredictionSet(md, O.uniform_locations(300, 2, 33))
    fsa.lib().fsa_ctx_destroy(ctx.h)
    ctx.h = None
    z = P.sample_probes(3, 1)  # the model and its context are still alive through P
    assert np.isfinite(z).all()
    fsa.lib().fsa_model_destroy(md.h)
    md.h = None
    assert np.isfinite(P.logdet())
    del pr, P, g
