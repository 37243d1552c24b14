"""INT8 tensor-core (tcgen05 kind::i8) Ozaki emulation of the fp64 dense passes.

The projection U V and the expansion U^T W (U = L^{-1} Sigma_mn) must match an
fp64 product to the accuracy of an fp64 GEMM (errors measured against
sum |U||V|, the quantity an fp64 GEMM's rounding is proportional to), and the
full loglik/gradient evaluation must agree between the Ozaki path, the DMMA
path and the oracle.
"""
import numpy as np
import pytest
from scipy.linalg import solve_triangular

from oracle import oracle as O

pytestmark = pytest.mark.gpu

fsa = pytest.importorskip("paper_2405_14492_b200.fsa")


def model(n, m, seed=3, gamma=0.05, rho=0.05, ctx=None):
    locs = O.uniform_locations(n, 2, seed)
    ind = O.select_kmeanspp(locs, m, seed + 1)
    kw = dict(nu=1.5, taper_family=1, gamma=gamma, sigma2=0.05, sigma1_2=1.0, rho=rho)
    om = O.Model(locs, ind, **kw)
    U = solve_triangular(np.tril(om.dense(7)), om.dense(1), lower=True)
    return locs, ind, kw, om, U, fsa.FsaModel.assemble(locs, ind, ctx=ctx, **kw)


@pytest.mark.parametrize("n,m,k", [(3000, 100, 8), (9000, 300, 51), (20000, 500, 64), (5000, 130, 1)])
def test_ozaki_products_match_fp64(n, m, k):
    ctx = fsa.Context(0)
    _, _, _, _, U, md = model(n, m, ctx=ctx)
    rng = np.random.default_rng(k)
    V = rng.standard_normal((n, k))
    W = rng.standard_normal((m, k))
    ref_p, ref_e = U @ V, U.T @ W
    scale_p, scale_e = np.abs(U) @ np.abs(V), np.abs(U.T) @ np.abs(W)
    out = {}
    for mode in ("ozaki", "dmma"):
        ctx.set_gemm_mode(mode)
        out[mode] = (md.lowrank_project(V), md.lowrank_expand(W))
    (po, eo), (pd, ed) = out["ozaki"], out["dmma"]
    # Ozaki vs the fp64 DMMA product with the same device U: the emulation error itself
    dp = np.max(np.abs(po - pd) / scale_p)
    de = np.max(np.abs(eo - ed) / scale_e)
    # both against U from the oracle's own Cholesky (differs from the device U by rounding,
    # amplified by the conditioning of Sigma_m)
    rp = np.max(np.abs(pd - ref_p) / scale_p)
    re = np.max(np.abs(ed - ref_e) / scale_e)
    # expansion: the scaling groups are a point's whole U column and a whole W column, so the
    # error bound is normwise per group: |dY_ij| <= 2^-53 (max_k|U_ki| sum_k|W_kj| + max_k|W_kj|
    # sum_k|U_ki|) (digit truncation at 2^-56 of each group's exponent + the dropped weight >= 10
    # products). Relative to the componentwise sum|U||W| it is ~2e-15 typically and larger only
    # where a W entry happens to be tiny exactly where U_i is concentrated (measured below).
    Ua, Wa = np.abs(U), np.abs(W)
    bound = 2.0 ** -53 * (Ua.max(axis=0)[:, None] * Wa.sum(axis=0)[None, :]
                          + Ua.sum(axis=0)[:, None] * Wa.max(axis=0)[None, :])
    dn = np.max(np.abs(eo - ed) / bound)
    comp = np.abs(eo - ed) / scale_e
    print(n, m, k, "ozaki-dmma project", dp, "expand", de, "(p99.9", np.quantile(comp, 0.999), ", normwise",
          dn, ") | dmma-ref", rp, re)
    assert dp < 5e-15
    assert dn < 1.0
    assert np.quantile(comp, 0.999) < 1e-14
    assert rp < 1e-13 and re < 1e-11


def test_ozaki_nll_matches_dmma_and_oracle():
    n, m = 8000, 150
    locs = O.uniform_locations(n, 2, 7)
    ind = O.select_kmeanspp(locs, m, 8)
    kw = dict(nu=1.5, taper_family=1, gamma=0.05, sigma2=0.05, sigma1_2=1.0, rho=0.06)
    y = fsa.simulate_rff(locs, 1.5, 1.0, 0.06, 0.05, 256, 9)
    X = np.column_stack([np.ones(n), locs[:, 1]])
    res = {}
    for mode in ("ozaki", "dmma"):
        ctx = fsa.Context(0)
        ctx.set_gemm_mode(mode)
        md = fsa.FsaModel.assemble(locs, ind, ctx=ctx, **kw)
        P = fsa.make_preconditioner(md, "fitc")
        res[mode] = fsa.iterative_nll_grad(md, P, y, X, num_probes=20, seed=4, tol=1e-3)
    om = O.Model(locs, ind, **kw)
    ref = O.iterative_nll_grad(om, O.Precond(om, "fitc"), y, X, num_probes=20, seed=4, tol=1e-3)
    a, b = res["ozaki"], res["dmma"]
    assert a["cg_iterations"] == b["cg_iterations"] == ref["cg_iterations"]
    assert a["nll"] == pytest.approx(b["nll"], rel=1e-10)
    np.testing.assert_allclose(a["grad"], b["grad"], rtol=1e-8, atol=1e-8)
    assert a["nll"] == pytest.approx(ref["nll"], rel=1e-6)
    np.testing.assert_allclose(a["grad"], ref["grad"], rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(a["beta"], ref["beta"], rtol=1e-6)


def test_ozaki_pcg_solution_matches_oracle():
    locs, ind, kw, om, U, md = model(6000, 120, seed=11)
    B = np.random.default_rng(2).standard_normal((6000, 40))
    P = fsa.make_preconditioner(md, "fitc")
    ref = O.pcg_solve_multi(om, O.Precond(om, "fitc"), B, tol=1e-3, max_iter=400)
    res = {}
    for mode in ("dmma", "ozaki"):
        md.ctx.set_gemm_mode(mode)
        res[mode] = fsa.pcg_solve_multi(md, P, B, tol=1e-3, max_iter=400)
    # ~70 iterations: any two fp64 implementations (the DMMA path vs the oracle included)
    # may stop one iteration apart on a few columns and drift apart by rounding
    # amplification; the Ozaki path must stay within the same envelope
    for mode, got in res.items():
        assert np.abs(got["iterations"] - ref["iterations"]).max() <= 1, mode
        same = np.flatnonzero(got["iterations"] == ref["iterations"])
        assert len(same) >= B.shape[1] * 3 // 4, mode
        for j in same:
            x, ox = got["X"][:, j], ref["X"][:, j]
            assert np.linalg.norm(x - ox) / np.linalg.norm(ox) < 1e-6, mode
            np.testing.assert_allclose(got["tridiags"][j][0][:20], ref["tridiags"][j][0][:20], rtol=1e-8)
    d = res["dmma"]["X"] - ref["X"]
    o = res["ozaki"]["X"] - res["dmma"]["X"]
    assert np.abs(o).max() <= 10 * np.abs(d).max() + 1e-12
    # the easy case (few iterations) matches exactly like the DMMA path does
    B2 = P.sample_probes(8, 3)
    md.ctx.set_gemm_mode("ozaki")
    got = fsa.pcg_solve_multi(md, P, B2, tol=1e-1)
    want = O.pcg_solve_multi(om, O.Precond(om, "fitc"), B2, tol=1e-1)
    assert np.array_equal(got["iterations"], want["iterations"])
    assert np.abs(got["X"] - want["X"]).max() <= 1e-8 * np.abs(want["X"]).max()


def test_ozaki_pair_72_columns_matches_dmma():
    """t = 65 -> t_pad = 72 (config 4's block): the two INT8 column tiles of ozaki_*_pair (CTA
    pairs sharing the U planes through L2) against the all-DMMA solve."""
    n, m = 12000, 200
    locs = O.uniform_locations(n, 2, 21)
    ind = O.select_kmeanspp(locs, m, 22)
    kw = dict(nu=1.5, taper_family=1, gamma=0.03, sigma2=0.05, sigma1_2=1.0, rho=0.05)
    y = fsa.simulate_rff(locs, 1.5, 1.0, 0.05, 0.05, 256, 23)
    res = {}
    for mode in ("ozaki", "dmma"):
        ctx = fsa.Context(0)
        ctx.set_gemm_mode(mode)
        md = fsa.FsaModel.assemble(locs, ind, ctx=ctx, **kw)
        P = fsa.make_preconditioner(md, "fitc")
        res[mode] = (fsa.iterative_nll_grad(md, P, y, num_probes=64, seed=4, tol=1e-3), ctx.last_cg()["iterations"])
    (a, ia), (b, ib) = res["ozaki"], res["dmma"]
    assert np.array_equal(ia, ib)
    assert a["nll"] == pytest.approx(b["nll"], rel=1e-10)
    np.testing.assert_allclose(a["grad"], b["grad"], rtol=1e-8, atol=0)
