"""Row-sharded fit path on one GPU.

``Context.group(0, P)`` makes P ranks on cuda:0 whose collectives are host
barriers plus device copies (no kernel waits on another kernel). Each rank owns
a contiguous block of the Hilbert-sorted points, keeps a halo of the points its
taper rows reference, exchanges the halo rows of the RHS block every PCG sweep
and sums the m x t projections and the per-column dots. The sharded
``iterative_nll_grad`` must give the single-rank answer (same CG iteration
counts; nll, gradient, logdet and beta to summation-order rounding) and the
oracle's answer to the north-star tolerance.
"""
import threading

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

fsa = pytest.importorskip("paper_2405_14492_b200.fsa")


def run_ranks(ctxs, fn):
    out, errs = [None] * len(ctxs), [None] * len(ctxs)

    def work(r):
        try:
            out[r] = fn(r, ctxs[r])
        except BaseException as e:  # noqa: BLE001 - reported below
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(len(ctxs))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in errs:
        if e is not None:
            raise e
    return out


def problem(n, m, gamma, seed, p=1):
    locs = O.uniform_locations(n, 2, seed)
    ind = O.select_kmeanspp(locs, m, seed + 1)
    kw = dict(nu=1.5, taper_family=1, gamma=gamma, sigma2=0.3, sigma1_2=1.0, rho=0.12)
    y = fsa.simulate_rff(locs, 1.5, 1.0, 0.12, 0.3, 256, seed + 2)
    X = np.column_stack([np.ones(n), locs[:, 0]])[:, :p] if p > 0 else None
    return locs, ind, kw, y, X


def nll_on(ctx, locs, ind, kw, y, X, L=12, seed=5, tol=1e-6, cv="optimal", resident=True):
    g = fsa.Geometry(locs, kw["gamma"], ctx=ctx)
    md = fsa.FsaModel.assemble(None, ind, geometry=g, **kw)
    P = fsa.make_preconditioner(md, "fitc")
    if resident:
        g.set_response(y, X)
        r = fsa.iterative_nll_grad(md, P, None, num_probes=L, seed=seed, tol=tol, cv=cv)
    else:
        r = fsa.iterative_nll_grad(md, P, y, X, num_probes=L, seed=seed, tol=tol, cv=cv)
    r["shard"] = g.shard_info()
    r["P_logdet"] = P.logdet()
    r["traces"] = [P.deriv_trace(k) for k in range(3)]
    return r


def close(a, b, tol):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.all(np.abs(a - b) <= tol * np.maximum(np.abs(b), 1.0))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_nll_matches_single_rank(world):
    locs, ind, kw, y, X = problem(6000, 80, 0.05, 11, p=2)
    one = nll_on(fsa.Context(0), locs, ind, kw, y, X)
    ctxs = fsa.Context.group(0, world)
    outs = run_ranks(ctxs, lambda r, c: nll_on(c, locs, ind, kw, y, X))
    # blocks tile [0, n) and every rank has a halo
    blocks = sorted(o["shard"][:2] for o in outs)
    assert blocks[0][0] == 0 and blocks[-1][1] == 6000
    assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
    assert all(o["shard"][2] > 0 for o in outs)
    for o in outs:
        # identical on every rank (same reductions in the same order)
        assert o["nll"] == outs[0]["nll"] and np.array_equal(o["grad"], outs[0]["grad"])
        assert o["cg_iterations"] == one["cg_iterations"]
        assert close(o["nll"], one["nll"], 1e-10)
        assert close(o["logdet"], one["logdet"], 1e-10)
        assert close(o["grad"], one["grad"], 1e-8)
        assert close(o["beta"], one["beta"], 1e-9)
        assert close(o["P_logdet"], one["P_logdet"], 1e-12)
        assert close(o["traces"], one["traces"], 1e-10)


def test_sharded_72_column_pair_path_matches_single_rank():
    """t = 65 -> t_pad = 72 (config 4's block: the paired INT8 passes, ozaki_*_pair) on 2 row
    ranks against one rank: the pair path under sharding (projection summed over ranks after the
    paired launch, r.z partials of both column tiles)."""
    locs, ind, kw, y, X = problem(8000, 150, 0.04, 31, p=0)
    one = nll_on(fsa.Context(0), locs, ind, kw, y, X, L=64, tol=1e-3)
    outs = run_ranks(fsa.Context.group(0, 2), lambda r, c: nll_on(c, locs, ind, kw, y, X, L=64, tol=1e-3))
    for o in outs:
        assert o["nll"] == outs[0]["nll"]
        assert o["cg_iterations"] == one["cg_iterations"]
        assert close(o["nll"], one["nll"], 1e-10)
        assert close(o["grad"], one["grad"], 1e-8)


def test_sharded_nll_matches_oracle_host_inputs():
    locs, ind, kw, y, X = problem(4000, 64, 0.06, 23, p=1)
    ctxs = fsa.Context.group(0, 2)
    outs = run_ranks(ctxs, lambda r, c: nll_on(c, locs, ind, kw, y, X, L=10, seed=3, resident=False))
    om = O.Model(locs, ind, **kw)
    ref = O.iterative_nll_grad(om, O.Precond(om, "fitc"), y, X, num_probes=10, seed=3, tol=1e-6, cv="optimal")
    for o in outs:
        assert o["cg_iterations"] == ref["cg_iterations"]
        assert o["nll"] == pytest.approx(ref["nll"], rel=1e-6)
        np.testing.assert_allclose(o["grad"], ref["grad"], rtol=1e-6, atol=1e-8)


def test_sharded_without_covariates_and_narrow_halo():
    # tiny taper range: blocks barely touch; p = 0 (no GLS step)
    locs, ind, kw, y, _ = problem(3000, 40, 0.015, 31, p=0)
    one = nll_on(fsa.Context(0), locs, ind, kw, y, None, L=8)
    outs = run_ranks(fsa.Context.group(0, 4), lambda r, c: nll_on(c, locs, ind, kw, y, None, L=8))
    for o in outs:
        assert o["cg_iterations"] == one["cg_iterations"]
        assert close(o["nll"], one["nll"], 1e-10)
        assert close(o["grad"], one["grad"], 1e-8)


def test_sharded_context_rejects_host_block_calls():
    locs, ind, kw, y, X = problem(1500, 30, 0.08, 41)

    def body(r, c):
        assert c.rank_world() == (r, 2)
        g = fsa.Geometry(locs, kw["gamma"], ctx=c)
        md = fsa.FsaModel.assemble(None, ind, geometry=g, **kw)
        errs = 0
        for call in (lambda: md.matmat(np.ones((1500, 1))), lambda: g.pattern(),
                     lambda: fsa.make_preconditioner(md, "diagonal"),
                     lambda: fsa.make_prediction_set(md, locs[:10])):
            try:
                call()
            except ValueError:
                errs += 1
        return errs

    assert run_ranks(fsa.Context.group(0, 2), body) == [4, 4]


def test_nccl_context_single_rank():
    """NCCL communicator path (dlopen, unique id, init) at world size 1 gives the plain answer."""
    locs, ind, kw, y, X = problem(2500, 40, 0.06, 51, p=1)
    one = nll_on(fsa.Context(0), locs, ind, kw, y, X, L=6)
    uid = fsa.nccl_unique_id()
    assert len(uid) == 128
    c = fsa.Context.nccl(0, 0, 1, uid)
    assert c.rank_world() == (0, 1)
    r = nll_on(c, locs, ind, kw, y, X, L=6)
    assert r["nll"] == one["nll"] and np.array_equal(r["grad"], one["grad"])


@pytest.mark.parametrize("cv", [False, True])
def test_replicated_prediction_shards_probe_batches(cv):
    """Replicated mode: whole model per rank, predict_var_sim's probe batches split over ranks."""
    locs, ind, kw, y, X = problem(4000, 60, 0.06, 61, p=0)
    plocs = O.uniform_locations(500, 2, 62)

    def run(c):
        md = fsa.FsaModel.assemble(locs, ind, ctx=c, **kw)
        pr = fsa.make_prediction_set(md, plocs)
        out = pr.predict_var_sim(num_probes=600, seed=3, tol=1e-6, tol_s=1e-6, control_variate=cv)
        out["mean"] = pr.predict_mean_iterative(y, fsa.make_preconditioner(md, "fitc"), tol=1e-6)
        return out

    one = run(fsa.Context(0))
    ctxs = fsa.Context.group(0, 3)
    for c in ctxs:
        c.set_replicated(True)
    outs = run_ranks(ctxs, lambda r, c: run(c))
    for o in outs:  # 3 batches of <= 256 probes, one per rank; sums in another order
        np.testing.assert_allclose(o["var"], one["var"], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(o["se"], one["se"], rtol=1e-9, atol=1e-14)
        np.testing.assert_allclose(o["mean"], one["mean"], rtol=1e-13, atol=1e-14)
        assert o["cg_iterations"] == one["cg_iterations"]


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_fisher_matches_single(P):
    # fisher_ste (fsa.cpp:284-301) over row blocks: the probe rows, halo exchanges and the
    # summed 3 x 3 dots give the single-rank matrix
    locs, ind, kw, y, X = problem(3000, 60, 0.05, 23, p=0)

    def fisher_on(ctx):
        g = fsa.Geometry(locs, kw["gamma"], ctx=ctx)
        md = fsa.FsaModel.assemble(None, ind, geometry=g, **kw)
        Pc = fsa.make_preconditioner(md, "fitc")
        return fsa.fisher_ste(md, num_probes=6, seed=3, P=Pc, tol=1e-10)

    want = fisher_on(fsa.Context(0))
    got = run_ranks(fsa.Context.group(0, P), lambda r, c: fisher_on(c))
    for F in got:
        assert np.abs(F - want).max() <= 1e-8 * np.abs(want).max()
