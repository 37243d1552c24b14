"""Round-2 diagnostics on the B200: Ozaki expansion accuracy on the config-2 factor, and the
config-2 solve / loglik+grad in both GEMM modes saved for comparison with the oracle fixture."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from scipy.linalg import solve_triangular  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2405_14492_b200 import fsa  # noqa: E402
from tests.golden.configs import CONFIGS, sample_rows  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
os.makedirs(OUT, exist_ok=True)
which = sys.argv[1:] or ["ozaki", "c2"]


def inputs(cfg):
    coords = fsa.uniform_locations(cfg["n"], 2, 1)
    gamma = fsa.gamma_for_avg_row_nnz(cfg["n"], cfg["nnz"])
    ind = fsa.select_kmeanspp(coords, cfg["m"], 2, device=True)
    y = fsa.simulate_rff(coords, cfg["nu"], cfg["s12"], cfg["rho"], cfg["s2"], 1024, 3)
    return coords, ind, gamma, y


if "ozaki" in which:
    for (n, m, rho) in [(20000, 500, 0.05), (100000, 500, 0.05)]:
        locs = O.uniform_locations(n, 2, 1)
        ind = O.select_kmeanspp(locs, m, 2)
        kw = dict(nu=1.5, taper_family=1, gamma=O.gamma_for_avg_row_nnz(n, 80), sigma2=0.05, sigma1_2=1.0, rho=rho)
        om = O.Model(locs, ind, **kw)
        U = solve_triangular(np.tril(om.dense(7)), om.dense(1), lower=True)
        ctx = fsa.Context(0)
        md = fsa.FsaModel.assemble(locs, ind, ctx=ctx, **kw)
        rng = np.random.default_rng(1)
        Wr = rng.standard_normal((m, 51))
        Vr = rng.standard_normal((n, 51))
        ctx.set_gemm_mode("dmma")
        Wreal = md.lowrank_project(Vr)  # S = U V: the projection shape the sweep expands after Q^{-1}
        for name, W in (("random", Wr), ("projected", Wreal)):
            res = {}
            for mode in ("ozaki", "dmma"):
                ctx.set_gemm_mode(mode)
                res[mode] = md.lowrank_expand(W)
            scale = np.abs(U.T) @ np.abs(W)
            err = np.abs(res["ozaki"] - res["dmma"]) / scale
            rowerr = err.max(axis=1)
            worst = np.argsort(rowerr)[-5:]
            umax = np.abs(U).max(axis=0)
            dyn = umax * np.abs(W).sum(axis=0).max() / np.maximum((np.abs(U.T) @ np.abs(W)).max(axis=1), 1e-300)
            print(f"expand n={n} m={m} W={name}: max err/scale {err.max():.3e}, p99 {np.quantile(rowerr, 0.99):.3e}, "
                  f"median {np.median(rowerr):.3e}; worst rows {worst.tolist()} err {rowerr[worst]} "
                  f"dyn-range {dyn[worst]} |U_i|max {umax[worst]}", flush=True)
            ctx.set_gemm_mode("ozaki")
            po = md.lowrank_project(Vr)
            ctx.set_gemm_mode("dmma")
            pd = md.lowrank_project(Vr)
            ps = np.abs(U) @ np.abs(Vr)
            print(f"project n={n}: max err/scale {(np.abs(po - pd) / ps).max():.3e}", flush=True)
        del md, ctx

if "c2" in which:
    cfg = CONFIGS[2]
    coords, ind, gamma, y = inputs(cfg)
    kw = dict(nu=cfg["nu"], taper_family=1, gamma=gamma, sigma2=cfg["s2"], sigma1_2=cfg["s12"], rho=cfg["rho"])
    rows = sample_rows(cfg["n"])
    save = {}
    for mode in ("ozaki", "dmma"):
        ctx = fsa.Context(0)
        ctx.set_gemm_mode(mode)
        md = fsa.FsaModel.assemble(coords, ind, ctx=ctx, **kw)
        P = fsa.make_preconditioner(md, "fitc")
        t0 = time.time()
        r = fsa.iterative_nll_grad(md, P, y, num_probes=cfg["L"], seed=0, tol=cfg["tol"])
        lc = ctx.last_cg()
        print(f"c2 {mode}: nll={r['nll']!r} grad={r['grad'].tolist()} logdet={r['logdet']!r} sweeps={r['sweeps']} "
              f"({time.time() - t0:.1f} s)", flush=True)
        Z = P.sample_probes(cfg["L"], 0)
        B = np.column_stack([Z, y])
        sol = fsa.pcg_solve_multi(md, P, B, tol=cfg["tol"])
        lc2 = ctx.last_cg()
        AX = md.matmat(sol["X"])
        true_res = np.linalg.norm(B - AX, axis=0)
        rec = np.array([h[-1] for h in lc2["rnorm"]])
        print(f"c2 {mode} solve: its {sol['iterations'].min()}..{sol['iterations'].max()}, true residual / tol max "
              f"{(true_res / cfg['tol']).max():.6f}, recursive/true max rel gap "
              f"{np.max(np.abs(rec - true_res) / true_res):.3e}", flush=True)
        rn = np.zeros((len(lc["iterations"]), max(lc["iterations"])))
        for j, h in enumerate(lc["rnorm"]):
            rn[j, : len(h)] = h
        save.update({f"{mode}_nll": r["nll"], f"{mode}_grad": r["grad"], f"{mode}_logdet": r["logdet"],
                     f"{mode}_its": lc["iterations"], f"{mode}_rnorm": rn, f"{mode}_solve_its": sol["iterations"],
                     f"{mode}_xrows": sol["X"][rows], f"{mode}_true_res": true_res})
        del P, md, ctx
    np.savez_compressed(os.path.join(OUT, "diag_c2.npz"), rows=rows, **save)
