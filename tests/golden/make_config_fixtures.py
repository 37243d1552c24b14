#!/usr/bin/env python
"""Generate the oracle fixtures of the BASELINE configurations (test infrastructure).

The oracle (oracle/fsa_oracle.cpp, the C++ restatement of the reference path) is run at the
full size of each benched configuration on seeded inputs made by the oracle's own generators:

  config 1  n = 1e4,  m = 200 random,     Matern-1/2, 50 probes, FITC, tol 1e-3  (loglik + grad)
  config 2  n = 1e5,  m = 500 k-means++,  Matern-3/2, 50 probes, FITC, tol 1e-3  (loglik + grad)
  config 5  n = 2e5 clustered, m = 1000,  Matern-5/2, 50 probes, FITC, tol 1e-4  (loglik + grad)
            plus cmd_bench_precond: Sigma x = y with none / diagonal / fitc (row n1)
  config 3  n = n_p = 1e5, m = 500: predict_var_sim with 1000 simulation vectors

and the results the GPU parity tests compare against are written to tests/golden/config*.npz:
scalars (nll, gradient, logdet, beta), per-column CG iteration counts, the residual-norm
history of every column (for the tie rule: a count mismatch is acceptable only where the
stopping residual sits within roundoff of tol), the solution X on a fixed row sample, input
checksums (so the GPU box verifies it regenerated the same inputs) and the predictive
variances on a fixed point sample.

Usage: python tests/golden/make_config_fixtures.py [1 2 3 5 ...]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.golden.configs import CONFIGS, calibrate_gamma, model_kw, sample_rows  # noqa: E402


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:32]


def oracle_inputs(cfg):
    n, m = cfg["n"], cfg["m"]
    if cfg["points"] == "uniform":
        coords = O.uniform_locations(n, 2, 1)
        gamma = O.gamma_for_avg_row_nnz(n, cfg["nnz"])
    else:
        coords = O.blob_locations(n, 2, 50, 0.01, 1)
        gamma = calibrate_gamma(n, cfg["nnz"], lambda g: O.taper_pattern(coords, g)[0][-1])
    ind = O.select_random(coords, m, 2) if cfg["inducing"] == "random" else O.select_kmeanspp(coords, m, 2)
    y = O.simulate_rff(coords, cfg["nu"], cfg["s12"], cfg["rho"], cfg["s2"], 1024, 3)
    return coords, ind, gamma, y


def run_nll(k, cfg, out):
    coords, ind, gamma, y = oracle_inputs(cfg)
    kw = model_kw(cfg, gamma)
    t0 = time.time()
    om = O.Model(coords, ind, **kw)
    P = O.Precond(om, "fitc")
    rows = sample_rows(cfg["n"])
    r = O.iterative_nll_grad_ex(om, P, y, num_probes=cfg["L"], seed=0, tol=cfg["tol"], max_iter=1000, rows=rows)
    dt = time.time() - t0
    its = r["iterations"]
    rn = np.zeros((len(its), max(int(its.max()), 1)))
    for j, h in enumerate(r["rnorm"]):
        rn[j, : len(h)] = h
    out.update(coords_sha=digest(coords), ind_sha=digest(ind), y_sha=digest(y), gamma=gamma, nll=r["nll"],
               grad=r["grad"], logdet=r["logdet"], cg_iterations=r["cg_iterations"], iterations=its, rnorm=rn,
               rows=rows, xrows=r["xrows"], oracle_seconds=dt)
    print(f"config {k}: nll={r['nll']!r} grad={r['grad']!r} logdet={r['logdet']!r} "
          f"its={int(its.min())}..{int(its.max())} ({dt:.0f} s)", flush=True)
    return om, coords, ind, gamma, y


def run_self_spread(k, cfg, om, y, out):
    """The oracle against itself under a round-off-level perturbation: the same lockstep PCG on
    [Z | y] with every entry of the right-hand side moved by one unit in the last place (random
    sign). Any two fp64 implementations of the reference sequence (krylov.cpp:56-93) differ by
    perturbations of this size at every step; the spread of the two runs' residual-norm histories
    and solutions is the round-off envelope another implementation (the GPU one) is held to."""
    P = O.Precond(om, "fitc")
    Z = P.sample_probes(cfg["L"], 0)
    B = np.asfortranarray(np.column_stack([Z, y]))
    sign = np.where(np.random.default_rng(7).random(B.shape) < 0.5, -1.0, 1.0)
    Bp = np.asfortranarray(B * (1.0 + sign * 2.0 ** -52))
    rows = out["rows"]
    t0 = time.time()
    r = O.pcg_solve_multi_ex(om, P, Bp, tol=cfg["tol"], max_iter=1000)
    ib = r["iterations"]
    rb = np.zeros((len(ib), max(int(ib.max()), 1)))
    for j, h in enumerate(r["rnorm"]):
        rb[j, : len(h)] = h
    xb = r["X"][rows].copy()
    out.update(spread_iterations=ib, spread_rnorm=rb, spread_xrows=xb)
    ia, ra, xa = out["iterations"], out["rnorm"], out["xrows"]
    same = ia == ib
    w = min(ra.shape[1], rb.shape[1])
    both = (ra[:, :w] > 0) & (rb[:, :w] > 0)
    rel = np.where(both, np.abs(ra[:, :w] - rb[:, :w]) / np.where(both, ra[:, :w], 1.0), 0.0)
    xrel = np.linalg.norm(xa - xb, axis=0) / np.linalg.norm(xa, axis=0)
    print(f"config {k} oracle self-spread ({time.time() - t0:.0f} s): counts equal {int(same.sum())}/{len(same)}, "
          f"rnorm rel by sweep {[float(rel[:, s].max()) for s in range(0, w, 10)]}, "
          f"X rel max {xrel[same].max():.3e}", flush=True)


def run_bench_precond(k, cfg, om, y, out, max_iter=1000):
    """cmd_bench_precond (tools/commands.cpp:462-510): solve Sigma x = y with each preconditioner
    ('none' -> Identity, 'diagonal', 'fitc') at the config's tolerance and the reference default
    cg.max_iter = 1000; per preconditioner the iteration count, converged flag and the
    residual-norm history (the unpreconditioned arm may stop at max_iter unconverged, as the
    reference reports it)."""
    for name in ("none", "diagonal", "fitc"):
        P = O.Precond(om, name)
        t0 = time.time()
        r = O.pcg_solve_multi_ex(om, P, y.reshape(-1, 1), tol=cfg["tol"], max_iter=max_iter)
        dt = time.time() - t0
        out.update({f"bp_{name}_iterations": int(r["iterations"][0]), f"bp_{name}_converged": bool(r["converged"][0]),
                    f"bp_{name}_rnorm": r["rnorm"][0], f"bp_{name}_seconds": dt})
        print(f"config {k} bench_precond {name}: its={int(r['iterations'][0])} converged={bool(r['converged'][0])} "
              f"final residual {r['rnorm'][0][-1]:.3e} ({dt:.0f} s)", flush=True)


def run_prediction(k, cfg, out):
    coords, ind, gamma, y = oracle_inputs(cfg)
    kw = model_kw(cfg, gamma)
    plocs = O.uniform_locations(cfg["np"], 2, 101)
    t0 = time.time()
    om = O.Model(coords, ind, **kw)
    pr = O.PredictionSet(om, plocs)
    res = pr.predict_var_sim(num_probes=cfg["L"], seed=0, tol=cfg["tol"], tol_s=cfg["tol"])
    dt = time.time() - t0
    rows = sample_rows(cfg["np"])
    out.update(coords_sha=digest(coords), ind_sha=digest(ind), plocs_sha=digest(plocs), gamma=gamma,
               rows=rows, var=res["var"][rows], se=res["se"][rows], clamped=res["clamped"],
               cg_iterations=res["cg_iterations"], var_mean=float(np.mean(res["var"])),
               se_mean=float(np.mean(res["se"])), oracle_seconds=dt)
    print(f"config {k}: var_mean={out['var_mean']!r} se_mean={out['se_mean']!r} its={res['cg_iterations']} "
          f"clamped={res['clamped']} ({dt:.0f} s)", flush=True)


def add_spread(k):
    """Append the ulp-perturbation self-spread to an existing fixture."""
    path = os.path.join(HERE, f"config{k}_oracle.npz")
    out = dict(np.load(path))
    cfg = CONFIGS[k]
    coords, ind, gamma, y = oracle_inputs(cfg)
    om = O.Model(coords, ind, **model_kw(cfg, gamma))
    run_self_spread(k, cfg, om, y, out)
    np.savez_compressed(path, **out)


def main(which):
    if which and which[0] == 0:  # 0 k...: add the self-spread run to existing fixtures
        for k in which[1:]:
            add_spread(k)
        return
    for k in which:
        cfg = CONFIGS[k]
        out = {"config": json.dumps(cfg, sort_keys=True)}
        if k == 3:
            run_prediction(k, cfg, out)
        else:
            om, coords, ind, gamma, y = run_nll(k, cfg, out)
            if k in (1, 2, 5):
                run_self_spread(k, cfg, om, y, out)
            if k == 5:
                run_bench_precond(k, cfg, om, y, out)
        np.savez_compressed(os.path.join(HERE, f"config{k}_oracle.npz"), **out)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 5, 3])
