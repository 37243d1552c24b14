"""Config-2-sized Ozaki projection / expansion for profiling (ncu) and timing."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2405_14492_b200 import fsa

n, m, k = 100_000, 500, 51
reps = int(os.environ.get("REPS", "5"))
coords = fsa.uniform_locations(n, 2, 1)
ind = fsa.select_random(coords, m, 2)
gamma = fsa.gamma_for_avg_row_nnz(n, 80)
ctx = fsa.Context(0)
md = fsa.FsaModel.assemble(coords, ind, ctx=ctx, nu=1.5, gamma=gamma, sigma2=0.05, sigma1_2=1.0, rho=0.05)
V = np.random.default_rng(0).standard_normal((n, k))
W = np.random.default_rng(1).standard_normal((m, k))
for mode in ("ozaki", "dmma"):
    ctx.set_gemm_mode(mode)
    md.lowrank_project(V); md.lowrank_expand(W)
    ctx.set_profiling(True); ctx.reset_timers()
    for _ in range(reps):
        md.lowrank_project(V); md.lowrank_expand(W)
    t = ctx.timers(); ctx.set_profiling(False)
    print(mode, {kk: round(v["ms"] / v["count"], 4) for kk, v in t.items()})
