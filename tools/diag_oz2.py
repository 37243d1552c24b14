"""Which entries of the Ozaki expansion planes are off? Expand identity columns (exact U rows)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2405_14492_b200 import fsa

n, m = 100000, 500
locs = O.uniform_locations(n, 2, 1)
ind = O.select_kmeanspp(locs, m, 2)
kw = dict(nu=1.5, taper_family=1, gamma=O.gamma_for_avg_row_nnz(n, 80), sigma2=0.05, sigma1_2=1.0, rho=0.05)
ctx = fsa.Context(0)
md = fsa.FsaModel.assemble(locs, ind, ctx=ctx, **kw)
for trial in range(2):
    Uo, Ud = np.zeros((n, m)), np.zeros((n, m))
    for c0 in range(0, m, 64):
        w = min(64, m - c0)
        E = np.zeros((m, w)); E[np.arange(c0, c0 + w), np.arange(w)] = 1.0
        ctx.set_gemm_mode("ozaki"); Uo[:, c0:c0 + w] = md.lowrank_expand(E)
        ctx.set_gemm_mode("dmma"); Ud[:, c0:c0 + w] = md.lowrank_expand(E)
    rmax = np.abs(Ud).max(axis=1)
    err = np.abs(Uo - Ud) / rmax[:, None]
    bad = np.argwhere(err > 1e-14)
    print("trial", trial, "max rel-to-row-max err", err.max(), "entries > 1e-14:", len(bad), flush=True)
    rows = np.unique(bad[:, 0])
    print("bad rows", rows[:20].tolist(), "count", len(rows))
    for r in rows[:5]:
        cs = bad[bad[:, 0] == r][:, 1]
        print(" row", r, "rowmax", rmax[r], "cols", cs[:10].tolist(), "ozaki", Uo[r, cs[:4]], "dmma", Ud[r, cs[:4]])
    # second model build: are the bad rows the same (deterministic) or random (race)?
    del md
    md = fsa.FsaModel.assemble(locs, ind, ctx=ctx, **kw)
