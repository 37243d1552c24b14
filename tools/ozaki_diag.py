"""Compare the Ozaki (INT8 tensor core) and DMMA paths on one FITC-PCG problem."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2405_14492_b200 import fsa

n, m, k = 6000, 120, 40
locs = O.uniform_locations(n, 2, 11)
ind = O.select_kmeanspp(locs, m, 12)
kw = dict(nu=1.5, taper_family=1, gamma=0.05, sigma2=0.05, sigma1_2=1.0, rho=0.05)
B = np.random.default_rng(2).standard_normal((n, k))
om = O.Model(locs, ind, **kw)
ref = O.pcg_solve_multi(om, O.Precond(om, "fitc"), B, tol=1e-3, max_iter=400)
out = {}
for mode in ("dmma", "ozaki"):
    ctx = fsa.Context(0)
    ctx.set_gemm_mode(mode)
    md = fsa.FsaModel.assemble(locs, ind, ctx=ctx, **kw)
    P = fsa.make_preconditioner(md, "fitc")
    out[mode] = fsa.pcg_solve_multi(md, P, B, tol=1e-3, max_iter=400)
    V = np.random.default_rng(5).standard_normal((n, 8))
    out[mode + "_proj"] = md.lowrank_project(V)
    out[mode + "_exp"] = md.lowrank_expand(np.random.default_rng(6).standard_normal((m, 8)))
    out[mode + "_mat"] = md.matmat(V)
a, b = out["ozaki"], out["dmma"]
print("iterations oracle", ref["iterations"].tolist())
print("iterations dmma  ", b["iterations"].tolist())
print("iterations ozaki ", a["iterations"].tolist())
print("X ozaki-dmma", np.abs(a["X"] - b["X"]).max() / np.abs(b["X"]).max(), "dmma-oracle",
      np.abs(b["X"] - ref["X"]).max() / np.abs(ref["X"]).max())
for key in ("proj", "exp", "mat"):
    x, y = out["ozaki_" + key], out["dmma_" + key]
    print(key, "rel diff", np.abs(x - y).max() / np.abs(y).max())
j = int(np.argmax(a["iterations"] != b["iterations"])) if np.any(a["iterations"] != b["iterations"]) else 0
print("column", j, "tdiag tail dmma", b["tridiags"][j][0][-3:], "ozaki", a["tridiags"][j][0][-3:])
