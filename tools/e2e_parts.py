"""Where the e2e (host-buffer) evaluation spends its extra time at config 2: geometry build,
host probe draws, uploads (timing helper, not a test)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_14492_b200 import fsa  # noqa: E402

n, m = 100_000, 500
coords = fsa.uniform_locations(n, 2, 1)
ind = fsa.select_kmeanspp(coords, m, 2, device=os.environ.get("DEVKM", "1") == "1")
gamma = fsa.gamma_for_avg_row_nnz(n, 80)
y = fsa.simulate_rff(coords, 1.5, 1.0, 0.05, 0.05, 1024, 3)
ctx = fsa.Context(0)
kw = dict(nu=1.5, taper_family=1, gamma=gamma, sigma2=0.05, sigma1_2=1.0, rho=0.05)


def t(f, reps=5):
    f()
    ctx.synchronize()
    out = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ctx.synchronize()
        out.append((time.perf_counter() - t0) * 1e3)
    return sorted(out)[len(out) // 2]


STAGE = int(os.environ.get("STAGE", "9"))
print("geometry build ms", t(lambda: fsa.Geometry(coords, gamma, ctx)))
if STAGE <= 1:
    sys.exit(0)
g = fsa.Geometry(coords, gamma, ctx)
print("assemble (geometry given) ms", t(lambda: fsa.FsaModel.assemble(None, ind, geometry=g, **kw)))
if STAGE <= 2:
    sys.exit(0)
print("assemble (from coords) ms", t(lambda: fsa.FsaModel.assemble(coords, ind, ctx=ctx, **kw)))
if STAGE <= 3:
    sys.exit(0)
md = fsa.FsaModel.assemble(None, ind, geometry=g, **kw)
P = fsa.make_preconditioner(md, "fitc")
print("probe draws (sample_probes, 50) ms", t(lambda: P.sample_probes(50, 0)))
