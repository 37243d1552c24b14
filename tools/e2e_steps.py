"""Phases of bench.py's e2e step at config 2 (host buffers through the C ABI), wall clock."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_14492_b200 import fsa
from tests.golden.configs import CONFIGS, model_kw
import bench
cfg = CONFIGS[2]
ctx = fsa.Context(0)
coords, ind, gamma, y = bench.make_inputs(cfg, fsa, ctx)
kw = model_kw(cfg, gamma)
for i in range(4):
    ctx.synchronize()
    t0 = time.perf_counter()
    md = fsa.FsaModel.assemble(coords, ind, ctx=ctx, **kw)
    t1 = time.perf_counter()
    P = fsa.make_preconditioner(md, "fitc")
    t2 = time.perf_counter()
    ctx.synchronize()
    t3 = time.perf_counter()
    r = fsa.iterative_nll_grad(md, P, y, num_probes=cfg["L"], seed=0, tol=cfg["tol"])
    ctx.synchronize()
    t4 = time.perf_counter()
    print(f"assemble call {1e3*(t1-t0):.2f} ms, precond call {1e3*(t2-t1):.2f}, sync {1e3*(t3-t2):.2f}, "
          f"nll {1e3*(t4-t3):.2f} (pcg {r['pcg_ms']:.2f}), total {1e3*(t4-t0):.2f}", flush=True)
    del P, md
# the resident (bench value) path for comparison: geometry built once, response and probes cached
geo = fsa.Geometry(coords, gamma, ctx)
geo.set_response(y)
geo.cache_probes(True)
for i in range(4):
    ctx.synchronize()
    t0 = time.perf_counter()
    md = fsa.FsaModel.assemble(None, ind, geometry=geo, **kw)
    t1 = time.perf_counter()
    P = fsa.make_preconditioner(md, "fitc")
    t2 = time.perf_counter()
    ctx.synchronize()
    t3 = time.perf_counter()
    r = fsa.iterative_nll_grad(md, P, None, num_probes=cfg["L"], seed=0, tol=cfg["tol"])
    ctx.synchronize()
    t4 = time.perf_counter()
    print(f"resident: assemble call {1e3*(t1-t0):.2f} ms, precond call {1e3*(t2-t1):.2f}, sync {1e3*(t3-t2):.2f}, "
          f"nll {1e3*(t4-t3):.2f} (pcg {r['pcg_ms']:.2f}), total {1e3*(t4-t0):.2f}", flush=True)
    del P, md
