"""One config-2 loglik+grad evaluation (as bench.py's step) inside an NVTX range "one_eval" after
warm-up evaluations: for ncu --nvtx --nvtx-include one_eval/ launch lists. Prints the clean wall time
and PCG time of the evaluations (CUDA events) when run without a profiler."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_14492_b200 import fsa
from tests.golden.configs import CONFIGS, model_kw
import bench

cfg = CONFIGS[int(os.environ.get("CFG", "2"))]
torch.cuda.set_device(0)
ctx = fsa.Context(0)
coords, ind, gamma, y = bench.make_inputs(cfg, fsa, ctx)
kw = model_kw(cfg, gamma)
geo = fsa.Geometry(coords, gamma, ctx)
geo.set_response(y)
geo.cache_probes(True)
stream = torch.cuda.ExternalStream(ctx.stream())


def step():
    md = fsa.FsaModel.assemble(None, ind, geometry=geo, **kw)
    P = fsa.make_preconditioner(md, "fitc")
    r = fsa.iterative_nll_grad(md, P, None, num_probes=cfg["L"], seed=0, tol=cfg["tol"])
    del P, md
    return r


for _ in range(3):
    step()
ctx.synchronize()
for i in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    torch.cuda.nvtx.range_push("one_eval")
    r = step()
    torch.cuda.nvtx.range_pop()
    e1.record(stream)
    ctx.synchronize()
    torch.cuda.synchronize()
    print(f"eval {i}: {e0.elapsed_time(e1):.3f} ms, pcg {r['pcg_ms']:.3f} ms, sweeps {r['sweeps']}", flush=True)
