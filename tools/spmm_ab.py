"""Time one sweep kernel group (config 2; WHICH = 0 SpMM + direction update, 1 projection, 2 expansion)
for the current FSA_* environment switches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_14492_b200 import fsa
from tests.golden.configs import CONFIGS, model_kw
cfg = CONFIGS[int(os.environ.get("CFG", "2"))]
ctx = fsa.Context(0)
coords = fsa.uniform_locations(cfg["n"], 2, 1)
gamma = fsa.gamma_for_avg_row_nnz(cfg["n"], cfg["nnz"])
ind = fsa.select_kmeanspp(coords, cfg["m"], 2, device=True, ctx=ctx)
md = fsa.FsaModel.assemble(coords, ind, ctx=ctx, **model_kw(cfg, gamma))
tag = os.environ.get("TAG", "")
k = int(os.environ.get("K", "51"))
flags = [int(f) for f in os.environ.get("FLAGS", "0").split(",")]
which = int(os.environ.get("WHICH", "0"))  # 0 SpMM, 1 projection, 2 expansion
name = {0: "spmm", 1: "project", 2: "expand"}[which]
for fl in flags:
    ms = min(md.debug_kernel_bench(which, k, 50, fl) for _ in range(3))
    print(f"{tag:12s} k={k} flags={fl:2d} {name} {ms*1e3:8.1f} us", flush=True)
