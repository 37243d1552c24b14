"""One k_spmm launch group at config 2 (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_14492_b200 import fsa
from tests.golden.configs import CONFIGS, model_kw
cfg = CONFIGS[2]
ctx = fsa.Context(0)
coords = fsa.uniform_locations(cfg["n"], 2, 1)
gamma = fsa.gamma_for_avg_row_nnz(cfg["n"], cfg["nnz"])
ind = fsa.select_kmeanspp(coords, cfg["m"], 2, device=True, ctx=ctx)
md = fsa.FsaModel.assemble(coords, ind, ctx=ctx, **model_kw(cfg, gamma))
which = int(sys.argv[1]) if len(sys.argv) > 1 else 0
print(md.debug_kernel_bench(which, 51, 3, 0))
