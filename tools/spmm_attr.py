"""Attribute k_spmm_rt time (config 2): each component switched off in turn (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_14492_b200 import fsa
from tests.golden.configs import CONFIGS
cfg = CONFIGS[2]
ctx = fsa.Context(0)
coords = fsa.uniform_locations(cfg["n"], 2, 1)
gamma = fsa.gamma_for_avg_row_nnz(cfg["n"], cfg["nnz"])
ind = fsa.select_kmeanspp(coords, cfg["m"], 2, device=True, ctx=ctx)
md = fsa.FsaModel.assemble(coords, ind, ctx=ctx, nu=1.5, taper_family=1, gamma=gamma, sigma2=0.05, sigma1_2=1.0, rho=0.05)
names = {16: "full, no L2 prefetch", 0: "full", 1: "no DMMA", 2: "no epilogue", 4: "no RHS gather", 8: "no A tiles", 3: "no DMMA+epi",
         12: "no loads", 13: "no loads+DMMA", 14: "no loads+epi", 15: "nothing"}
for k in (51,):
    for fl, nm in names.items():
        ms = md.debug_kernel_bench(0, k, 50, fl)
        print(f"spmm k={k} {nm:16s} {ms*1e3:8.1f} us", flush=True)
    print(f"project k={k} {md.debug_kernel_bench(1, k, 50, 0)*1e3:8.1f} us")
    print(f"expand  k={k} {md.debug_kernel_bench(2, k, 50, 0)*1e3:8.1f} us")
