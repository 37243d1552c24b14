"""Config 5 (clustered, nugget 1e-3, m = 1000): accuracy of the FITC preconditioner application.
z = P^{-1} r from (a) the oracle (the reference's formulation: core = Sigma_m + Sigma_mn D^-1 Sigma_mn^T,
preconditioners.cpp) and (b) the GPU's U-form (Q = I + U D^-1 U^T); residual ||P z - r|| / ||r|| with P
applied afresh as U^T U z + D z (fp64 DMMA products of the GPU's U)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2405_14492_b200 import fsa
from tests.golden.configs import CONFIGS, calibrate_gamma, model_kw
cfg = CONFIGS[5]
ctx = fsa.Context(0)
coords = fsa.blob_locations(cfg["n"], 2, 50, 0.01, 1)
gamma = calibrate_gamma(cfg["n"], cfg["nnz"], lambda g: fsa.Geometry(coords, g, ctx).nnz())
ind = fsa.select_kmeanspp(coords, cfg["m"], 2, device=True, ctx=ctx)
y = fsa.simulate_rff(coords, cfg["nu"], cfg["s12"], cfg["rho"], cfg["s2"], 1024, 3)
kw = model_kw(cfg, gamma)
md = fsa.FsaModel.assemble(coords, ind, ctx=ctx, **kw)
ctx.set_gemm_mode("dmma")
P = fsa.make_preconditioner(md, "fitc")
sdiag, low = md.diagonals()
rng = np.random.default_rng(0)
R = np.column_stack([y, rng.standard_normal(cfg["n"]), P.sample_probes(2, 0)])
def apply_P(Z):
    return md.lowrank_expand(md.lowrank_project(Z)) + sdiag[:, None] * Z
zg = P.solve_mat(R)
t0 = time.time()
om = O.Model(coords, ind, **kw)
op = O.Precond(om, "fitc")
zo = op.solve_mat(R)
print(f"oracle build+solve {time.time() - t0:.0f} s", flush=True)
for name, z in (("gpu U-form", zg), ("oracle (reference formulation)", zo)):
    res = np.linalg.norm(apply_P(z) - R, axis=0) / np.linalg.norm(R, axis=0)
    print(f"{name:32s} ||P z - r|| / ||r|| per column: {res}")
print("relative difference gpu vs oracle z:", np.linalg.norm(zg - zo, axis=0) / np.linalg.norm(zg, axis=0))
print("logdet P: gpu", P.logdet(), "oracle", op.logdet())
