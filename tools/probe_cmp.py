"""Device probe streams (k_probe_gaussian) against the host libstdc++ streams, both pushed through
the same device transform z = U^T e1 + sqrt(D) e2: run once with FSA_HOST_PROBES=1 (host draws) and
once without; the second run compares (differences come from the draws alone)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from paper_2405_14492_b200 import fsa
n, m = 20000, 300
locs = O.uniform_locations(n, 2, 5)
ind = O.select_random(locs, m, 6)
kw = dict(nu=1.5, taper_family=1, gamma=0.02, sigma2=0.1, sigma1_2=1.0, rho=0.1)
md = fsa.FsaModel.assemble(locs, ind, **kw)
P = fsa.make_preconditioner(md, "fitc")
out = sys.argv[1]
Zs = {f"{L}_{seed}": P.sample_probes(L, seed) for L, seed in ((7, 3), (50, 0))}
if os.environ.get("FSA_HOST_PROBES"):
    np.savez(out, **Zs)
else:
    ref = np.load(out)
    for k, Z in Zs.items():
        R = ref[k]
        print(f"{k}: normwise rel diff {np.abs(Z - R).max() / np.abs(R).max():.3e}, "
              f"entries differing {np.mean(Z != R):.4%}")
