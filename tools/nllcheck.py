import sys
sys.path.insert(0, '/root/repo')
from paper_2405_14492_b200 import fsa
n, m = 20000, 200
locs = fsa.uniform_locations(n, 2, 1); ind = fsa.select_random(locs, m, 2)
g = fsa.gamma_for_avg_row_nnz(n, 60.0)
y = fsa.simulate_rff(locs, 1.5, 1.0, 0.05, 0.05, 512, 3)
md = fsa.FsaModel.assemble(locs, ind, gamma=g, sigma2=0.05, sigma1_2=1.0, rho=0.05)
r = fsa.iterative_nll_grad(md, fsa.make_preconditioner(md, "fitc"), y, num_probes=30, seed=0)
print(repr(r["nll"]), repr(r["grad"][2]), r["cg_iterations"])
