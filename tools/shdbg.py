import sys, os, threading
sys.path.insert(0, '/root/repo')
import numpy as np
from oracle import oracle as O
from paper_2405_14492_b200 import fsa
sys.path.insert(0,'/root/repo/tests')
import test_gpu_sharded as T
locs, ind, kw, y, X = T.problem(6000, 80, 0.05, 11, p=2)
mode = sys.argv[1]
ref = None
for rep in range(8):
    try:
        if mode == "single":
            o = T.nll_on(fsa.Context(0), locs, ind, kw, y, X)
        elif mode == "single_threads":  # single-rank contexts driven from 2 threads at once
            outs = T.run_ranks([fsa.Context(0), fsa.Context(0)], lambda r, c: T.nll_on(c, locs, ind, kw, y, X))
            o = outs[0]
        else:
            outs = T.run_ranks(fsa.Context.group(0, int(mode)), lambda r, c: T.nll_on(c, locs, ind, kw, y, X))
            o = outs[0]
        ref = ref or o["nll"]
        print(mode, rep, o["nll"], o["cg_iterations"], o["nll"] - ref, flush=True)
    except Exception as e:
        print(mode, rep, "ERR", e, flush=True)
        os._exit(0)
