"""Row-sharded loglik/gradient over REAL NCCL ranks: one process per GPU.

Needs >= 2 visible GPUs and self-skips otherwise (the round's GPU box has one). Each process
creates ``Context.nccl(rank, rank, W, uid)`` on its own device, builds the sharded geometry and
runs iterative_nll_grad; the halo rows travel by ncclSend/Recv and the sums by the fixed-order
allreduce (NCCL all-gather + rank-ordered add, comm.cu). Because that order is the in-process
thread group's order, the NCCL ranks must reproduce the one-GPU thread-group run with the same
world size BITWISE, and the single-rank answer to 1e-10 (the row partials only re-associate).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
fsa = pytest.importorskip("paper_2405_14492_b200.fsa")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import json, os, sys, time
sys.path.insert(0, %(root)r)
from tests import test_gpu_sharded as T
from paper_2405_14492_b200 import fsa
rank, world, uid_path = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
if rank == 0:
    with open(uid_path + ".tmp", "wb") as f:
        f.write(fsa.nccl_unique_id())
    os.replace(uid_path + ".tmp", uid_path)
t0 = time.time()
while not os.path.exists(uid_path):
    time.sleep(0.05)
    if time.time() - t0 > 120:
        raise SystemExit("no unique id")
uid = open(uid_path, "rb").read()
ctx = fsa.Context.nccl(rank, rank, world, uid)
locs, ind, kw, y, X = T.problem(6000, 80, 0.05, 11, p=2)
r = T.nll_on(ctx, locs, ind, kw, y, X)
print(json.dumps({"rank": rank, "nll": r["nll"], "grad": list(r["grad"]), "logdet": r["logdet"],
                  "beta": list(r["beta"]), "cg_iterations": r["cg_iterations"], "shard": list(r["shard"])}))
"""


@pytest.mark.parametrize("world", [2])
def test_nccl_processes_match_thread_group_and_single_rank(world, tmp_path):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, {torch.cuda.device_count()} visible")
    from tests import test_gpu_sharded as T

    uid_path = str(tmp_path / "uid")
    code = WORKER % {"root": ROOT}
    procs = [subprocess.Popen([sys.executable, "-c", code, str(r), str(world), uid_path], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=600)
        assert p.returncode == 0, e[-3000:]
        outs.append(json.loads(o.strip().splitlines()[-1]))
    locs, ind, kw, y, X = T.problem(6000, 80, 0.05, 11, p=2)
    one = T.nll_on(fsa.Context(0), locs, ind, kw, y, X)
    grp = T.run_ranks(fsa.Context.group(0, world), lambda r, c: T.nll_on(c, locs, ind, kw, y, X))
    for o in outs:
        assert o["nll"] == outs[0]["nll"] and o["grad"] == outs[0]["grad"]  # identical on every rank
        g = grp[o["rank"]]
        assert o["nll"] == g["nll"] and np.array_equal(np.array(o["grad"]), g["grad"])  # = thread group
        assert o["cg_iterations"] == one["cg_iterations"]
        assert abs(o["nll"] - one["nll"]) <= 1e-10 * abs(one["nll"])
        np.testing.assert_allclose(o["grad"], one["grad"], rtol=1e-8, atol=1e-8)
