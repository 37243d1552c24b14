"""Row-sharded decomposition under a real multi-process gloo group (CPU).

Each rank runs ``tests/shard_mirror.py``: the block split and halo plan of
``shard_pattern`` (shard.cu), the neighbour halo exchange, and the FITC PCG
whose m x t projections and per-column dots are summed with all_reduce
(fsa_core.cu). The assembled solution, iteration counts and FITC log-determinant
must match the single-process oracle (krylov.cpp:18-106), so the decomposition
is exact up to summation order.
"""
import os
import socket

import numpy as np
import pytest
from scipy.linalg import solve_triangular

from oracle import oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, data, q):
    import torch
    import torch.distributed as dist

    from tests import shard_mirror as SM

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        P = SM.plan(data["ptr"], data["idx"], rank, world)
        r0, r1 = P["r0"], P["r1"]
        vals = data["val"][data["ptr"][r0]:data["ptr"][r1]]
        X, it, ld = SM.sharded_fitc_pcg(dist, torch, P, data["U"][:, r0:r1], vals, data["D"][r0:r1],
                                        data["B"][r0:r1], data["tol"], data["max_iter"])
        q.put((rank, r0, r1, X, it, ld, len(P["halo"]), [p[0] for p in P["peers"]]))
    finally:
        dist.destroy_process_group()


def _problem(n=900, m=24, gamma=0.07, seed=4, k=5):
    locs = O.uniform_locations(n, 2, seed)
    ind = O.select_kmeanspp(locs, m, seed + 1)
    kw = dict(nu=1.5, taper_family=1, gamma=gamma, sigma2=0.2, sigma1_2=1.0, rho=0.15)
    om = O.Model(locs, ind, **kw)
    # a locality-preserving order (any permutation is valid; blocks of it are the shards)
    perm = np.lexsort((locs[:, 1], np.floor(locs[:, 0] * 8)))
    iperm = np.empty(n, np.int64)
    iperm[perm] = np.arange(n)
    optr, oidx, oval = om.csr(1)
    ptr = np.zeros(n + 1, np.int64)
    rows_i, rows_v = [], []
    for s_, o in enumerate(perm):
        c = iperm[oidx[optr[o]:optr[o + 1]]]
        v = oval[optr[o]:optr[o + 1]]
        order = np.argsort(c)
        rows_i.append(c[order])
        rows_v.append(v[order])
        ptr[s_ + 1] = ptr[s_] + len(c)
    idx, val = np.concatenate(rows_i), np.concatenate(rows_v)
    Lm = om.dense(7)
    U = solve_triangular(np.tril(Lm), om.dense(1), lower=True)
    assert np.allclose((U ** 2).sum(0), om.dense(6), rtol=1e-10, atol=1e-12)
    D = np.array([val[ptr[i]:ptr[i + 1]][idx[ptr[i]:ptr[i + 1]] == i][0] for i in range(n)])
    B = np.random.default_rng(seed).standard_normal((n, k))
    return om, perm, dict(ptr=ptr, idx=idx, val=val, U=U[:, perm], D=D, B=B[perm], tol=1e-8, max_iter=500), B


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fitc_pcg_matches_oracle(world):
    import torch.multiprocessing as mp

    om, perm, data, B = _problem()
    ref = O.pcg_solve_multi(om, O.Precond(om, "fitc"), B, tol=1e-8, max_iter=500)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    env_before = os.environ.get("MASTER_ADDR")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    procs = [ctx.Process(target=_rank, args=(r, world, port, data, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if env_before is None:
        os.environ.pop("MASTER_ADDR", None)
    outs.sort()
    Xs = np.zeros_like(B)
    covered = 0
    for rank, r0, r1, X, it, ld, nhalo, peers in outs:
        Xs[perm[r0:r1]] = X
        covered += r1 - r0
        assert nhalo > 0 and len(peers) >= 1
        assert np.array_equal(it, ref["iterations"])
        assert ld == pytest.approx(O.Precond(om, "fitc").logdet(), rel=1e-12)
    assert covered == B.shape[0]
    assert np.abs(Xs - ref["X"]).max() <= 1e-8 * np.abs(ref["X"]).max()


def test_halo_plan_is_consistent():
    """Every received halo segment is exactly what the owning peer sends, in order."""
    from tests import shard_mirror as SM

    _, _, data, _ = _problem(n=700, gamma=0.09)
    world = 4
    plans = [SM.plan(data["ptr"], data["idx"], r, world) for r in range(world)]
    for r, P in enumerate(plans):
        for q, send, ra, rb in P["peers"]:
            # what q sends to r == the part of r's halo owned by q
            Pq = plans[q]
            sent = [s for (qq, s, _, _) in Pq["peers"] if qq == r]
            recv = P["halo"][ra:rb]
            got = (sent[0] + Pq["r0"]) if sent else np.zeros(0, np.int64)
            assert np.array_equal(got, recv)
            assert np.all((recv >= Pq["r0"]) & (recv < Pq["r1"]))
        # local columns index [local | halo]
        assert P["lcol"].max() < P["nl"] + len(P["halo"])
