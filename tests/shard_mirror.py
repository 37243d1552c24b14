"""NumPy + torch.distributed restatement of the row-sharded fit path.

Test infrastructure: it restates, rank by rank, what the CUDA library does on a
row-sharded context (paper_2405_14492_b200/csrc/shard.cu ``shard_pattern``,
comm.cu, fsa_core.cu ``pcg_solve_multi`` / ``FitcPrecond``) so that the
decomposition itself -- block split, halo plan, neighbour exchange, the m x t
allreduce of the projections and the per-column dot allreduce -- runs under a
real multi-process ``gloo`` group on CPU and can be checked against the
single-process oracle (krylov.cpp:18-106, preconditioners.cpp:16-115).
"""
from __future__ import annotations

import numpy as np


def block(n, q, world):  # shard.cu: rank q owns [n q / W, n (q + 1) / W)
    return n * q // world, n * (q + 1) // world


def plan(ptr, idx, rank, world):
    """Halo plan of ``rank`` for a symmetric CSR pattern in sorted order."""
    n = len(ptr) - 1
    r0, r1 = block(n, rank, world)
    nl = r1 - r0
    cols = idx[ptr[r0]:ptr[r1]]
    halo = np.unique(cols[(cols < r0) | (cols >= r1)])
    ext = np.where((cols >= r0) & (cols < r1), cols - r0, nl + np.searchsorted(halo, cols))
    lptr = ptr[r0:r1 + 1] - ptr[r0]
    peers = []
    for q in range(world):
        if q == rank:
            continue
        q0, q1 = block(n, q, world)
        qc = idx[ptr[q0]:ptr[q1]]
        send = np.unique(qc[(qc >= r0) & (qc < r1)]) - r0  # owned rows q's rows reference
        ra, rb = np.searchsorted(halo, q0), np.searchsorted(halo, q1)  # q's segment of the halo
        if len(send) or rb > ra:
            peers.append((q, send, ra, rb))
    return dict(r0=r0, r1=r1, nl=nl, halo=halo, lptr=lptr, lcol=ext, peers=peers)


def halo_exchange(dist, torch, P, Hloc):
    """[local | halo] rows of an n_loc x k block (neighbour send/recv, no collective)."""
    nl, k = Hloc.shape
    Hext = np.zeros((nl + len(P["halo"]), k))
    Hext[:nl] = Hloc
    reqs, bufs = [], []
    for q, send, ra, rb in P["peers"]:
        if len(send):
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(Hloc[send])), q))
        if rb > ra:
            buf = torch.zeros((rb - ra, k), dtype=torch.float64)
            reqs.append(dist.irecv(buf, q))
            bufs.append((ra, rb, buf))
    for r in reqs:
        r.wait()
    for ra, rb, buf in bufs:
        Hext[nl + ra:nl + rb] = buf.numpy()
    return Hext


def allreduce(dist, torch, a):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).copy())
    dist.all_reduce(t)
    return t.numpy()


def spmm(P, vals, Hext):
    """Local rows of Sigma_s H over the extended (local | halo) block."""
    nl = P["nl"]
    out = np.zeros((nl, Hext.shape[1]))
    lptr, lcol = P["lptr"], P["lcol"]
    for i in range(nl):
        a, b = lptr[i], lptr[i + 1]
        out[i] = vals[a:b] @ Hext[lcol[a:b]]
    return out


def sharded_fitc_pcg(dist, torch, P, U_loc, vals, D_loc, B_loc, tol, max_iter):
    """Lockstep FITC-preconditioned PCG of one rank (same control flow as krylov.cpp:18-106)."""
    m = U_loc.shape[0]
    k = B_loc.shape[1]
    Dinv = 1.0 / D_loc
    Q = np.eye(m) + allreduce(dist, torch, (U_loc * Dinv) @ U_loc.T)
    logdet = np.linalg.slogdet(Q)[1] + allreduce(dist, torch, np.array([np.log(D_loc).sum()]))[0]

    def psolve(R):
        S = allreduce(dist, torch, U_loc @ (Dinv[:, None] * R))
        return Dinv[:, None] * (R - U_loc.T @ np.linalg.solve(Q, S))

    def matvec(H):
        UH = allreduce(dist, torch, U_loc @ H)
        return U_loc.T @ UH + spmm(P, vals, halo_exchange(dist, torch, P, H))

    def coldots(A, Bm):
        return allreduce(dist, torch, np.einsum("ij,ij->j", A, Bm))

    X = np.zeros_like(B_loc)
    R = B_loc.copy()
    rr = coldots(R, R)
    active = np.sqrt(rr) >= tol
    iters = np.zeros(k, int)
    Z = psolve(R)
    rz = coldots(R, Z)
    H = np.where(active[None, :], Z, 0.0)
    for it in range(max_iter):
        if not active.any():
            break
        V = matvec(H)  # every rank runs every sweep (collectives stay matched)
        hv = coldots(H, V)
        alpha = np.where(active, rz / np.where(active, hv, 1.0), 0.0)
        X += alpha[None, :] * H
        R -= alpha[None, :] * V
        iters[active] = it + 1
        rr = coldots(R, R)
        done = active & (np.sqrt(rr) < tol)
        active = active & ~done
        Z = psolve(R)
        rzn = coldots(R, Z)
        beta = np.where(active, rzn / np.where(active, rz, 1.0), 0.0)
        H = np.where(active[None, :], Z + beta[None, :] * H, H)
        rz = np.where(active, rzn, rz)
    return X, iters, logdet
