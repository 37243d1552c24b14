#!/usr/bin/env python
"""Benchmark of the B200 FSA iterative core (BASELINE.json metric).

One step = one FSA log-likelihood + gradient evaluation as the reference's fit objective
performs it (estimation.cpp:255-284): FsaModel::assemble at the current parameters,
FitcPrecond::from_fsa, iterative_nll_grad (probes, lockstep FITC-PCG over [Z | y], SLQ
log-determinant, STE gradient traces with the optimal control variate). The taper pattern
(parameter independent) is built once per run.

value  = PCG RHS-iterations per second over the whole evaluation (inputs resident in HBM:
         response and probe draws cached on the device, as in a fit loop)
e2e    = the same metric through the reference-facing C-ABI calls with host buffers
         (fsa_model_assemble + fsa_make_preconditioner + fsa_iterative_nll_grad),
         host<->device copies inside the timed region.
`--impl reference` times the CPU oracle port of the reference path (oracle/) on the host
cores: a bounded FITC-PCG sample of the same workload, inputs made by the oracle's own
generators (the product library is never loaded on that arm).

Configs (tests/golden/configs.py, BASELINE.json): 2 (default, the metric's 1-GPU config),
1, 4 (n = 1e6, the north-star size; --mode strong shards it), 5 (clustered stress; adds
the cmd_bench_precond arm: FITC vs unpreconditioned CG on Sigma x = y), 3 (predictive
variances; metric = wall time).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from tests.golden.configs import CONFIGS, calibrate_gamma, model_kw  # noqa: E402

METRIC = "PCG RHS-iterations/s over FSA loglik+grad evaluations"


def make_inputs(cfg, fsa, ctx=None):
    """The product's host / device generators (pinned equal to the oracle's, tests/test_boundary_cpu.py)."""
    n, m = cfg["n"], cfg["m"]
    if cfg["points"] == "uniform":
        coords = fsa.uniform_locations(n, 2, 1)
        gamma = fsa.gamma_for_avg_row_nnz(n, cfg["nnz"])
    else:
        coords = fsa.blob_locations(n, 2, 50, 0.01, 1)
        gamma = calibrate_gamma(n, cfg["nnz"], lambda g: fsa.Geometry(coords, g, ctx).nnz())
    if cfg["inducing"] == "random":
        ind = fsa.select_random(coords, m, 2)
    else:  # device k-means++ (bit-identical to the oracle's host k-means++)
        ind = fsa.select_kmeanspp(coords, m, 2, device=True, ctx=ctx)
    y = fsa.simulate_rff(coords, cfg["nu"], cfg["s12"], cfg["rho"], cfg["s2"], 1024, 3)
    return coords, ind, gamma, y


def oracle_inputs(cfg):
    """The same seeded workload from the oracle's own generators (reference arm / CPU legs)."""
    from oracle import oracle as O

    n, m = cfg["n"], cfg["m"]
    if cfg["points"] == "uniform":
        coords = O.uniform_locations(n, 2, 1)
        gamma = O.gamma_for_avg_row_nnz(n, cfg["nnz"])
    else:
        coords = O.blob_locations(n, 2, 50, 0.01, 1)
        gamma = calibrate_gamma(n, cfg["nnz"], lambda g: O.taper_pattern(coords, g)[0][-1])
    ind = O.select_random(coords, m, 2) if cfg["inducing"] == "random" else O.select_kmeanspp(coords, m, 2)
    y = O.simulate_rff(coords, cfg["nu"], cfg["s12"], cfg["rho"], cfg["s2"], 1024, 3)
    nnz = int(O.taper_pattern(coords, gamma)[0][-1])
    return coords, ind, gamma, y, nnz


def config_dict(args, cfg, n, nnz, gamma, world, sharded):
    """Identical on both arms (built from the workload only)."""
    k = cfg["L"] + 1
    return {"workload": (f"config{args.config}: loglik+grad, FITC-PCG"
                         + (f", n = {n // world} x {world} GPUs" if sharded and args.mode == "weak" else "")),
            "n": n, "m": cfg["m"], "nnz": nnz, "avg_row_nnz": nnz / n, "probes": cfg["L"], "rhs": k,
            "tol": cfg["tol"], "nu": cfg["nu"], "rho": cfg["rho"], "sigma2": cfg["s2"], "sigma1_2": cfg["s12"],
            "gamma": gamma, "points": cfg["points"], "inducing": cfg["inducing"],
            "parallelism": (f"row-sharded x{world} ({args.mode}; NCCL halo exchange + allreduce)"
                            if sharded else ("replicas" if world > 1 else "single")),
            "l2": "inputs larger than L2 (U is m x n fp64 = %.0f MB)" % (8 * cfg["m"] * n / 1e6)}


def effective_cfg(args):
    cfg = dict(CONFIGS[args.config])
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and args.mode == "weak":
        cfg["n"] = cfg["n"] * world
    return cfg


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measure_fp64_peak(torch):
    """cuBLAS DGEMM throughput (FP64 peak is absent from MEASURED_PEAKS.json)."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    del a, b
    torch.cuda.empty_cache()
    return 2 * 8192 ** 3 / (ms * 1e-3) / 1e12


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def cpu_pcg_sample(cfg, coords, ind, gamma, y, sweeps=2):
    """The oracle port at the full workload: FITC setup untimed, then a bounded number of
    lockstep PCG sweeps on the [Z | y] block (the reference's per-column Woodbury GEMVs,
    krylov.cpp:83); RHS-iterations / s."""
    from oracle import oracle as O

    kw = model_kw(cfg, gamma)
    om = O.Model(coords, ind, **kw)
    P = O.Precond(om, "fitc", plain=True)
    Z = P.sample_probes(cfg["L"], 0)
    B = np.asfortranarray(np.column_stack([Z, y]))
    t0 = time.perf_counter()
    r = O.pcg_solve_multi(om, P, B, tol=cfg["tol"], max_iter=sweeps)
    dt = time.perf_counter() - t0
    its = int(np.sum(r["iterations"]))
    return its / dt, its, dt


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = effective_cfg(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    sharded = args.mode != "replicas" and (world > 1 or args.mode == "strong")
    coords, ind, gamma, y, nnz = oracle_inputs(cfg)
    if args.config == 3:
        run_reference_prediction(args, cfg, coords, ind, gamma, y, nnz)
        return
    vals = []
    for i in range(args.warmup + args.steps):
        v, its, dt = cpu_pcg_sample(cfg, coords, ind, gamma, y, sweeps=args.ref_sweeps)
        if i >= args.warmup:
            vals.append((v, its, dt))
    value = statistics.median(v for v, _, _ in vals)
    sample = (f"oracle port (oracle/fsa_oracle.cpp, C++ restatement of krylov.cpp:18-106 + "
              f"preconditioners.cpp:58-61, OpenMP over RHS columns) at n={cfg['n']}, m={cfg['m']}, "
              f"t={cfg['L'] + 1}: {args.ref_sweeps} PCG sweeps per step, FITC setup untimed")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "RHS-iterations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(dt for _, _, dt in vals), "higher_is_better": True,
            "scaling": "strong" if (sharded and args.mode == "strong") else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded; BASELINE config)",
            "config": config_dict(args, cfg, cfg["n"], nnz, gamma, world, sharded),
            "cpu_baseline": {"value": value, "unit": "RHS-iterations/s", "cores": cpu_threads(), "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "RHS-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def cpu_prediction_sample(cfg, coords, ind, gamma, plocs, cols=16, probes=32):
    """Config 3 on the oracle port, a bounded sample: make_prediction_set (timed), the deterministic
    pieces' two m-RHS solves on `cols` of their m columns (independent per-column recurrences:
    x m / cols), `probes` simulation vectors of a batch (x L / probes); the small dense remainder of the
    deterministic pieces is not counted (the estimate is conservative)."""
    from oracle import oracle as O

    kw = model_kw(cfg, gamma)
    om = O.Model(coords, ind, **kw)
    t0 = time.perf_counter()
    pr = O.PredictionSet(om, plocs)
    t_set = time.perf_counter() - t0
    t = pr.sample_timing(cols=cols, probes=probes, seed=0, tol=cfg["tol"], tol_s=cfg["tol"])
    scale = cfg["m"] / cols
    total = t_set + (t["x1"] + t["x2"]) * scale + t["batch"] * cfg["L"] / probes
    sampled = t_set + t["x1"] + t["x2"] + t["batch"]
    return total * 1e3, sampled, t


def run_reference_prediction(args, cfg, coords, ind, gamma, y, nnz):
    from oracle import oracle as O

    plocs = O.uniform_locations(cfg["np"], 2, 101)
    vals = []
    for i in range(min(args.warmup, 1) + max(1, min(args.steps, 3))):
        ms, sampled, t = cpu_prediction_sample(cfg, coords, ind, gamma, plocs)
        if i >= min(args.warmup, 1):
            vals.append(ms)
    value = statistics.median(vals)
    sample = (f"oracle port (prediction.cpp:72-172) at n = n_p = {cfg['n']}, m = {cfg['m']}: make_prediction_set + "
              f"16 of the {cfg['m']} columns of each deterministic m-RHS solve (x {cfg['m'] / 16:g}) + 32 "
              f"simulation vectors (x {cfg['L'] / 32:g}); {sampled:.1f} s of CPU work per step")
    line = {"impl": "reference", "metric": "predictive-variance wall time (make_prediction_set + predict_var_sim)",
            "value": value, "unit": "ms", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": value, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; BASELINE config 3)", "config": prediction_config(cfg, nnz, gamma),
            "cpu_baseline": {"value": value, "unit": "ms", "cores": cpu_threads(), "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def prediction_config(cfg, nnz, gamma):
    return {"workload": "config3: make_prediction_set + predict_var_sim", "n": cfg["n"], "np": cfg["np"],
            "m": cfg["m"], "nnz": nnz, "probes": cfg["L"], "tol": cfg["tol"], "gamma": gamma,
            "parallelism": "single"}


def run_prediction(args, cfg):
    """Config 3: make_prediction_set + predict_var_sim (1000 Rademacher simulation vectors,
    FITC-PCG with m RHS + Jacobi-PCG on Sigma_s), device-timed per evaluation."""
    import torch

    from paper_2405_14492_b200 import fsa

    torch.cuda.set_device(0)
    ctx = fsa.Context(0)
    coords, ind, gamma, y = make_inputs(cfg, fsa, ctx)
    plocs = fsa.uniform_locations(cfg["np"], 2, 101)
    kw = model_kw(cfg, gamma)
    geo = fsa.Geometry(coords, gamma, ctx)
    nnz = geo.nnz()
    md = fsa.FsaModel.assemble(None, ind, geometry=geo, **kw)
    stream = torch.cuda.ExternalStream(ctx.stream())

    def step():
        pr = fsa.make_prediction_set(md, plocs)
        return pr.predict_var_sim(num_probes=cfg["L"], seed=0, tol=cfg["tol"], tol_s=cfg["tol"])

    for _ in range(args.warmup):
        step()
    ctx.set_profiling(True)
    ctx.reset_timers()
    sampler = ClockSampler(0)
    sampler.start()
    ctx.synchronize()
    l0 = fsa.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res = [step() for _ in range(args.steps)]
    e1.record(stream)
    ctx.synchronize()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    timers = ctx.timers()
    ctx.set_profiling(False)
    last = res[-1]
    # roofline of the simulation solves: Jacobi-PCG on Sigma_s over 256-column batches
    # (per sweep 12 nnz + 16 n t bytes for the SpMM with h.v, the vector update
    # X, R, H, V + r.z: 6 x 8 n t) -- the "spmm" group of these solves
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6550.0)
    sp = timers.get("spmm")
    roofline = None
    if sp and sp["count"]:
        avg = sp["ms"] / sp["count"]
        units = sp["units"] / sp["count"]
        ach = units / (avg * 1e-3) / 1e9
        roofline = {"kernel": "k_spmm_v3 (Jacobi-PCG SpMM of the simulation / Sigma_s solves, 64-column tiles)",
                    "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                    "traffic": None, "avg_launch_ms": avg, "launches": sp["count"],
                    "share_of_step": sp["ms"] / (ms * args.steps), "units_per_launch": units,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"}
    # e2e: host coordinates in, variances out, through the C ABI (model already assembled)
    e2e_ms = []
    for i in range(1 + args.e2e_steps):
        ctx.synchronize()
        t0 = time.perf_counter()
        pr = fsa.make_prediction_set(md, plocs)
        r = pr.predict_var_sim(num_probes=cfg["L"], seed=0, tol=cfg["tol"], tol_s=cfg["tol"])
        ctx.synchronize()
        if i > 0:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        del pr, r
    cpu = None
    if not args.no_cpu_baseline:
        try:
            from oracle import oracle as O  # noqa: F401

            cms, sampled, t = cpu_prediction_sample(cfg, coords, ind, gamma, plocs)
            cpu = {"value": cms, "unit": "ms", "cores": cpu_threads(), "kind": "port",
                   "sample": f"oracle port: make_prediction_set + 16 of {cfg['m']} columns of each deterministic "
                             f"m-RHS solve (x {cfg['m'] / 16:g}: X1 {t['x1']:.1f} s, X2 {t['x2']:.1f} s) + 32 "
                             f"simulation vectors ({t['batch']:.1f} s, x {cfg['L'] / 32:g}); {sampled:.1f} s sampled"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "ms", "cores": cpu_threads(), "kind": "port", "sample": f"failed: {exc}"}
    e2e_v = statistics.median(e2e_ms) if e2e_ms else None
    line = {"metric": "predictive-variance wall time (make_prediction_set + predict_var_sim)", "value": ms,
            "unit": "ms", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; BASELINE config 3)", "config": prediction_config(cfg, nnz, gamma),
            "det_ms": last["det_ms"], "sim_ms": last["sim_ms"], "cg_iterations": last["cg_iterations"],
            "clamped": last["clamped"], "var_mean": float(np.mean(last["var"])),
            "se_mean": float(np.mean(last["se"])), "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": e2e_v, "unit": "ms", "h2d_bytes_per_step": 8 * 2 * cfg["np"],
                    "d2h_bytes_per_step": 8 * 2 * cfg["np"]},
            "gpu_launches": fsa.launch_count() - l0, "clocks": clocks,
            "timers_ms": {k: round(v["ms"] / args.steps, 3) for k, v in timers.items()}}
    print(json.dumps(line))


def time_steps(step, n, ctx, stream, torch, barrier, max_over_ranks):
    """W warm-up steps are the caller's; n timed steps between barriers + device syncs,
    CUDA events on the library stream, max over ranks."""
    barrier()
    ctx.synchronize()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    results = [step() for _ in range(n)]
    e1.record(stream)
    ctx.synchronize()
    torch.cuda.synchronize()
    barrier()
    return results, max_over_ranks(e0.elapsed_time(e1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # defaults: 20 timed steps after 5 warm-up steps at configs 2 / 5 (a 40 ms step: one slow outlier in
    # five moved the mean by 4 %), 3 after 3 at the second-scale configs 3 / 4
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--ref-sweeps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dmma-arm", action="store_true", help="skip the fp64-DMMA comparison run")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--mode", default="weak", choices=["weak", "strong", "replicas"],
                    help="N>1: weak = n scales with N (row-sharded, n/N rows per GPU fixed); strong = the "
                         "config's n row-sharded over N GPUs; replicas = N independent copies")
    ap.add_argument("--no-strong-sub", action="store_true", help="N>1: skip the config-4 strong-scaling record")
    args = ap.parse_args()
    fast = args.config in (2, 5) and args.impl != "reference"
    if args.steps is None:
        args.steps = 20 if fast else 3
    if args.warmup is None:
        args.warmup = 5 if fast else 3
    if args.e2e_steps is None:
        args.e2e_steps = 10 if fast else 3
    if args.impl == "reference":
        run_reference(args)
        return
    cfg = effective_cfg(args)
    if args.config == 3:
        run_prediction(args, cfg)
        return

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)

    from paper_2405_14492_b200 import fsa

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # rows of one problem split over the ranks: NCCL halo exchange + allreduce (--mode strong at
    # N = 1 runs the same NCCL-context code path with one rank)
    sharded = args.mode != "replicas" and (world > 1 or args.mode == "strong")

    def make_ctx():
        if sharded:
            uid = [fsa.nccl_unique_id() if rank == 0 else None]
            if dist is not None:
                dist.broadcast_object_list(uid, src=0)
            return fsa.Context.nccl(local, rank, world, uid[0])
        return fsa.Context(local)

    ctx = make_ctx()
    coords, ind, gamma, y = make_inputs(cfg, fsa, ctx)
    fp64_peak = measure_fp64_peak(torch)
    kw = model_kw(cfg, gamma)
    L, tol = cfg["L"], cfg["tol"]
    stream = torch.cuda.ExternalStream(ctx.stream())

    # ---- device-resident fit-loop step (value) ---------------------------------------
    geo = fsa.Geometry(coords, gamma, ctx)
    geo.set_response(y)
    geo.cache_probes(True)
    nnz = geo.nnz()

    def step():
        md = fsa.FsaModel.assemble(None, ind, geometry=geo, **kw)
        P = fsa.make_preconditioner(md, "fitc")
        r = fsa.iterative_nll_grad(md, P, None, num_probes=L, seed=0, tol=tol)
        del P, md
        return r

    for _ in range(args.warmup):
        step()
    # timed pass (the headline): library timers off, so the PCG sweeps run as replayed CUDA graphs
    sampler = ClockSampler(local)
    sampler.start()
    l0 = fsa.launch_count()
    results, ms = time_steps(step, args.steps, ctx, stream, torch, barrier, max_over_ranks)
    launches = fsa.launch_count() - l0
    clocks = sampler.stop()
    # second timed pass with the per-kernel-group CUDA-event timers (eager launches): the roofline
    # entries' average launch durations and shares come from here
    ctx.set_profiling(True)
    ctx.reset_timers()
    presults, pms = time_steps(step, args.steps, ctx, stream, torch, barrier, max_over_ranks)
    timers = ctx.timers()
    ctx.set_profiling(False)
    copies = 1 if sharded else world  # replicas each solve the whole problem
    rhs_its = sum(r["rhs_iterations"] for r in results) * copies
    value = rhs_its / (ms * 1e-3)
    pcg_ms = statistics.median(r["pcg_ms"] for r in results)
    pcg_rate = results[-1]["rhs_iterations"] / (pcg_ms * 1e-3)

    # ---- roofline ----------------------------------------------------------------------
    # every kernel group of the PCG sweep against its bound, with its ALGORITHMIC bytes per launch
    # at the unpadded sizes: SpMM + direction update 12 nnz + 48 n t,
    # projection 8 m n + 8 n t, expansion + Woodbury epilogue 8 m n + 24 n t; time = the group's
    # average CUDA-event launch time inside the timed region. Headline = largest share of the step.
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6550.0)
    step_ms = ms / args.steps
    n_, m_ = cfg["n"] // (world if sharded else 1), cfg["m"]
    t_ = L + 1
    tp_ = 8 * math.ceil(t_ / 8)
    traffic = {}
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic_config%d.json" % args.config)))
    except Exception:
        pass

    def entry(name, kernel, units_per_launch):
        t = timers.get(name)
        if not t or not t["count"]:
            return None
        avg = t["ms"] / t["count"]
        ach = units_per_launch / (avg * 1e-3) / 1e9
        return {"kernel": kernel, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": traffic.get(kernel.split()[0]), "avg_launch_ms": avg, "launches": t["count"],
                "share_of_step": t["ms"] / pms, "units_per_launch": units_per_launch}

    int8 = tp_ <= 64
    pair = 64 < tp_ <= 96  # (ozaki_*_pair: one launch, CTA pairs stream the same U planes)
    nnz_loc = nnz / (world if sharded else 1)
    b_spmm = 12.0 * nnz_loc + 48.0 * n_ * t_
    b_proj = 8.0 * m_ * n_ + 8.0 * n_ * t_
    b_exp = 8.0 * m_ * n_ + 24.0 * n_ * t_
    b_xr = 48.0 * n_ * t_
    kernels = [
        entry("spmm", "k_spmm_v3 (32-row groups, DMMA.8x8x4 fp64 block product + direction update)", b_spmm),
        entry("lowrank_expand", "k_oz_expand (tcgen05 kind::i8 Ozaki, + k_oz_planes_w)" if int8 else
              ("k_oz_expand<paired> (two %d-column INT8 tiles on CTA pairs, + planes)" % (tp_ // 2) if pair else
               "k_oz_expand 64-column INT8 tiles + DMMA remainder (+ planes)"), b_exp),
        entry("lowrank_project", "k_oz_gemm (tcgen05 kind::i8 Ozaki, + k_oz_planes_y, k_oz_reduce)" if int8 else
              ("k_oz_gemm<paired> (two %d-column INT8 tiles on CTA pairs, + planes, reduce)" % (tp_ // 2) if pair
               else "k_oz_gemm 64-column INT8 tiles + DMMA remainder (+ planes, reduce)"), b_proj),
    ]
    kernels = [k for k in kernels if k]
    dom = max(kernels, key=lambda k: k["share_of_step"])
    roofline = dict(dom)
    roofline["peak_source"] = "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"
    roofline["all"] = kernels
    roofline["fp64_dgemm_tflops_measured"] = fp64_peak
    sweeps = sum(r["sweeps"] for r in presults)
    sweep_groups = ("spmm", "lowrank_project", "lowrank_expand", "core_solve", "cg_blas1", "allreduce",
                    "halo_exchange")
    t_sweep = sum(timers[k]["ms"] for k in sweep_groups if k in timers) / max(sweeps, 1)
    # this build's own per-sweep HBM floor: every byte its sweep must move once
    floor_bytes = b_spmm + b_xr + b_proj + b_exp
    t_floor = floor_bytes / (hbm * 1e9) * 1e3
    # SURVEY §8d unit: one PCG sweep of the REFERENCE operation sequence (krylov.cpp:56-93,
    # fsa.cpp:65-68, preconditioners.cpp:58-61: SpMM + four m x n passes + vector streams) at the
    # measured HBM bandwidth and cuBLAS DGEMM rate
    phases = {
        "spmm": (12.0 * nnz_loc + 4.0 * (n_ + 1), 2.0 * nnz_loc * t_),
        "lowrank": (4 * 8.0 * m_ * n_, 8.0 * m_ * n_ * t_ + 4.0 * m_ ** 2 * t_),
        "vectors": (80.0 * n_ * t_, 12.0 * n_ * t_),
    }
    t_roof = sum(max(b / (hbm * 1e9), f / (fp64_peak * 1e12)) for b, f in phases.values()) * 1e3
    roofline["profiled_pass_ms_per_step"] = pms / args.steps
    roofline["sweep"] = {"unit": "one PCG sweep", "t_measured_ms": t_sweep,
                         "own_floor": {"bytes": floor_bytes, "t_floor_ms": t_floor,
                                       "frac": t_floor / t_sweep if t_sweep else None,
                                       "note": "this build's two-pass sweep: SpMM + update + projection + "
                                               "expansion algorithmic bytes at the measured HBM bandwidth"},
                         "reference_sequence": {"t_roof_ms": t_roof, "frac": t_roof / t_sweep if t_sweep else None,
                                                "note": "SURVEY 8d: the reference's four-pass sequence at HBM "
                                                        "bandwidth / cuBLAS DGEMM rate; can exceed 1"}}

    # ---- the same evaluation with the dense passes on fp64 DMMA (no INT8 emulation) ----------
    dmma = None
    if not args.no_dmma_arm and not sharded:
        ctx.set_gemm_mode("dmma")
        for _ in range(2):
            step()
        dres, dms = time_steps(step, args.steps, ctx, stream, torch, barrier, max_over_ranks)
        ctx.set_gemm_mode("auto")
        drhs = sum(r["rhs_iterations"] for r in dres) * copies
        dmma = {"value": drhs / (dms * 1e-3), "ms_per_step": dms / args.steps, "nll": dres[-1]["nll"],
                "grad": list(dres[-1]["grad"]), "cg_iterations": dres[-1]["cg_iterations"],
                "note": "same step with FSA dense passes on fp64 DMMA (fsa_ctx_set_gemm_mode 1)"}

    # ---- config 5: cmd_bench_precond (tools/commands.cpp:462-510), row n1 ----------------------
    bench_precond = None
    if args.config == 5:
        md = fsa.FsaModel.assemble(None, ind, geometry=geo, **kw)
        bench_precond = {}
        for name in ("fitc", "diagonal", "none"):
            P = fsa.make_preconditioner(md, name)
            for cap in (1000, 50000):
                ctx.synchronize()
                t0 = time.perf_counter()
                sol = fsa.pcg_solve_multi(md, P, y.reshape(-1, 1), tol=tol, max_iter=cap)
                ctx.synchronize()
                dt = (time.perf_counter() - t0) * 1e3
                lc = ctx.last_cg()
                bench_precond[f"{name}" + ("" if cap == 1000 else "_uncapped")] = {
                    "iterations": int(sol["iterations"][0]), "converged": bool(sol["converged"][0]),
                    "residual": float(lc["rnorm"][0][-1]) if len(lc["rnorm"][0]) else None, "wall_ms": dt,
                    "max_iter": cap}
                if sol["converged"][0]:
                    break
            del P
        del md

    # ---- end to end through the reference-facing API with host buffers (e2e) -------
    del geo
    e2e_ms = []
    n, m = cfg["n"], cfg["m"]
    for i in range(1 + args.e2e_steps if args.e2e_steps > 0 else 0):
        barrier()
        ctx.synchronize()
        t0 = time.perf_counter()
        md = fsa.FsaModel.assemble(coords, ind, ctx=ctx, **kw)
        P = fsa.make_preconditioner(md, "fitc")
        r = fsa.iterative_nll_grad(md, P, y, num_probes=L, seed=0, tol=tol)
        ctx.synchronize()
        dt = time.perf_counter() - t0
        del P, md
        if i > 0:
            e2e_ms.append(max_over_ranks(dt * 1e3))
    e2e_step_ms = statistics.median(e2e_ms) if e2e_ms else float("nan")
    e2e_value = results[-1]["rhs_iterations"] * copies / (e2e_step_ms * 1e-3) if e2e_ms else None
    k = L + 1
    mp_ = 128 * math.ceil(m / 128)
    # per rank: coordinates (n x 2), inducing points (m x 2), y (n) -- the FITC probe draws are
    # generated on the device (k_probe_gaussian, round 2; FSA_HOST_PROBES=1 uploads the host draws:
    # + m_pad x t_pad + n_rank x L doubles); back: nll, grad, logdet, beta and the Lanczos
    # coefficients of its columns
    n_rank = n // world if sharded else n
    host_probes = os.environ.get("FSA_HOST_PROBES") is not None
    h2d = 8 * world * (n * 2 + m * 2 + n + ((mp_ * tp_ + n_rank * L) if host_probes else 0))
    d2h = 8 * world * (5 + 3 * k * results[-1]["sweeps"] + 2 * k)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, its, dt = cpu_pcg_sample(cfg, coords, ind, gamma, y, sweeps=args.ref_sweeps)
            cpu = {"value": v, "unit": "RHS-iterations/s", "cores": cpu_threads(), "kind": "port",
                   "sample": f"oracle port, FITC setup untimed, {args.ref_sweeps} lockstep PCG sweeps on the "
                             f"full n={n}, t={k} block ({its} RHS-iterations in {dt:.2f} s)"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "RHS-iterations/s", "cores": cpu_threads(), "kind": "port",
                   "sample": f"failed: {exc}"}

    # ---- N > 1: the north-star strong-scaling case (config 4 sharded over the same ranks) -------
    strong = None
    if world > 1 and not args.no_strong_sub and args.config != 4:
        strong = strong_record(args, fsa, torch, world, rank, local, dist, barrier, max_over_ranks)

    if rank == 0:
        last = results[-1]
        line = {
            "metric": METRIC, "value": value, "unit": "RHS-iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong" if (sharded and args.mode == "strong") else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded; BASELINE config)",
            "config": config_dict(args, cfg, n, nnz, gamma, world, sharded),
            "loglik_grad_ms": step_ms, "pcg_ms": pcg_ms, "pcg_only_rhs_iter_per_s": pcg_rate,
            "cg_iterations": last["cg_iterations"], "sweeps": last["sweeps"], "nll": last["nll"],
            "grad": list(last["grad"]), "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "RHS-iterations/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_step_ms},
            "gpu_launches": launches, "clocks": clocks, "dmma_mode": dmma,
            "timers_ms": {k2: round(v["ms"] / args.steps, 3) for k2, v in timers.items()},
        }
        if bench_precond is not None:
            line["bench_precond"] = bench_precond
        if strong is not None:
            line["config4_strong"] = strong
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def strong_record(args, fsa, torch, world, rank, local, dist, barrier, max_over_ranks):
    """Config 4 (n = 1e6, m = 1000, t = 65) row-sharded over the job's ranks (strong scaling):
    device-timed loglik+grad evaluations, max over ranks."""
    cfg = dict(CONFIGS[4])
    uid = [fsa.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ctx = fsa.Context.nccl(local, rank, world, uid[0])
    coords, ind, gamma, y = make_inputs(cfg, fsa, ctx)
    kw = model_kw(cfg, gamma)
    geo = fsa.Geometry(coords, gamma, ctx)
    geo.set_response(y)
    geo.cache_probes(True)
    stream = torch.cuda.ExternalStream(ctx.stream())

    def step():
        md = fsa.FsaModel.assemble(None, ind, geometry=geo, **kw)
        P = fsa.make_preconditioner(md, "fitc")
        r = fsa.iterative_nll_grad(md, P, None, num_probes=cfg["L"], seed=0, tol=cfg["tol"])
        del P, md
        return r

    step()
    steps = max(2, min(args.steps, 3))
    res, ms = time_steps(step, steps, ctx, stream, torch, barrier, max_over_ranks)
    rhs = sum(r["rhs_iterations"] for r in res)
    return {"workload": "config4: n = 1e6, m = 1000, t = 65, row-sharded (strong)", "n_gpus": world,
            "value": rhs / (ms * 1e-3), "unit": "RHS-iterations/s", "ms_per_step": ms / steps, "steps": steps,
            "sweeps": res[-1]["sweeps"], "nll": res[-1]["nll"]}


if __name__ == "__main__":
    main()
