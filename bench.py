#!/usr/bin/env python
"""Benchmark of the B200 FSA iterative core (BASELINE.json metric).

One step = one FSA log-likelihood + gradient evaluation as the reference's fit
objective performs it (estimation.cpp:255-284): FsaModel::assemble at the current
parameters, FitcPrecond::from_fsa, iterative_nll_grad (probes, lockstep FITC-PCG
over [Z | y], SLQ log-determinant, STE gradient traces with the optimal control
variate). The taper pattern (parameter independent) is built once per run.

value  = PCG RHS-iterations per second over the whole evaluation (inputs resident
         in HBM: response and probe draws cached on the device, as in a fit loop)
e2e    = the same metric through the reference-facing C-ABI calls with host buffers
         (fsa_model_assemble + fsa_make_preconditioner + fsa_iterative_nll_grad),
         host<->device copies inside the timed region.
`--impl reference` times the CPU oracle port of the reference path (oracle/) on
the host cores: a bounded FITC-PCG sample of the same workload.
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

CONFIGS = {
    1: dict(n=10_000, m=200, inducing="random", nu=0.5, s12=1.0, rho=0.1, s2=0.1, nnz=30, L=50, tol=1e-3,
            points="uniform"),
    2: dict(n=100_000, m=500, inducing="kmeans", nu=1.5, s12=1.0, rho=0.05, s2=0.05, nnz=80, L=50, tol=1e-3,
            points="uniform"),
    3: dict(n=100_000, m=500, inducing="kmeans", nu=1.5, s12=1.0, rho=0.05, s2=0.05, nnz=80, L=1000, tol=1e-3,
            points="uniform", np=100_000),
    4: dict(n=1_000_000, m=1000, inducing="kmeans", nu=1.5, s12=1.0, rho=0.03, s2=0.05, nnz=80, L=64, tol=1e-3,
            points="uniform"),
    5: dict(n=200_000, m=1000, inducing="kmeans", nu=2.5, s12=1.0, rho=0.3, s2=1e-3, nnz=120, L=50, tol=1e-4,
            points="blobs"),
}
METRIC = "PCG RHS-iterations/s over FSA loglik+grad evaluations"


def make_inputs(cfg, fsa, device_kmeans=True):
    n, m = cfg["n"], cfg["m"]
    if cfg["points"] == "uniform":
        coords = fsa.uniform_locations(n, 2, 1)
        gamma = fsa.gamma_for_avg_row_nnz(n, cfg["nnz"])
    else:
        coords = fsa.blob_locations(n, 2, 50, 0.01, 1)
        gamma = None
    if cfg["inducing"] == "random":
        ind = fsa.select_random(coords, m, 2)
    else:
        # device k-means++ (the same inducing set as the host restatement's, which the CPU arm uses)
        ind = fsa.select_kmeanspp(coords, m, 2, device=device_kmeans)
    y = fsa.simulate_rff(coords, cfg["nu"], cfg["s12"], cfg["rho"], cfg["s2"], 1024, 3)
    return coords, ind, gamma, y


def calibrate_gamma(coords, target, fsa, ctx):
    """bisection on the measured nnz/row (clustered points)."""
    n = coords.shape[0]
    lo, hi = 1e-5, 0.2
    for _ in range(30):
        mid = math.sqrt(lo * hi)
        g = fsa.Geometry(coords, mid, ctx)
        avg = g.nnz() / n
        del g
        if avg < target:
            lo = mid
        else:
            hi = mid
        if abs(avg - target) / target < 0.02:
            return mid
    return math.sqrt(lo * hi)


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


def cpu_pcg_sample(cfg, coords, ind, gamma, sweeps=2):
    """The oracle port at the full workload: FITC setup untimed, then a bounded
    number of lockstep PCG sweeps on the [Z | y] block; RHS-iterations / s."""
    from oracle import oracle as O

    kw = dict(nu=cfg["nu"], taper_family=1, gamma=gamma, sigma2=cfg["s2"], sigma1_2=cfg["s12"], rho=cfg["rho"])
    om = O.Model(coords, ind, **kw)
    P = O.Precond(om, "fitc", plain=True)
    Z = P.sample_probes(cfg["L"], 0)
    y = np.random.default_rng(0).standard_normal(cfg["n"])
    B = np.asfortranarray(np.column_stack([Z, y]))
    t0 = time.perf_counter()
    r = O.pcg_solve_multi(om, P, B, tol=cfg["tol"], max_iter=sweeps)
    dt = time.perf_counter() - t0
    its = int(np.sum(r["iterations"]))
    return its / dt, its, dt


def last_sweeps(results):
    return int(results[-1]["sweeps"]) if results else 0


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2405_14492_b200 import fsa

    coords, ind, gamma, y = make_inputs(cfg, fsa, device_kmeans=False)  # host input generators only
    if gamma is None:
        gamma = fsa.gamma_for_avg_row_nnz(cfg["n"], cfg["nnz"])
    vals = []
    for i in range(args.warmup + args.steps):
        v, its, dt = cpu_pcg_sample(cfg, coords, ind, gamma, sweeps=args.ref_sweeps)
        if i >= args.warmup:
            vals.append((v, its, dt))
    value = statistics.median(v for v, _, _ in vals)
    cores = os.cpu_count()
    sample = (f"oracle port (oracle/fsa_oracle.cpp, C++ restatement of krylov.cpp:18-106 + "
              f"preconditioners.cpp:58-61, OpenMP over RHS columns) at n={cfg['n']}, m={cfg['m']}, "
              f"t={cfg['L'] + 1}: {args.ref_sweeps} PCG sweeps per step, FITC setup untimed")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "RHS-iterations/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(dt for _, _, dt in vals), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": {"workload": f"config{args.config}", **{k: cfg[k] for k in ("n", "m", "nnz", "L", "tol")}},
            "cpu_baseline": {"value": value, "unit": "RHS-iterations/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "RHS-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_prediction(args, cfg):
    """Config 3: make_prediction_set + predict_var_sim (1000 Rademacher simulation vectors,
    FITC-PCG with m RHS + Jacobi-PCG on Sigma_s), device-timed per evaluation."""
    import torch

    from paper_2405_14492_b200 import fsa

    torch.cuda.set_device(0)
    ctx = fsa.Context(0)
    coords, ind, gamma, y = make_inputs(cfg, fsa)
    plocs = fsa.uniform_locations(cfg["np"], 2, 101)
    kw = dict(nu=cfg["nu"], taper_family=1, gamma=gamma, sigma2=cfg["s2"], sigma1_2=cfg["s12"], rho=cfg["rho"])
    geo = fsa.Geometry(coords, gamma, ctx)
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
    last = res[-1]
    line = {"metric": "predictive-variance wall time (make_prediction_set + predict_var_sim)", "value": ms,
            "unit": "ms", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; BASELINE config 3)",
            "config": {"workload": "config3: predict_var_sim", "n": cfg["n"], "np": cfg["np"], "m": cfg["m"],
                       "probes": cfg["L"], "tol": cfg["tol"], "gamma": gamma},
            "det_ms": last["det_ms"], "sim_ms": last["sim_ms"], "cg_iterations": last["cg_iterations"],
            "clamped": last["clamped"], "var_mean": float(np.mean(last["var"])),
            "se_mean": float(np.mean(last["se"])), "gpu_launches": fsa.launch_count() - l0, "clocks": clocks,
            "cpu_baseline": None,
            "timers_ms": {k: round(v["ms"] / args.steps, 3) for k, v in timers.items()}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--ref-sweeps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--mode", default="weak", choices=["weak", "strong", "replicas"],
                    help="N>1: weak = n scales with N (row-sharded, n/N rows per GPU fixed); strong = the "
                         "config's n row-sharded over N GPUs; replicas = N independent copies")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env > 1 and args.mode == "weak":
        cfg["n"] = cfg["n"] * world_env
    if args.impl == "reference":
        run_reference(args, cfg)
        return
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
    if sharded:
        uid = [fsa.nccl_unique_id() if rank == 0 else None]
        if dist is not None:
            dist.broadcast_object_list(uid, src=0)
        ctx = fsa.Context.nccl(local, rank, world, uid[0])
    else:
        ctx = fsa.Context(local)
    coords, ind, gamma, y = make_inputs(cfg, fsa)
    if gamma is None:
        gamma = calibrate_gamma(coords, cfg["nnz"], fsa, ctx)
    fp64_peak = measure_fp64_peak(torch)
    kw = dict(nu=cfg["nu"], taper_family=1, gamma=gamma, sigma2=cfg["s2"], sigma1_2=cfg["s12"], rho=cfg["rho"])
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
    ctx.set_profiling(True)
    ctx.reset_timers()
    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    ctx.synchronize()
    torch.cuda.synchronize()
    l0 = fsa.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    results = [step() for _ in range(args.steps)]
    e1.record(stream)
    ctx.synchronize()
    torch.cuda.synchronize()
    barrier()
    launches = fsa.launch_count() - l0
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    ms = max_over_ranks(ms)
    timers = ctx.timers()
    ctx.set_profiling(False)
    copies = 1 if sharded else world  # replicas each solve the whole problem
    rhs_its = sum(r["rhs_iterations"] for r in results) * copies
    value = rhs_its / (ms * 1e-3)
    pcg_ms = statistics.median(r["pcg_ms"] for r in results)
    pcg_rate = results[-1]["rhs_iterations"] / (pcg_ms * 1e-3)

    # roofline: every kernel group of the PCG sweep against its bound; the dominant one
    # (largest share of the step) is the headline entry. Algorithmic units per launch come
    # from the library's CUDA-event timers (units accumulated per launch).
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    step_ms = ms / args.steps
    n_, mp_ = cfg["n"], 128 * math.ceil(cfg["m"] / 128)
    np_ = 128 * math.ceil(n_ / 128)
    tp_ = 8 * math.ceil((L + 1) / 8)
    traffic = {}
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic_config%d.json" % args.config)))
    except Exception:
        pass

    def entry(name, kernel, bound, units_per_launch, unit_scale, peak, unit, tkey):
        t = timers.get(name)
        if not t or not t["count"]:
            return None
        avg = t["ms"] / t["count"]
        ach = units_per_launch / (avg * 1e-3) / unit_scale
        return {"kernel": kernel, "bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                "traffic": traffic.get(tkey), "avg_launch_ms": avg, "launches": t["count"],
                "share_of_step": t["ms"] / ms, "units_per_launch": units_per_launch}

    ozaki_on = tp_ <= 64
    sp = timers.get("spmm", {"units": 0.0, "count": 1})
    kernels = [
        entry("spmm", "k_spmm_rt (32-row groups, warp per 8-row tile, DMMA.8x8x4 fp64 block product)", "hbm",
              sp["units"] / max(sp["count"], 1), 1e9, hbm, "GB/s", "k_spmm_rt"),
        entry("lowrank_expand", "k_oz_expand (tcgen05 kind::i8, Ozaki 8 digit planes)" if ozaki_on else
              "k_dgemm expand (DMMA fp64)", "hbm", 8.0 * mp_ * np_ + 24.0 * n_ * tp_, 1e9, hbm, "GB/s",
              "k_oz_expand"),
        entry("lowrank_project", "k_oz_gemm (tcgen05 kind::i8, Ozaki 8 digit planes)" if ozaki_on else
              "k_dgemm reduce (DMMA fp64)", "hbm", 8.0 * mp_ * np_ + 16.0 * n_ * tp_, 1e9, hbm, "GB/s",
              "k_oz_gemm"),
    ]
    kernels = [k for k in kernels if k]
    dom = max(kernels, key=lambda k: k["share_of_step"])
    roofline = dict(dom)
    roofline["peak_source"] = "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"
    roofline["all"] = kernels
    roofline["fp64_dgemm_tflops_measured"] = fp64_peak
    # SURVEY §8d unit: one PCG sweep of the reference operation sequence (krylov.cpp:56-93,
    # fsa.cpp:65-68, preconditioners.cpp:58-61) at the measured peaks, T_roof = sum over phases
    # of max(bytes / BW, flop / P64), against the measured sweep time of this implementation
    nnz_ = nnz
    t_ = L + 1
    phases = {
        "spmm": (12.0 * nnz_ + 4.0 * (n_ + 1), 2.0 * nnz_ * t_),
        "lowrank": (4 * 8.0 * cfg["m"] * n_, 8.0 * cfg["m"] * n_ * t_ + 4.0 * cfg["m"] ** 2 * t_),
        "vectors": (80.0 * n_ * t_, 12.0 * n_ * t_),
    }
    t_roof = sum(max(b / (hbm * 1e9), f / (fp64_peak * 1e12)) for b, f in phases.values()) * 1e3
    sweeps = sum(r["sweeps"] for r in results)
    sweep_groups = ("spmm", "lowrank_project", "lowrank_expand", "core_solve", "cg_blas1", "allreduce",
                    "halo_exchange")
    t_sweep = sum(timers[k]["ms"] for k in sweep_groups if k in timers) / max(sweeps, 1)
    roofline["sweep"] = {"unit": "one PCG sweep (SURVEY.md 8d)", "t_roof_ms": t_roof, "t_measured_ms": t_sweep,
                         "frac": t_roof / t_sweep if t_sweep else None,
                         "note": "T_roof = reference operation sequence at the measured HBM bandwidth and "
                                 "cuBLAS DGEMM rate; this build does half the dense passes and runs them on "
                                 "the INT8 tensor cores, so frac can exceed 1"}

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
    tp = k if k <= 72 else k
    # every rank uploads coords (n x 2), inducing (m x 2) and y (n); reads back nll, grad and the
    # Lanczos coefficients of its columns
    h2d = 8 * world * (n * 2 + m * 2 + n)
    d2h = 8 * world * (5 + 2 * k * last_sweeps(results))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, its, dt = cpu_pcg_sample(cfg, coords, ind, gamma, sweeps=args.ref_sweeps)
            cpu = {"value": v, "unit": "RHS-iterations/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"oracle port, FITC setup untimed, {args.ref_sweeps} lockstep PCG sweeps on the "
                             f"full n={n}, t={k} block ({its} RHS-iterations in {dt:.2f} s)"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "RHS-iterations/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        last = results[-1]
        line = {
            "metric": METRIC, "value": value, "unit": "RHS-iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong" if (sharded and args.mode == "strong") else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded; BASELINE config)",
            "config": {"workload": (f"config{args.config}: loglik+grad, FITC-PCG"
                                    + (f", n = {n // world} x {world} GPUs" if sharded and args.mode == "weak" else "")),
                       "n": n, "m": m, "nnz": nnz,
                       "avg_row_nnz": nnz / n, "probes": L, "rhs": k, "tol": tol, "nu": cfg["nu"],
                       "rho": cfg["rho"], "sigma2": cfg["s2"], "sigma1_2": cfg["s12"], "gamma": gamma,
                       "parallelism": (f"row-sharded x{world} ({args.mode}; NCCL halo exchange + allreduce)"
                                       if sharded else ("replicas" if world > 1 else "single")),
                       "l2": "inputs larger than L2 (U is m x n fp64 = %.0f MB)" % (8 * m * n / 1e6)},
            "loglik_grad_ms": step_ms, "pcg_ms": pcg_ms, "pcg_only_rhs_iter_per_s": pcg_rate,
            "cg_iterations": last["cg_iterations"], "sweeps": last["sweeps"], "nll": last["nll"],
            "grad": list(last["grad"]), "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "RHS-iterations/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_step_ms},
            "gpu_launches": launches, "clocks": clocks,
            "timers_ms": {k2: round(v["ms"] / args.steps, 3) for k2, v in timers.items()},
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
