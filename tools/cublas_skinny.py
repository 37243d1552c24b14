"""cuBLAS (torch) fp64 throughput on the PCG's skinny shapes, as a practical roof
for the hand-written DMMA kernels (config 2: n = 1e5, m = 512, t = 56)."""
import sys

import torch


def bench(f, flops, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, flops / (ms * 1e-3) / 1e12


n, m, t = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (100096, 512, 56)))
U = torch.randn(n, m, dtype=torch.float64, device="cuda")   # one row per point (our U storage)
H = torch.randn(n, t, dtype=torch.float64, device="cuda")
W = torch.randn(m, t, dtype=torch.float64, device="cuda")
f = 2.0 * n * m * t
print("expand  U W      (n x m)(m x t): %.3f ms  %.1f TF/s" % bench(lambda: U @ W, f))
print("project U^T H    (m x n)(n x t): %.3f ms  %.1f TF/s" % bench(lambda: U.t() @ H, f))
print("square 8192^3 DGEMM:             %.3f ms  %.1f TF/s" % bench(
    lambda: torch.mm(A, A), 2 * 8192 ** 3) if (A := torch.randn(8192, 8192, dtype=torch.float64, device="cuda")) is not None else "")
