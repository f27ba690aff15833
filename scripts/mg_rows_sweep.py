"""Per-row cost of one batched K_x multigrid apply vs batch size (the
under-filled GPU of small time slabs), register kernel P = 8 x 128 threads
(2 CTAs/SM) vs P = 4 x 256 threads (HWG_MG_REG=4).  Measured: the P = 4
variant is slower at every batch size.

    python scripts/mg_rows_sweep.py [--K 10] [--rows 64 137 258 296 1025 2050]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_08875_b200.device import GpuContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=10)
ap.add_argument("--rows", type=int, nargs="+", default=[64, 137, 148, 200, 258, 296, 1025, 2050])
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
rmax = max(a.rows)
ctxs = {}
for name, env in (("P8x128", "1"), ("P4x256", "4")):
    os.environ["HWG_MG_REG"] = env
    ctxs[name] = GpuContext(2, 3, a.K, rows_max=rmax)
n = (2 ** a.K - 1) ** 2
B = torch.randn((rmax, n), dtype=torch.float64, device="cuda")
X = torch.empty_like(B)
ops = torch.ones(rmax, dtype=torch.int32, device="cuda")
for R in a.rows:
    line = [f"rows {R:5d}"]
    for name, ctx in ctxs.items():
        ctx.mg_rows_dev(ops[:R], B[:R], X[:R])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            ctx.mg_rows_dev(ops[:R], B[:R], X[:R])
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        line.append(f"{name}: {ms:8.2f} ms ({1e3 * ms / R:6.1f} us/row)")
    print("  ".join(line), flush=True)
