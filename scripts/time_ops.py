"""Time individual operators of one context on the GPU (CUDA events).

    python scripts/time_ops.py --J 10 --K 10 [--reps 3] [--ops wav,wavT,schur,kx,mg,dot]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_08875_b200 import discretization as disc  # noqa: E402
from paper_2009_08875_b200.device import GpuContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--J", type=int, default=10)
ap.add_argument("--K", type=int, default=10)
ap.add_argument("--d", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--ops", default="wav,wavT,schur,kx,mg,dot")
a = ap.parse_args()
ctx = GpuContext(a.d, a.J, a.K)
nt, nx = ctx.n_t, ctx.n_x
x = torch.randn((2 * nt, nx), dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
ops = {
    "wav": lambda: ctx.wavelet(x[:nt], y[:nt], False),
    "wavT": lambda: ctx.wavelet(x[:nt], y[:nt], True),
    "schur": lambda: ctx.schur(x[:nt], y[:nt]),
    "kx": lambda: ctx.kx(x[:nt], y[:nt]),
    "mg": lambda: ctx.mg_rows(0, x, y),
    "dot": lambda: ctx.dot(x[:nt], y[:nt]),
}
for name in a.ops.split(","):
    f = ops[name]
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        f()
    e.record()
    torch.cuda.synchronize()
    print(f"{name:6s} J={a.J} K={a.K}: {s.elapsed_time(e) / a.reps:9.3f} ms")
