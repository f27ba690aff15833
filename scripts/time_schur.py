"""Device time of S-hat applies (W, B-side, K_x batch, B^T-side, W^T) at a given size.

    python scripts/time_schur.py --J 9 --K 10 --reps 5
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_08875_b200 as hw  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--J", type=int, default=9)
ap.add_argument("--K", type=int, default=10)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
asm = hw.assemble_system(hw.decaying_heat(2), a.J, a.K, hw.SolveConfig(), host_rhs=False)
ctx = asm.ctx
x = torch.randn((ctx.n_t, ctx.n_x), dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
ctx.schur(x, y)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.reps):
    ctx.schur(x, y)
e.record()
torch.cuda.synchronize()
print(f"schur J={a.J} K={a.K}: {s.elapsed_time(e) / a.reps:.3f} ms per apply")
