"""Run a few batched MG applies / Schur applies for ncu (one GPU).

    python scripts/profile_mg.py --J 8 --K 8 --reps 2 [--what mg|schur|kx|pcg]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_08875_b200 as hw  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--J", type=int, default=8)
ap.add_argument("--K", type=int, default=8)
ap.add_argument("--d", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--what", default="mg")
ap.add_argument("--domain", default="square", choices=("square", "L"))
a = ap.parse_args()
prob = hw.lshape_problem() if a.domain == "L" else hw.decaying_heat(a.d)
asm = hw.assemble_system(prob, a.J, a.K, hw.SolveConfig(), host_rhs=False, domain=a.domain)
ctx = asm.ctx
n_t, n_x = ctx.n_t, ctx.n_x
x = torch.randn((2 * n_t, n_x), dtype=torch.float64, device="cuda")
if a.domain == "L":        # MG rows in the dof layout (the entry point scatters to the grid)
    pass
y = torch.empty_like(x)
for _ in range(a.reps):
    if a.what == "mg":
        ctx.mg_rows(0, x, y)
    elif a.what == "schur":
        ctx.schur(x[:n_t], y[:n_t])
    elif a.what == "kx":
        ctx.kx(x[:n_t], y[:n_t])
    elif a.what == "pcg":
        ctx.pcg(asm.rhs.f_hat.array, y[:n_t], 0.0, 1e-6)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.reps):
    ctx.mg_rows(0, x, y)
e.record()
torch.cuda.synchronize()
print(f"{a.what}: J={a.J} K={a.K} rows={2 * n_t}: {s.elapsed_time(e) / a.reps:.3f} ms per MG batch")
