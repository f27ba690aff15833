"""Per-level cost of the 1D register-resident multigrid: time per row of
one batched apply at K = 7..10 (differences = the cost of each streamed level).

    python scripts/mg1d_levels.py [J]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_08875_b200.device import GpuContext  # noqa: E402
from paper_2009_08875_b200 import discretization as disc  # noqa: E402

J = int(sys.argv[1]) if len(sys.argv) > 1 else 17
prev = 0.0
for K in (7, 8, 9, 10):
    ctx = GpuContext(1, J, K)
    n_t, n_x = ctx.n_t, ctx.n_x
    B = torch.randn((n_t, n_x), dtype=torch.float64, device="cuda")
    X = torch.empty_like(B)
    opsd = torch.from_numpy((1 + disc.level_of(J)).astype(np.int32)).cuda()
    for _ in range(3):
        ctx.mg_rows_dev(opsd, B, X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ctx.mg_rows_dev(opsd, B, X)
    e1.record()
    torch.cuda.synchronize()
    ns = e0.elapsed_time(e1) / 20 * 1e6 / n_t
    print(f"K={K}: {ns:6.2f} ns/row (+{ns - prev:5.2f})", flush=True)
    prev = ns
    del ctx, B, X
