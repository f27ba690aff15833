"""A/B of the mg2d_reg thread shapes on small batches: one batched K_x (or
C_j) multigrid apply per batch size, default shapes (P = 8) against the WIDE
shapes of levels chosen by HWG_REG_WIDE bitmasks (hw_mg2d_reg.cu).

    python scripts/mg_wide_sweep.py --K 10 --rows 64 136 272 --masks 0 128 384 896
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_08875_b200.device import GpuContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=10)
ap.add_argument("--op", type=int, default=1)
ap.add_argument("--rows", type=int, nargs="+", default=[64, 136, 148, 272, 296, 514, 1025])
ap.add_argument("--masks", type=int, nargs="+", default=[0, 128, 384, 896])
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--domain", default="square")
ap.add_argument("--var", default="HWG_REG_WIDE", help="env variable the values are tried on "
                "(HWG_REG_CLUSTER: 0 = one 256-thread CTA per n = 2047 row, 1 = CTA pair)")
ap.add_argument("--fixed", nargs="*", default=[], help="NAME=VALUE settings held fixed")
a = ap.parse_args()
for kv in a.fixed:
    name, val = kv.split("=")
    os.environ[name] = val
rmax = max(a.rows)
kw = {"domain": "L"} if a.domain == "L" else {}
ctx = GpuContext(2, 3, a.K, rows_max=rmax, **kw)
n = (2 ** a.K - 1) ** 2
B = torch.randn((rmax, n), dtype=torch.float64, device="cuda")
X = torch.empty_like(B)
ops = torch.full((rmax,), a.op, dtype=torch.int32, device="cuda")
ref = None
for R in a.rows:
    line = [f"rows {R:5d}"]
    for mask in a.masks:
        os.environ[a.var] = str(mask)
        ctx.mg_rows_dev(ops[:R], B[:R], X[:R])
        torch.cuda.synchronize()
        if mask == a.masks[0]:
            ref = X[:4].clone()
        else:
            d = float((X[:4] - ref).abs().max() / ref.abs().max())
            assert d < 1e-11, (mask, d)
            if d != 0.0:
                line.append(f"[diff {d:.1e}]")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            ctx.mg_rows_dev(ops[:R], B[:R], X[:R])
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        line.append(f"mask {mask}: {ms:7.3f} ms")
    print("  ".join(line), flush=True)
