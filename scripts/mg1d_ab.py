"""A/B timing and agreement of the 1D multigrid kernels on a cfg-3-shaped
batch (K = 10, 2^J + 1 rows, every row its own C_j operator).

    HWG_MG1D=1 python scripts/mg1d_ab.py [J]        # round-1/2 mg1d_reg (one warp, exact scans)
    HWG_RR_MINB=2 python scripts/mg1d_ab.py [J]     # mg1d_rr at 8 warps/SM (255 registers)
    HWG_RR_MINB=3 python scripts/mg1d_ab.py [J]     # mg1d_rr, 12 warps/SM as 3 CTAs, operator through L1
    python scripts/mg1d_ab.py [J]                   # default (persistent mg1d_rrp, operator in shared memory)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_08875_b200.device import GpuContext  # noqa: E402
from paper_2009_08875_b200 import discretization as disc  # noqa: E402

J = int(sys.argv[1]) if len(sys.argv) > 1 else 15
ctx = GpuContext(1, J, 10)
n_t, n_x = ctx.n_t, ctx.n_x
gen = torch.Generator(device="cuda").manual_seed(3)
B = torch.randn((n_t, n_x), dtype=torch.float64, device="cuda", generator=gen)
X = torch.empty_like(B)
ops = (1 + disc.level_of(J)).astype(np.int32)
opsd = torch.from_numpy(ops).cuda()
for _ in range(3):
    ctx.mg_rows_dev(opsd, B, X)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    ctx.mg_rows_dev(opsd, B, X)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
tag = "k" + os.environ.get("HWG_MG1D", "2") + "m" + os.environ.get("HWG_RR_MINB", "1")
np.save(f"/tmp/mg1d_X_{tag}.npy", X[:64].cpu().numpy())
print(f"HWG_MG1D={tag} J={J} rows={n_t}: {ms:.3f} ms per batch, {ms * 1e3 / n_t * 1e3:.1f} ns/row, "
      f"{16.0 * n_t * n_x / ms / 1e6:.1f} GB/s (b in, x out)")
other = "/tmp/mg1d_X_k1m1.npy"
if tag != "k1m1" and os.path.exists(other):
    A = np.load(other)
    Bf = X[:64].cpu().numpy()
    print(f"{tag} vs mg1d_reg: max rel diff", float(np.abs(A - Bf).max() / np.abs(A).max()))
