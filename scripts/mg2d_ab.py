"""A/B timing of the 2D multigrid batches of a cfg 4 PCG iteration (K = 10):
the 2,050-row K_x batch of S-hat and a 1,025-row C_j batch of K_X (every
row its wavelet level's operator).

    python scripts/mg2d_ab.py                                  # this build
    HWG_LIB_PATH=<other libhwgpu.so> python scripts/mg2d_ab.py # another build
Also saves 8 rows of each result to /tmp for a cross-build comparison.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_08875_b200.device import GpuContext  # noqa: E402
from paper_2009_08875_b200 import discretization as disc  # noqa: E402

J, K = 10, 10
ctx = GpuContext(2, J, K, rows_max=2 * (2 ** J + 1))
nt, nx = ctx.n_t, ctx.n_x
gen = torch.Generator(device="cuda").manual_seed(5)
B = torch.randn((2 * nt, nx), dtype=torch.float64, device="cuda", generator=gen)
X = torch.empty_like(B)
ops_kx = torch.zeros(2 * nt, dtype=torch.int32, device="cuda")
ops_cj = torch.from_numpy((1 + disc.level_of(J)).astype(np.int32)).cuda()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


tag = "alt" if os.environ.get("HWG_LIB_PATH") else "this"
ms = timed(lambda: ctx.mg_rows_dev(ops_kx, B, X))
np.save(f"/tmp/mg2d_kx_{tag}.npy", X[:8].cpu().numpy())
print(f"[{tag}] K_x 2050 rows: {ms:.2f} ms")
ms = timed(lambda: ctx.mg_rows_dev(ops_cj, B[:nt], X[:nt]))
np.save(f"/tmp/mg2d_cj_{tag}.npy", X[nt - 8:nt].cpu().numpy())
print(f"[{tag}] C_j 1025 rows: {ms:.2f} ms")
if tag == "alt" and os.path.exists("/tmp/mg2d_kx_this.npy"):
    for name in ("kx", "cj"):
        a, b = np.load(f"/tmp/mg2d_{name}_this.npy"), np.load(f"/tmp/mg2d_{name}_alt.npy")
        print(f"{name}: max rel diff between builds {np.abs(a - b).max() / np.abs(b).max():.2e}")
