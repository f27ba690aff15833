"""A/B timing of the Kronecker stencil kernels at BASELINE cfg 4 size
(J = 10, K = 10: 1025 temporal rows of 1,046,529 points).

    HWG_TMA=1 python scripts/kron_ab.py  # TMA-staged row strips
    python scripts/kron_ab.py            # direct cached loads (default)
Prints ms per call and the achieved HBM rate (compulsory bytes: bside reads
U, writes t1, t1'; bt_side reads g1, g1', writes out; A_x reads x, writes
A x) and a checksum of every output (the variants must agree bit for bit).
"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_08875_b200.device import GpuContext  # noqa: E402

J, K = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (10, 10)
ctx = GpuContext(2, J, K, rows_max=8)
nt, nx = ctx.n_t, ctx.n_x
gen = torch.Generator(device="cuda").manual_seed(1)
U = torch.randn((nt, nx), dtype=torch.float64, device="cuda", generator=gen)
T1 = torch.empty_like(U)
T2 = torch.empty_like(U)
E0 = torch.empty(nx, dtype=torch.float64, device="cuda")
tag = os.environ.get("HWG_TMA", "0")


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def digest(*ts):
    h = hashlib.sha1()
    for t in ts:
        h.update(t.cpu().numpy().tobytes())
    return h.hexdigest()[:16]


N = nt * nx
ms = timed(lambda: ctx.bside_rows(U, 0, T1, T2, 0, nt, E0))
print(f"HWG_TMA={tag} bside   {ms:7.3f} ms  {24 * N / ms / 1e9:7.1f} GB/s  {digest(T1, T2, E0)}")
ms = timed(lambda: ctx.bt_rows(T1, T2, E0, U))
print(f"HWG_TMA={tag} bt_side {ms:7.3f} ms  {24 * N / ms / 1e9:7.1f} GB/s  {digest(U)}")
ms = timed(lambda: ctx.spatial(1, U, T1))
print(f"HWG_TMA={tag} A_x     {ms:7.3f} ms  {16 * N / ms / 1e9:7.1f} GB/s  {digest(T1)}")
