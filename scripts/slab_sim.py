"""Strong-scaling estimate of the time-slab PCG from P virtual ranks on ONE GPU.

    python scripts/slab_sim.py --J 10 --K 10 --P 1 2 4 8

SimComm runs the P ranks' kernels one after another on the same device, so
the solve time T_sim(P) is the sum of the per-rank compute times: a rank of a
real P-GPU run computes for about T_sim(P) / P (its launches cover only its
slab's rows, exactly as on its own GPU).  T_1 / T_sim(P) is therefore the
compute-only parallel efficiency (load imbalance and the under-filled GPU of
a small slab included; NCCL transfer time not).  Per-rank times are also
reported (CUDA events around each rank's share of every operator would need
instrumentation; the max-rank share is approximated by the slab sizes).
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_08875_b200 as hw  # noqa: E402
from paper_2009_08875_b200 import distributed as D, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--J", type=int, default=10)
ap.add_argument("--K", type=int, default=10)
ap.add_argument("--d", type=int, default=2)
ap.add_argument("--P", type=int, nargs="+", default=[1, 2, 4, 8])
a = ap.parse_args()
d, J, K = a.d, a.J, a.K
n_t, n_x = 2 ** J + 1, (2 ** K - 1) ** d
F = inputs.forcing("uniform" if d == 2 else "normal", n_t, n_x)
u0 = inputs.u0_sines if d == 2 else inputs.u0_modes()
asm = hw.assemble_system(hw.ProblemData(D=np.eye(d), c=0.0, u0=u0), J, K, hw.SolveConfig(),
                         forcing=F, host_rhs=False)
f = asm.rhs.f_hat.array
w1 = torch.empty_like(f)
asm.ctx.pcg(f, w1, 0.0, 1e-6)                       # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
stats, _ = asm.ctx.pcg(f, w1, 0.0, 1e-6)
torch.cuda.synchronize()
t1 = time.perf_counter() - t0
its = stats["iterations"]
print(f"single GPU hwg_pcg: {t1 * 1e3:.1f} ms, {its} its")
del asm
dev = torch.device("cuda", 0)
for P in a.P:
    states = D.make_states(d, J, K, P, range(P), lambda p: dev)
    Fl = [D.scatter_wavelet(f, st.lay).clone() for st in states]
    Wl = [torch.zeros_like(x) for x in Fl]
    system = D.SlabSystem(states, D.SimComm(P))
    D.pcg(system, Fl, Wl, rtol=1e-6)                # warm-up
    for x in Wl:
        x.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = D.pcg(system, Fl, Wl, rtol=1e-6)
    torch.cuda.synchronize()
    tp = time.perf_counter() - t0
    rows = [st.lay.n_w for st in states]
    print(f"P={P}: T_sim {tp * 1e3:.1f} ms ({res.iterations} its), per-rank ~{tp / P * 1e3:.1f} ms, "
          f"compute-only efficiency T_1/T_sim = {t1 / tp:.3f}, wavelet rows per rank "
          f"{min(rows)}..{max(rows)}")
    del states, Fl, Wl, system
    torch.cuda.empty_cache()
