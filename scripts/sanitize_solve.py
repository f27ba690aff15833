"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck):
BASELINE cfg 1 (coarse-level multigrid only), J = 3 / K = 7 (the register
kernels mg2d_reg at n = 63, 127), the 1D K = 7 kernel, the L-shaped domain
at K = 6, and a 2-virtual-rank time-slab solve.

    compute-sanitizer --tool racecheck python scripts/sanitize_solve.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_08875_b200 as hw  # noqa: E402
from paper_2009_08875_b200 import distributed as D  # noqa: E402
from paper_2009_08875_b200 import inputs  # noqa: E402


def solve(d, J, K, dist, u0, domain="square", Dm=None):
    n_t = 2 ** J + 1
    n_x = hw.discretization.lshape_dofs(K) if domain == "L" else (2 ** K - 1) ** d
    F = inputs.forcing(dist, n_t, n_x)
    prob = hw.ProblemData(D=np.eye(d) if Dm is None else Dm, c=0.0, u0=u0)
    asm = hw.assemble_system(prob, J, K, hw.SolveConfig(), forcing=F, host_rhs=False, domain=domain)
    res = hw.pcg(asm.S, asm.K_X, asm.rhs, 0.0, rtol=1e-6)
    print(f"d={d} J={J} K={K} {domain}: {res.iterations} its", flush=True)
    return asm, res


solve(2, 4, 4, "uniform", inputs.u0_sines)                        # cfg 1
asm, res = solve(2, 3, 7, "uniform", inputs.u0_sines)            # register kernels
solve(1, 3, 7, "normal", inputs.u0_modes())                      # 1D kernel
solve(2, 2, 6, "lshape", inputs.u0_zero, domain="L", Dm=0.25 * np.eye(2))
f = asm.rhs.f_hat.array
dev = torch.device("cuda", 0)
states = D.make_states(2, 3, 7, 2, range(2), lambda p: dev)
Fl = [D.scatter_wavelet(f, st.lay).clone() for st in states]
Wl = [torch.zeros_like(x) for x in Fl]
r2 = D.pcg(D.SlabSystem(states, D.SimComm(2)), Fl, Wl, rtol=1e-6, graphs=False)
print(f"slabs x2: {r2.iterations} its (single GPU {res.iterations})", flush=True)
torch.cuda.synchronize()
print("done")
