"""Device time of ONE rank of a P-rank time-slab PCG iteration, measured alone
on one GPU (the other ranks' halo rows and all-gathered partials replaced by
zeros -- the arithmetic is meaningless, the kernel sequence and sizes are
exactly the rank's).  T_1 / (P * T_rank) is the compute-only strong-scaling
efficiency of a real P-GPU run (NCCL transfer time excluded; SURVEY §8e puts
it at ~1% of the iteration).  Also times each operator of the iteration.

    python scripts/slab_rank_time.py --J 10 --K 10 --P 1 2 4 8 [--ranks 0 -1]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_08875_b200 import distributed as D  # noqa: E402


class NullComm:
    """Exchanges are dropped; all-gathers return zeros with the rank's own slot."""

    def __init__(self, P, p):
        self.P, self.p = P, p

    def exchange(self, states, plan):
        pass

    def allgather(self, states, tensors):
        (t,) = tensors
        out = torch.zeros((self.P,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        out[self.p] = t
        return [out]


ap = argparse.ArgumentParser()
ap.add_argument("--J", type=int, default=10)
ap.add_argument("--K", type=int, default=10)
ap.add_argument("--d", type=int, default=2)
ap.add_argument("--P", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--ranks", type=int, nargs="+", default=[0, -1])
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--domain", default="square")
a = ap.parse_args()
dev = torch.device("cuda", 0)
Dm = 0.25 * np.eye(2) if a.domain == "L" else None


def ev():
    return torch.cuda.Event(enable_timing=True)


base = None
for P in a.P:
    for rr in a.ranks:
        p = rr % P
        states = D.make_states(a.d, a.J, a.K, P, [p], lambda q: dev, D=Dm, domain=a.domain)
        system = D.SlabSystem(states, NullComm(P, p))
        st = states[0]
        shape = (st.lay.n_w, st.mid.shape[1])
        g = torch.Generator(device="cuda").manual_seed(1)
        X = [torch.randn(shape, dtype=torch.float64, device=dev, generator=g)]
        Y = [torch.empty_like(X[0])]
        R = [X[0].clone()]
        Z = [torch.empty_like(X[0])]
        W = [torch.zeros_like(X[0])]

        def iteration(marks=None):
            e = [ev() for _ in range(4)] if marks is not None else None
            if e: e[0].record()
            system.schur(X, Y)
            if e: e[1].record()
            system.dot(X, Y)
            system.axpy(0.1, X, W)
            system.axpy(-0.1, Y, R)
            if e: e[2].record()
            system.kx_dot(R, Z)
            system.xpay(0.5, Z, X)
            if e: e[3].record()
            if marks is not None:
                marks.append(e)

        iteration()
        torch.cuda.synchronize()
        marks = []
        t0, t1 = ev(), ev()
        t0.record()
        for _ in range(a.iters):
            iteration(marks)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / a.iters
        parts = np.mean([[m[0].elapsed_time(m[1]), m[1].elapsed_time(m[2]),
                          m[2].elapsed_time(m[3])] for m in marks], axis=0)
        if P == 1:
            base = ms
        eff = base / (P * ms) if base else float("nan")
        print(f"P={P} rank {p}: {ms:7.2f} ms/iteration (schur {parts[0]:.2f}, dot+axpy "
              f"{parts[1]:.2f}, K_X+dot+xpay {parts[2]:.2f}); rows n_w={st.lay.n_w} "
              f"n_out={st.lay.n_out}; efficiency vs P=1 {eff:.3f}", flush=True)
        del states, system, st, X, Y, R, Z, W
        import gc
        gc.collect()
        torch.cuda.empty_cache()
