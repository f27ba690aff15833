"""Time-slab multi-GPU PCG (design (a)).

The reference distributes temporal rows over a thread pool with halo reads
(ParallelPlan / WorkerPool, /root/reference/pkg/src/heatwave/solver.py:
47-108); the paper distributes them over MPI ranks.  Here
P = 2^L0 GPUs each own a time slab:

* nodal rows (single-scale arrays of S): rank p owns nodes [pH, (p+1)H),
  H = 2^J / P, and the last rank also owns the end node 2^J;
* wavelet rows (PCG vectors, K_X): levels j <= L0 (the P + 1 coarsest rows)
  are REPLICATED on every rank; for j > L0 rank p owns the level-j wavelets
  centred in its slab, k in [p 2^(j-1)/P, (p+1) 2^(j-1)/P).

Exchanges per PCG iteration: one coarse-node and one wavelet halo row per
distributed synthesis stage, one halo row on each side for the temporal
bands of S, one fine-node halo on each side per transposed stage, an
allgather of the P + 1 level-L0 nodal rows, and an allgather of the per-row
dot partials.  The partials are reassembled in GLOBAL row order and reduced
with the reference's fixed pairwise tree on every rank, so inner products
(hence iterates and iteration counts) are identical for every P -- the
reference's worker-count determinism (tests/test_solver.py:129-142).  K_X
and every multigrid solve are row-local: no communication.

L-shaped domain (BASELINE cfg 5): every slab array is in the embedded grid
layout of the kernel contexts (removed quadrant held at zero); the
user-facing inputs and outputs (forcing rows, u0 moments, host f-hat / u in
``solve_host``) are in the dof layout and converted by hwg_grid_scatter /
hwg_grid_gather on the rank that owns them.

The code is SPMD over a list of rank states.  A real run holds its own
state and a ``TorchComm`` (NCCL between GPUs, gloo on CPUs); ``SimComm``
holds all P states in one process and delivers messages by copying, which
runs P virtual ranks one after another on one device (the tests; no kernel
ever waits for another rank).  Every exchange is a pure function of (rank
layout, stage) -> [Msg], so a real rank derives the receives it must post
from its neighbours' plans without seeing their data.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable, List, NamedTuple

import numpy as np

from . import discretization as disc


# --------------------------------------------------------------------------
# partition
# --------------------------------------------------------------------------
@dataclass
class RankLayout:
    p: int
    P: int
    J: int
    H: int
    L0: int
    last: bool
    n_out: int                    # nodal rows owned (H, +1 on the last rank)
    n_w: int                      # wavelet rows held (P + 1 replicated + H - 1 own)
    global_rows: np.ndarray       # global wavelet row of each local row
    owned: np.ndarray             # counts in dots (replicated rows only on rank 0)
    level_of: np.ndarray          # wavelet level of each local row
    block: dict                   # level j > L0 -> (local start, count)

    @property
    def left(self):
        return self.p - 1 if self.p > 0 else None

    @property
    def right(self):
        return self.p + 1 if not self.last else None


_LAYOUTS = {}


def slab_layout(J: int, P: int, p: int) -> RankLayout:
    key = (J, P, p)
    if key in _LAYOUTS:
        return _LAYOUTS[key]
    if P < 1 or P & (P - 1):
        raise ValueError("the number of ranks must be a power of two")
    if P > 2 ** (J - 1):
        raise ValueError(f"at most 2^(J-1) = {2 ** (J - 1)} ranks for J = {J}")
    if not 0 <= p < P:
        raise ValueError("rank out of range")
    L0 = P.bit_length() - 1
    H = 2 ** J // P
    rows = list(range(P + 1))
    block = {}
    for j in range(L0 + 1, J + 1):
        n = 2 ** (j - 1) // P
        block[j] = (len(rows), n)
        rows.extend(2 ** (j - 1) + 1 + p * n + k for k in range(n))
    g = np.array(rows, dtype=np.int64)
    owned = np.ones(len(g), dtype=bool)
    if p > 0:
        owned[:P + 1] = False
    last = p == P - 1
    lay = RankLayout(p, P, J, H, L0, last, H + (1 if last else 0), len(g), g, owned,
                     disc.level_of(J)[g], block)
    _LAYOUTS[key] = lay
    return lay


class Msg(NamedTuple):
    src: str          # source buffer name on the sending rank
    src_row: int
    dst: int          # destination rank
    dst_buf: str
    dst_row: int


# stage buffers share one layout: [left halo | own rows | right slot]
def _syn_buf(j, J):
    return "U" if j == J else ("B1" if (J - j) % 2 else "B2")


def _ana_buf(j, J):
    return "Xa" if j == J else ("B1" if (J - j) % 2 else "B2")


def edge_plan(lay: RankLayout, buf: str, n_own: int) -> List[Msg]:
    """First own row -> left neighbour's slot; last own row -> right
    neighbour's left halo (both buffers laid out [halo | n_own | slot])."""
    out = []
    if lay.left is not None:
        out.append(Msg(buf, 1, lay.left, buf, n_own + 1))
    if lay.right is not None:
        out.append(Msg(buf, n_own, lay.right, buf, 0))
    return out


def syn_plan(lay: RankLayout, j: int) -> List[Msg]:
    """Halos of synthesis stage j > L0: my first coarse node (row 1 of the
    previous stage's output) to the left neighbour's slot, my last level-j
    wavelet to the right neighbour's wavelet halo."""
    out = []
    n_c = 2 ** (j - 1) // lay.P
    if j > lay.L0 + 1 and lay.left is not None:
        prev = _syn_buf(j - 1, lay.J)
        out.append(Msg(prev, 1, lay.left, prev, n_c + 1))
    if lay.right is not None:
        off, n = lay.block[j]
        out.append(Msg("X", off + n - 1, lay.right, "D", 0))
    return out


# --------------------------------------------------------------------------
# communicators
# --------------------------------------------------------------------------
class SimComm:
    """All ranks in one process; messages are device copies."""

    def __init__(self, P):
        self.P = P

    def exchange(self, states, plan: Callable[[RankLayout], List[Msg]]):
        for st in states:
            for m in plan(st.lay):
                states[m.dst].bufs[m.dst_buf][m.dst_row].copy_(st.bufs[m.src][m.src_row])

    def allgather(self, states, tensors):
        import torch
        stacked = torch.stack(list(tensors))
        return [stacked for _ in states]

    def allreduce_max(self, tensors):
        import torch
        m = torch.stack(list(tensors)).amax(dim=0)
        for t in tensors:
            t.copy_(m)

    capturable = True         # device copies only: a whole iteration fits one CUDA graph


class TorchComm:
    """torch.distributed process group (NCCL between GPUs, gloo on CPUs)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.P = dist.get_world_size()
        self.rank = dist.get_rank()

    def exchange(self, states, plan):
        dist = self.dist
        (st,) = states
        lay = st.lay
        ops = []
        for m in plan(lay):
            ops.append(dist.P2POp(dist.isend, st.bufs[m.src][m.src_row].contiguous(), m.dst))
        for q in (lay.left, lay.right):
            if q is None:
                continue
            for m in plan(slab_layout(lay.J, lay.P, q)):
                if m.dst == lay.p:
                    ops.append(dist.P2POp(dist.irecv, st.bufs[m.dst_buf][m.dst_row], q))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def allgather(self, states, tensors):
        import torch
        (t,) = tensors
        if self.P == 1:
            return [t.unsqueeze(0)]
        out = torch.empty((self.P, *t.shape), dtype=t.dtype, device=t.device)
        if t.is_cuda:                        # NCCL: one gather into a flat buffer
            self.dist.all_gather_into_tensor(out, t.contiguous())
        else:                                # gloo has no flat all-gather
            self.dist.all_gather(list(out.unbind(0)), t.contiguous())
        return [out]

    def allreduce_max(self, tensors):
        (t,) = tensors
        if self.P > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)

    @property
    def capturable(self):
        # one rank: no collective at all.  P > 1: NCCL inside a captured graph
        # is opt-in (HWG_SLAB_GRAPH=1); by default the iteration is issued
        # eagerly, still with a single host synchronisation.
        import os
        return self.P == 1 or os.environ.get("HWG_SLAB_GRAPH") == "1"


# --------------------------------------------------------------------------
# per-rank state
# --------------------------------------------------------------------------
class RankState:
    """Buffers of one rank.  ``kern`` provides the local kernels (the C ABI's
    time-slab entry points via GpuContext, or a test double)."""

    def __init__(self, lay: RankLayout, kern, n_x, device, dtype=None):
        import torch
        dtype = dtype or torch.float64
        self.lay = lay
        self.k = kern
        H = lay.H
        z = lambda r: torch.zeros((r, n_x), dtype=dtype, device=device)  # noqa: E731
        self.bufs = {"U": z(H + 2), "Xa": z(H + 2), "B1": z(H + 2), "B2": z(H + 2),
                     "D": z(1), "X": None}            # D: the left neighbour's wavelet halo row
        self.CN = [z(2 ** j + 1) for j in range(lay.L0 + 1)]     # replicated coarse nodal
        self.T12 = z(2 * lay.n_out)
        self.G12 = z(2 * lay.n_out)
        self.E0 = z(1)[0] if lay.p == 0 else None
        self.mid = z(lay.n_w)
        self.part = torch.zeros(lay.n_w, dtype=dtype, device=device)
        self.owned = torch.as_tensor(lay.owned.astype(np.float64), dtype=dtype, device=device)
        self.ops_kx = torch.as_tensor(1 + lay.level_of, dtype=torch.int32, device=device)
        self.ops_zero = torch.zeros(2 * lay.n_out, dtype=torch.int32, device=device)
        # global-order assembly of dot partials (same on every rank)
        J, P = lay.J, lay.P
        src_idx, dst_idx = [], []
        for q in range(P):
            lq = slab_layout(J, P, q)
            own = np.nonzero(lq.owned)[0]
            src_idx.append(q * lq.n_w + own)
            dst_idx.append(lq.global_rows[own])
        n_w_max = max(slab_layout(J, P, q).n_w for q in range(P))
        assert all(slab_layout(J, P, q).n_w == n_w_max for q in range(P))
        self.gsrc = torch.as_tensor(np.concatenate(src_idx), device=device)
        self.gdst = torch.as_tensor(np.concatenate(dst_idx), device=device)
        self.glob = torch.zeros(2 ** J + 1, dtype=dtype, device=device)
        self.res = torch.zeros(1, dtype=dtype, device=device)
        self.contrib = torch.zeros(lay.n_w, dtype=dtype, device=device)
        # PCG scalars on the device: [rho, pq, rho_new, alpha, beta] (hwg_pcg's
        # layout) and their pinned host mirror, read once per iteration
        self.scal = torch.zeros(8, dtype=dtype, device=device)
        is_cuda = torch.device(device).type == "cuda"
        self.hscal = torch.zeros(8, dtype=dtype, pin_memory=is_cuda)
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)


# --------------------------------------------------------------------------
# distributed operators
# --------------------------------------------------------------------------
class SlabSystem:
    """S-hat, K_X and dots over time slabs."""

    def __init__(self, states, comm):
        self.states = states
        self.comm = comm
        self.P = states[0].lay.P
        self.J = states[0].lay.J
        self.L0 = states[0].lay.L0

    # W: wavelet X -> nodal rows in U[1 : 1 + n_out]
    def synthesis(self, X):
        J, L0, P = self.J, self.L0, self.P
        for st, x in zip(self.states, X):
            st.bufs["X"] = x
            st.CN[0].copy_(x[0:2])
            for j in range(1, L0 + 1):
                nc = 2 ** (j - 1) + 1
                st.k.syn_stage(j, st.CN[j - 1], 0, x[nc:2 ** j + 1], 0, st.CN[j], 0, 2 ** j + 1)
        for j in range(L0 + 1, J + 1):
            self.comm.exchange(self.states, lambda lay, j=j: syn_plan(lay, j))
            n_c = 2 ** (j - 1) // P
            for st, x in zip(self.states, X):
                lay = st.lay
                c0 = lay.p * n_c
                cin = st.CN[L0][lay.p:lay.p + 2] if j == L0 + 1 else \
                    st.bufs[_syn_buf(j - 1, J)][1:n_c + 2]
                off, n = lay.block[j]
                halo = st.bufs["D"][0] if lay.p > 0 else None     # wavelet c0 - 1
                out = st.bufs[_syn_buf(j, J)][1:]
                st.k.syn_stage(j, cin, c0, x[off:off + n], c0, out, 2 * c0,
                               2 * n_c + (1 if lay.last else 0), Dh=halo)

    # W^T: nodal rows in Xa[1 : 1 + n_out] -> wavelet Y
    def analysis(self, Y):
        J, L0, P = self.J, self.L0, self.P
        H = self.states[0].lay.H
        self.comm.exchange(self.states, lambda lay: edge_plan(lay, "Xa", H))
        for j in range(J, L0, -1):
            n_c = 2 ** (j - 1) // P
            for st, y in zip(self.states, Y):
                lay = st.lay
                c0 = lay.p * n_c
                xin = st.bufs[_ana_buf(j, J)][:2 * n_c + 2]
                cout = st.bufs[_ana_buf(j - 1, J)][1:]
                off, n = lay.block[j]
                st.k.ana_stage(j, xin, 2 * c0 - 1, cout, c0, n_c + (1 if lay.last else 0),
                               y[off:off + n], c0, n_c)
            if j > L0 + 1:
                buf = _ana_buf(j - 1, J)
                self.comm.exchange(self.states, lambda lay, b=buf, n=n_c: edge_plan(lay, b, n))
        # level-L0 nodes: rank p holds node p (and the last rank node P)
        buf = _ana_buf(L0, J)
        gathered = self.comm.allgather(self.states, [st.bufs[buf][1:3] for st in self.states])
        for st, y, g in zip(self.states, Y, gathered):
            cn = st.CN[L0]
            cn[:P].copy_(g[:, 0])
            cn[P].copy_(g[P - 1, 1])
            for j in range(L0, 0, -1):
                nc = 2 ** (j - 1) + 1
                dst_c = y[0:2] if j == 1 else st.CN[j - 1]
                st.k.ana_stage(j, st.CN[j], 0, dst_c, 0, nc, y[nc:2 ** j + 1], 0, 2 ** (j - 1))
            if L0 == 0:
                y[0:2].copy_(cn[0:2])

    def schur(self, X, Y):
        """Y = S-hat X (system.py:116-147, 182-187), time-slab distributed."""
        self.synthesis(X)
        H = self.states[0].lay.H
        self.comm.exchange(self.states, lambda lay: edge_plan(lay, "U", H))
        for st in self.states:
            lay = st.lay
            n = lay.n_out
            st.k.bside_rows(st.bufs["U"], lay.p * H - 1, st.T12[:n], st.T12[n:], lay.p * H, n,
                            st.E0)
            st.k.mg_rows_dev(st.ops_zero, st.T12, st.G12)
            st.k.bt_rows(st.G12[:n], st.G12[n:], st.E0, st.bufs["Xa"][1:1 + n])
        self.analysis(Y)

    def kx(self, X, Y):
        """Y = K_X X (system.py:242-276): row-local, no communication."""
        for st, x, y in zip(self.states, X, Y):
            st.k.mg_rows_dev(st.ops_kx, x, y)
            st.k.spatial(1, y, st.mid)
            st.k.mg_rows_dev(st.ops_kx, st.mid, y)

    def kx_dot_dev(self, X, Y, slot):
        """Y = K_X X and <X, Y> -> scal[slot] on every rank's device, the
        per-row partials fused into the last multigrid pass (the same kernels
        as the single-GPU hwg_pcg)."""
        for st, x, y in zip(self.states, X, Y):
            st.k.mg_rows_dev(st.ops_kx, x, y)
            st.k.spatial(1, y, st.mid)
            st.k.mg_rows_dev_dot(st.ops_kx, st.mid, y, x, st.part)
        self._reduce_partials(slot)

    def dot_dev(self, X, Y, slot):
        """<X, Y> -> scal[slot] (device) with the reference's fixed tree over
        the per-row partials in GLOBAL row order (solver.py:111-129) --
        identical for every number of ranks."""
        for st, x, y in zip(self.states, X, Y):
            st.k.row_partials(x, y, st.part)
        self._reduce_partials(slot)

    def kx_dot(self, X, Y):
        self.kx_dot_dev(X, Y, 5)
        return self.read_scalar(5)

    def dot(self, X, Y):
        self.dot_dev(X, Y, 5)
        return self.read_scalar(5)

    def _reduce_partials(self, slot):
        import torch
        for st in self.states:
            torch.mul(st.part, st.owned, out=st.contrib)
        gathered = self.comm.allgather(self.states, [st.contrib for st in self.states])
        for st, g in zip(self.states, gathered):
            st.glob[st.gdst] = g.reshape(-1)[st.gsrc]
            st.k.tree_sum(st.glob, st.glob.numel(), st.scal[slot:slot + 1])

    def read_scalar(self, slot):
        """One scalar from rank-local device memory (a host synchronisation;
        every rank holds the same value)."""
        return float(self.states[0].scal[slot].item())

    def read_scalars(self):
        """The pinned mirror filled at the end of an iteration (one sync)."""
        import torch
        if self.states[0].scal.is_cuda:
            torch.cuda.current_stream(self.states[0].scal.device).synchronize()
        return self.states[0].hscal.tolist()

    def any_nonzero(self, X):
        """any(X != 0) over all ranks (the reference's zero right-hand side
        test, np.any(f), solver.py:196-198)."""
        for st, x in zip(self.states, X):
            st.flag.zero_()
            st.k.any_nonzero(x, st.flag)
        self.comm.allreduce_max([st.flag for st in self.states])
        return bool(int(self.states[0].flag.item()))

    def iteration(self, F, W, R, Pv, Q, Z, recompute):
        """One PCG iteration (solver.py:212-256) with every scalar on the
        device: q = S p; p.q; alpha; r -= alpha q (w += alpha p deferred into
        the p pass, or applied first when the residual is recomputed);
        z = K_X r with r.z fused; beta; w/p update; the scalars copied to the
        pinned host mirror.  No host synchronisation inside, so it can be
        captured as one CUDA graph."""
        self.schur(Pv, Q)
        self.dot_dev(Pv, Q, 1)
        for st, w, r, p, q in zip(self.states, W, R, Pv, Q):
            st.k.pcg_scalar(0, st.scal)
            st.k.pcg_update_wr(w, r, p, q, st.scal, recompute, not recompute)
        if recompute:
            self.schur(W, Z)
            for st, f, z, r in zip(self.states, F, Z, R):
                st.k.sub(f, z, r)
        self.kx_dot_dev(R, Z, 2)
        for st, w, p, z in zip(self.states, W, Pv, Z):
            st.k.pcg_scalar(1, st.scal)
            st.k.pcg_update_wp(w, p, z, st.scal, not recompute)
            st.hscal.copy_(st.scal, non_blocking=True)

    @property
    def capturable(self):
        # per-launch profiling events (hwg_profile_enable) need plain launches
        profiling = any(getattr(getattr(st.k, "ctx", None), "profiling", False) for st in self.states)
        return all(st.scal.is_cuda for st in self.states) and self.comm.capturable and not profiling

    def axpy(self, a, X, Y):
        for st, x, y in zip(self.states, X, Y):
            st.k.axpy(a, x, y)

    def xpay(self, a, X, Y):
        for st, x, y in zip(self.states, X, Y):
            st.k.xpay(a, x, y)


# --------------------------------------------------------------------------
# PCG (solver.py:181-263) over time slabs
# --------------------------------------------------------------------------
@dataclass
class SlabPCGResult:
    iterations: int
    residual_norms: list
    alphas: list = field(default_factory=list)
    betas: list = field(default_factory=list)
    seconds: float = 0.0


def pcg(system: SlabSystem, F, W, epsilon=0.0, rtol=0.0, max_iterations=200,
        recompute_every=50, graphs=None):
    """F, W: lists (one per local state) of wavelet-local arrays; W is
    overwritten with the solution.  Same stopping rule as `api.pcg`.

    Scalars stay on the device (hwg_pcg's kernels): each iteration ends with
    ONE host synchronisation to read p.q, r.z, alpha and beta.  On CUDA with a
    capturable communicator (one rank, or the in-process SimComm) every
    iteration without residual recomputation is replayed as one CUDA graph
    (``graphs=False`` forces plain launches)."""
    import torch
    if not (epsilon > 0) and not (rtol > 0):
        raise ValueError("tolerance must be positive")
    t0 = time.perf_counter()
    R = [f.clone() for f in F]
    Z = [torch.empty_like(f) for f in F]
    Pv = [torch.empty_like(f) for f in F]
    Q = [torch.empty_like(f) for f in F]
    for w in W:
        w.zero_()
    if not system.any_nonzero(F):
        return SlabPCGResult(0, [0.0])
    system.kx_dot_dev(R, Z, 0)                    # rho -> scal[0]
    rho = system.read_scalar(0)
    hist = [math.sqrt(max(rho, 0.0))]
    eps = rtol * hist[0] if rtol > 0 else epsilon
    if rho <= eps ** 2:
        return SlabPCGResult(0, hist, seconds=time.perf_counter() - t0)
    for p_, z in zip(Pv, Z):
        p_.copy_(z)
    use_graph = system.capturable if graphs is None else (graphs and system.capturable)
    graph = None
    alphas, betas = [], []
    for it in range(1, max_iterations + 1):
        recompute = it % recompute_every == 0
        if use_graph and not recompute:
            if graph is None:
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    system.iteration(F, W, R, Pv, Q, Z, False)
            graph.replay()
        else:
            system.iteration(F, W, R, Pv, Q, Z, recompute)
        _, pq, rho_new, alpha, beta = system.read_scalars()[:5]
        if not pq > 0:
            raise RuntimeError(f"operator lost positive definiteness (p^T S p = {pq:g})")
        alphas.append(alpha)
        betas.append(beta)
        hist.append(math.sqrt(max(rho_new, 0.0)))
        if rho_new <= eps ** 2:
            return SlabPCGResult(it, hist, alphas, betas, time.perf_counter() - t0)
    from ._lib import IterationLimitError
    raise IterationLimitError(f"PCG did not reach tolerance {eps:g} within {max_iterations} "
                              "iterations", hist)


# --------------------------------------------------------------------------
# the CUDA kernel provider and helpers
# --------------------------------------------------------------------------
class CudaKernels:
    """Local kernels of one rank: a kernel-only hwg context on its GPU."""

    def __init__(self, d, J, K, alpha=0.3, vcycles=2, smooth=3, device=0, rows_max=0, D=None,
                 c=0.0, domain="square"):
        from .device import GpuContext
        self.ctx = GpuContext(d, J, K, alpha, vcycles, smooth, D, c, device, rows_max=rows_max,
                              domain=domain)
        ctx = self.ctx
        self.domain = domain
        self.n_dof = ctx.n_x
        self.grid_scatter = ctx.grid_scatter
        self.grid_gather = ctx.grid_gather
        self.syn_stage = ctx.syn_stage
        self.ana_stage = ctx.ana_stage
        self.bside_rows = ctx.bside_rows
        self.bt_rows = ctx.bt_rows
        self.mg_rows_dev = ctx.mg_rows_dev
        self.mg_rows_dev_dot = ctx.mg_rows_dev_dot
        self.row_partials = ctx.row_partials
        self.tree_sum = ctx.tree_sum
        self.axpy = ctx.axpy
        self.xpay = ctx.xpay
        self.pcg_scalar = ctx.pcg_scalar
        self.pcg_update_wr = ctx.pcg_update_wr
        self.pcg_update_wp = ctx.pcg_update_wp
        self.sub = ctx.sub
        self.any_nonzero = ctx.any_nonzero
        self.spatial = ctx.spatial
        self.temporal_rows = ctx.temporal_rows


def make_states(d, J, K, P, ranks, device_of, alpha=0.3, vcycles=2, smooth=3, D=None, c=0.0,
                domain="square"):
    """RankStates (CUDA kernels) for the given ranks of a P-rank slab run
    (arrays in the kernels' grid layout: (2^K - 1)^d points per row)."""
    import torch
    states = []
    n_x = (2 ** K - 1) ** d
    for p in ranks:
        lay = slab_layout(J, P, p)
        dev = device_of(p)
        rows_max = max(2 * lay.n_out, lay.n_w, 2 ** J // P + 2) + 2
        kern = CudaKernels(d, J, K, alpha, vcycles, smooth, dev.index or 0, rows_max=rows_max,
                           D=D, c=c, domain=domain)
        states.append(RankState(lay, kern, n_x, dev, torch.float64))
    return states


def _is_lshape(st):
    return getattr(st.k, "domain", "square") == "L"


def to_grid(st, X):
    """dof-layout rows -> the rank's grid layout (identity on the square)."""
    import torch
    if not _is_lshape(st):
        return X
    Y = torch.empty((X.shape[0], st.mid.shape[1]), dtype=X.dtype, device=X.device)
    st.k.grid_scatter(X.contiguous(), Y)
    return Y


def from_grid(st, X):
    """grid-layout rows -> dof layout (identity on the square)."""
    import torch
    if not _is_lshape(st):
        return X
    Y = torch.empty((X.shape[0], st.k.n_dof), dtype=X.dtype, device=X.device)
    st.k.grid_gather(X.contiguous(), Y)
    return Y


def scatter_wavelet(X, lay: RankLayout):
    """Local wavelet rows of rank `lay.p` from a global (N_t, N_x) array."""
    import torch
    idx = torch.as_tensor(lay.global_rows, device=X.device) if hasattr(X, "device") else lay.global_rows
    return X[idx]


def gather_wavelet(parts, layouts, out):
    """Global array from the ranks' local wavelet rows (owned rows only)."""
    import torch
    for x, lay in zip(parts, layouts):
        own = np.nonzero(lay.owned)[0]
        if hasattr(out, "device"):
            out[torch.as_tensor(lay.global_rows[own], device=out.device)] = \
                x[torch.as_tensor(own, device=x.device)]
        else:
            out[lay.global_rows[own]] = x[own]
    return out


# --------------------------------------------------------------------------
# right-hand side over time slabs (system.py:295-324)
# --------------------------------------------------------------------------
def rhs(system: SlabSystem, forcing_rows, u0proj):
    """Local slices of f-hat = W^T( B^T K_Y (N (x) M_x) F + e_0 (x) <u0, phi> ).

    forcing_rows(r0, r1) -> nodal forcing rows [r0, r1) as a tensor on the
    rank's device (the blockwise-seeded generator makes them independent of
    P); u0proj: the N_x moments <u0, phi_i> (used by rank 0 only); both in
    the dof layout.  Returns
    one wavelet-local array per state.  Each rank assembles the test-space
    load of the time elements touching its slab (one halo element), applies
    K_Y = O^-1 (x) K_x (O = I) row-locally, B^T on its nodal rows and the
    distributed W^T."""
    import torch
    J, P = system.J, system.P
    nt = 2 ** J + 1
    G = []
    for st in system.states:
        lay = st.lay
        H = lay.H
        e0, e1 = max(lay.p * H - 1, 0), min(lay.p * H + H, nt - 1)     # time elements
        Fr = to_grid(st, forcing_rows(e0, e1 + 1))                     # nodes e0..e1
        MxF = torch.empty_like(Fr)
        st.k.spatial(0, Fr, MxF)
        y = torch.empty((2 * (e1 - e0), Fr.shape[1]), dtype=Fr.dtype, device=Fr.device)
        st.k.temporal_rows("N", MxF, e0, y, 2 * e0, 2 * (e1 - e0))
        ky = torch.empty_like(y)
        st.k.mg_rows_dev(torch.zeros(y.shape[0], dtype=torch.int32, device=y.device), y, ky)
        n = lay.n_out
        w1 = torch.empty((n, Fr.shape[1]), dtype=Fr.dtype, device=Fr.device)
        w2 = torch.empty_like(w1)
        st.k.temporal_rows("TT", ky, 2 * e0, w1, lay.p * H, n)
        st.k.temporal_rows("NT", ky, 2 * e0, w2, lay.p * H, n)
        st.k.bt_rows(w1, w2, None, st.bufs["Xa"][1:1 + n])
        G.append(torch.empty((lay.n_w, Fr.shape[1]), dtype=Fr.dtype, device=Fr.device))
    system.analysis(G)
    U = []
    for st in system.states:
        xa = st.bufs["Xa"]
        xa.zero_()
        if st.lay.p == 0 and u0proj is not None:
            xa[1].copy_(to_grid(st, u0proj.reshape(1, -1))[0])
        U.append(torch.empty_like(G[len(U)]))
    system.analysis(U)
    return [g + u for g, u in zip(G, U)]


def solve_host(system: SlabSystem, f_host, u_host, rtol=1e-6, epsilon=0.0, max_iterations=200):
    """End-to-end slab solve with host buffers (bench e2e leg): copies this
    rank's f-hat rows in, runs PCG, forms its nodal rows of u = W w and
    copies them out.  f_host / u_host: lists of pinned host tensors per
    state ((n_w, N_x) and (n_out, N_x), dof layout)."""
    import torch
    F = [to_grid(st, fh.to(st.bufs["U"].device, non_blocking=True))
         for fh, st in zip(f_host, system.states)]
    W = [torch.empty_like(f) for f in F]
    res = pcg(system, F, W, epsilon=epsilon, rtol=rtol, max_iterations=max_iterations)
    system.synthesis(W)
    for st, uh in zip(system.states, u_host):
        uh.copy_(from_grid(st, st.bufs["U"][1:1 + st.lay.n_out]), non_blocking=True)
    torch.cuda.synchronize()
    return res
