"""Time-slab distribution: layout properties, the SPMD
orchestration against the CPU oracle (bit-for-bit) with simulated ranks and
with a real 2-rank gloo process group, and (GPU) P virtual ranks on one
device against the single-GPU solver."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from paper_2009_08875_b200 import distributed as D
from paper_2009_08875_b200 import inputs


@pytest.mark.parametrize("J,P", [(3, 1), (3, 2), (3, 4), (4, 8), (8, 4), (10, 8)])
def test_layout_partitions_rows(J, P):
    n_t = 2 ** J + 1
    owned_rows = []
    for p in range(P):
        lay = D.slab_layout(J, P, p)
        assert lay.n_w == P + lay.H
        assert len(lay.global_rows) == lay.n_w
        owned_rows.extend(lay.global_rows[lay.owned].tolist())
        assert set(range(P + 1)) <= set(lay.global_rows.tolist())     # replicated coarse rows
        for j, (off, n) in lay.block.items():
            g = lay.global_rows[off:off + n]
            assert np.all(lay.level_of[off:off + n] == j)
            # wavelets centred in the slab [p/P, (p+1)/P)
            k = g - 2 ** (j - 1) - 1
            centre = (2 * k + 1) / 2 ** j
            assert np.all((centre >= p / P) & (centre < (p + 1) / P))
    assert sorted(owned_rows) == list(range(n_t))


def test_layout_rejects_bad_P():
    with pytest.raises(ValueError):
        D.slab_layout(4, 3, 0)
    with pytest.raises(ValueError):
        D.slab_layout(3, 8, 0)


def _oracle_case(d, J, K, dist="uniform", domain="square"):
    from oracle import heatwave_oracle as O
    if domain == "L":
        system = O.assemble(d, J, K, D=0.25 * np.eye(2), domain="L")
    else:
        system = O.assemble(d, J, K)
    n_t, n_x = system.shape
    u0 = inputs.u0_sines if dist in ("uniform", "lshape") else inputs.u0_modes()
    f = system.rhs(inputs.forcing(dist, n_t, n_x), u0)
    eps = 1e-6 * np.sqrt(O.dot(f, system.kx(f)))
    ref = O.pcg(system, f, eps)
    return O, system, f, eps, ref


def _run_slabs(system, f, eps, P, comm, ranks):
    from slab_numpy import NumpyKernels
    n_x = system.shape[1]
    J = system.J
    states = [D.RankState(D.slab_layout(J, P, p), NumpyKernels(system), n_x, "cpu")
              for p in ranks]
    ft = torch.from_numpy(f)
    F = [D.scatter_wavelet(ft, st.lay).clone() for st in states]
    W = [torch.zeros_like(x) for x in F]
    res = D.pcg(D.SlabSystem(states, comm), F, W, epsilon=eps)
    return states, W, res


@pytest.mark.parametrize("d,J,K,P", [(2, 4, 4, 2), (2, 4, 4, 4), (2, 4, 4, 8), (1, 6, 6, 4),
                                     (2, 3, 5, 2)])
def test_simulated_ranks_match_oracle_bitwise(d, J, K, P):
    O, system, f, eps, ref = _oracle_case(d, J, K, "uniform" if d == 2 else "normal")
    states, W, res = _run_slabs(system, f, eps, P, D.SimComm(P), range(P))
    assert res.iterations == ref.iterations
    assert res.residual_norms == ref.residual_norms
    w = D.gather_wavelet([x.numpy() for x in W], [st.lay for st in states], np.zeros_like(f))
    assert np.array_equal(w, ref.w)
    # replicated coarse rows are identical on every rank
    for st, x in zip(states, W):
        assert np.array_equal(x[:P + 1].numpy(), ref.w[:P + 1])


@pytest.mark.parametrize("J,K,P", [(3, 4, 2), (4, 5, 4)])
def test_simulated_ranks_lshape_match_oracle_bitwise(J, K, P):
    """The L-shaped domain (BASELINE cfg 5) over time slabs: bit-identical
    to the oracle's single-process PCG."""
    O, system, f, eps, ref = _oracle_case(2, J, K, "lshape", domain="L")
    states, W, res = _run_slabs(system, f, eps, P, D.SimComm(P), range(P))
    assert res.iterations == ref.iterations
    w = D.gather_wavelet([x.numpy() for x in W], [st.lay for st in states], np.zeros_like(f))
    assert np.array_equal(w, ref.w)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, outdir, d, J, K, domain="square"):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        O, system, f, eps, ref = _oracle_case(d, J, K, "lshape" if domain == "L" else "uniform",
                                              domain=domain)
        states, W, res = _run_slabs(system, f, eps, world, D.TorchComm(), [rank])
        np.save(os.path.join(outdir, f"w{rank}.npy"), W[0].numpy())
        np.save(os.path.join(outdir, f"its{rank}.npy"), np.array([res.iterations]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,domain", [(2, "square"), (2, "L")])
def test_gloo_two_ranks_match_oracle_bitwise(world, domain):
    d, J, K = 2, 4, 4
    port = _free_port()
    with tempfile.TemporaryDirectory() as tmp:
        torch.multiprocessing.spawn(_gloo_worker, args=(world, port, tmp, d, J, K, domain),
                                    nprocs=world, join=True)
        O, system, f, eps, ref = _oracle_case(d, J, K, "lshape" if domain == "L" else "uniform",
                                              domain=domain)
        parts = [np.load(os.path.join(tmp, f"w{r}.npy")) for r in range(world)]
        its = [int(np.load(os.path.join(tmp, f"its{r}.npy"))[0]) for r in range(world)]
    assert its == [ref.iterations] * world
    lays = [D.slab_layout(J, world, p) for p in range(world)]
    w = D.gather_wavelet(parts, lays, np.zeros_like(f))
    assert np.array_equal(w, ref.w)


# ---------------------------------------------------------------------------
# GPU: P virtual ranks on one device vs the single-GPU solver
# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("d,J,K,Ps", [(2, 4, 4, (1, 2, 4, 8)), (2, 3, 6, (1, 2, 4)),
                                      (1, 6, 6, (2, 4)), (2, 8, 8, (1, 4))])
def test_gpu_virtual_ranks_match_single_gpu(d, J, K, Ps):
    import paper_2009_08875_b200 as hw
    dist_name = "uniform" if d == 2 else "normal"
    u0 = inputs.u0_sines if d == 2 else inputs.u0_modes()
    n_t, n_x = 2 ** J + 1, (2 ** K - 1) ** d
    F = inputs.forcing(dist_name, n_t, n_x)
    asm = hw.assemble_system(hw.ProblemData(D=np.eye(d), c=0.0, u0=u0), J, K, hw.SolveConfig(),
                             forcing=F, host_rhs=False)
    f = asm.rhs.f_hat.array
    w1 = torch.empty_like(f)
    stats, rc = asm.ctx.pcg(f, w1, 0.0, 1e-6)
    assert rc == 0
    dev = torch.device("cuda", 0)
    for P in Ps:
        states = D.make_states(d, J, K, P, range(P), lambda p: dev)
        Fl = [D.scatter_wavelet(f, st.lay).clone() for st in states]
        Wl = [torch.zeros_like(x) for x in Fl]
        res = D.pcg(D.SlabSystem(states, D.SimComm(P)), Fl, Wl, rtol=1e-6)
        assert res.iterations == stats["iterations"], P
        w = D.gather_wavelet(Wl, [st.lay for st in states], torch.zeros_like(f))
        assert torch.equal(w, w1), (P, float((w - w1).abs().max()))


@pytest.mark.parametrize("P", [2, 4])
def test_simulated_rhs_matches_oracle_bitwise(P):
    from oracle import heatwave_oracle as O
    from slab_numpy import NumpyKernels
    d, J, K = 2, 4, 4
    system = O.assemble(d, J, K)
    n_t, n_x = system.shape
    F = inputs.forcing("uniform", n_t, n_x)
    want = system.rhs(F, inputs.u0_sines)
    u0p = torch.from_numpy(O.project_initial(system.finest, inputs.u0_sines))
    states = [D.RankState(D.slab_layout(J, P, p), NumpyKernels(system), n_x, "cpu")
              for p in range(P)]
    sysd = D.SlabSystem(states, D.SimComm(P))
    parts = D.rhs(sysd, lambda a, b: torch.from_numpy(F[a:b].copy()), u0p)
    got = D.gather_wavelet([x.numpy() for x in parts], [st.lay for st in states], np.zeros_like(want))
    assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("d,J,K,P", [(2, 4, 4, 4), (2, 8, 8, 4), (1, 6, 6, 2)])
def test_gpu_virtual_ranks_rhs(d, J, K, P):
    import paper_2009_08875_b200 as hw
    from paper_2009_08875_b200 import discretization as disc
    dist_name = "uniform" if d == 2 else "normal"
    u0 = inputs.u0_sines if d == 2 else inputs.u0_modes()
    n_t, n_x = 2 ** J + 1, (2 ** K - 1) ** d
    F = inputs.forcing(dist_name, n_t, n_x)
    asm = hw.assemble_system(hw.ProblemData(D=np.eye(d), c=0.0, u0=u0), J, K, hw.SolveConfig(),
                             forcing=F, host_rhs=False)
    dev = torch.device("cuda", 0)
    states = D.make_states(d, J, K, P, range(P), lambda p: dev)
    u0p = torch.from_numpy(disc.project_initial(disc.FineMesh(d, K), u0)).to(dev)
    Ft = torch.from_numpy(F).to(dev)
    parts = D.rhs(D.SlabSystem(states, D.SimComm(P)), lambda a, b: Ft[a:b], u0p)
    got = D.gather_wavelet(parts, [st.lay for st in states], torch.zeros_like(asm.rhs.f_hat.array))
    assert torch.equal(got, asm.rhs.f_hat.array)


@pytest.mark.gpu
@pytest.mark.parametrize("J,K,Ps", [(3, 5, (2, 4)), (4, 7, (1, 4)), (4, 11, (2,))])
def test_gpu_virtual_ranks_lshape(J, K, Ps):
    """L-shaped domain: P virtual ranks (grid layout, dof-layout RHS inputs)
    reproduce the single-GPU solve bit for bit -- f-hat and w."""
    import paper_2009_08875_b200 as hw
    from paper_2009_08875_b200 import discretization as disc
    prob = hw.lshape_problem(u0=inputs.u0_sines)
    n_t = 2 ** J + 1
    n_x = disc.lshape_dofs(K)
    F = inputs.forcing("lshape", n_t, n_x)
    asm = hw.assemble_system(prob, J, K, hw.SolveConfig(), forcing=F, host_rhs=False, domain="L")
    ctx = asm.ctx
    f = asm.rhs.f_hat.array
    w1 = torch.empty_like(f)
    stats, rc = ctx.pcg(f, w1, 0.0, 1e-6)
    assert rc == 0
    fg = torch.empty((n_t, ctx.n_grid), dtype=torch.float64, device="cuda")
    ctx.grid_scatter(f, fg)
    dev = torch.device("cuda", 0)
    u0p = torch.from_numpy(disc.project_initial(disc.FineMesh(2, K, "L"), prob.u0)).to(dev)
    Ft = torch.from_numpy(F).to(dev)
    for P in Ps:
        states = D.make_states(2, J, K, P, range(P), lambda p: dev, D=0.25 * np.eye(2),
                               domain="L")
        system = D.SlabSystem(states, D.SimComm(P))
        parts = D.rhs(system, lambda a, b: Ft[a:b], u0p)
        got = D.gather_wavelet(parts, [st.lay for st in states], torch.zeros_like(fg))
        assert torch.equal(got, fg), P
        Wl = [torch.zeros_like(x) for x in parts]
        res = D.pcg(system, parts, Wl, rtol=1e-6)
        assert res.iterations == stats["iterations"], P
        wg = D.gather_wavelet(Wl, [st.lay for st in states], torch.zeros_like(fg))
        w = torch.empty_like(w1)
        ctx.grid_gather(wg, w)
        assert torch.equal(w, w1), (P, float((w - w1).abs().max()))


@pytest.mark.gpu
@pytest.mark.parametrize("d,J,K", [(2, 6, 7), (2, 4, 10)])
def test_nccl_world1_slab_matches_hwg_pcg(d, J, K):
    """The time-slab solver under a real NCCL process group of one rank (the
    bench's --slab / torchrun path at N = 1): device-resident scalars, the
    iteration replayed as a CUDA graph, bit-identical to the single-GPU
    hwg_pcg (same kernels, same reduction tree)."""
    import torch.distributed as dist
    import paper_2009_08875_b200 as hw
    n_t, n_x = 2 ** J + 1, (2 ** K - 1) ** d
    F = inputs.forcing("uniform", n_t, n_x)
    asm = hw.assemble_system(hw.ProblemData(D=np.eye(d), c=0.0, u0=inputs.u0_sines), J, K,
                             hw.SolveConfig(), forcing=F, host_rhs=False)
    f = asm.rhs.f_hat.array
    w1 = torch.empty_like(f)
    stats, rc = asm.ctx.pcg(f, w1, 0.0, 1e-6)
    assert rc == 0
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0,
                            world_size=1, device_id=dev)
    try:
        states = D.make_states(d, J, K, 1, [0], lambda p: dev)
        system = D.SlabSystem(states, D.TorchComm())
        assert system.capturable
        Fl = [D.scatter_wavelet(f, states[0].lay).clone()]
        Wl = [torch.zeros_like(Fl[0])]
        res = D.pcg(system, Fl, Wl, rtol=1e-6)
        assert res.iterations == stats["iterations"]
        assert res.residual_norms == stats["residual_norms"]
        w = D.gather_wavelet(Wl, [states[0].lay], torch.zeros_like(f))
        assert torch.equal(w, w1)
        # plain launches give the same iterates as the graph replays
        Wl2 = [torch.zeros_like(Fl[0])]
        res2 = D.pcg(system, Fl, Wl2, rtol=1e-6, graphs=False)
        assert res2.residual_norms == res.residual_norms and torch.equal(Wl2[0], Wl[0])
    finally:
        dist.destroy_process_group()


def test_slab_zero_rhs_uses_any_nonzero():
    """A right-hand side whose squared norm underflows to zero is still
    non-zero (np.any(f), solver.py:196-198): the slab solver iterates."""
    from slab_numpy import NumpyKernels
    from oracle import heatwave_oracle as O
    system = O.assemble(2, 3, 3)
    n_t, n_x = system.shape
    f = np.zeros((n_t, n_x))
    f[3, 4] = 1e-170                         # f.f = 1e-340 -> 0.0 in fp64
    assert O.dot(f, f) == 0.0 and np.any(f)
    states = [D.RankState(D.slab_layout(3, 2, p), NumpyKernels(system), n_x, "cpu")
              for p in range(2)]
    sysd = D.SlabSystem(states, D.SimComm(2))
    F = [D.scatter_wavelet(torch.from_numpy(f), st.lay).clone() for st in states]
    assert sysd.any_nonzero(F)
    Z = [torch.zeros_like(x) for x in F]
    assert not sysd.any_nonzero(Z)
    res = D.pcg(sysd, Z, [torch.zeros_like(x) for x in F], epsilon=1e-6)
    assert res.iterations == 0 and res.residual_norms == [0.0]
