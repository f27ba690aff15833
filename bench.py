"""Benchmark: space-time DoF x PCG iterations / s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One step = one full PCG solve of S-hat w = f-hat to rtol 1e-6 (the BASELINE
stopping rule sqrt(r^T K_X r) <= 1e-6 sqrt(f^T K_X f)) with f-hat resident
in HBM.  value = N_dofs * iterations * steps / time (device time, CUDA events,
max over ranks).  `e2e` repeats the measurement through the C ABI's host-
buffer entry point hwg_solve_host: pinned host f-hat -> device, PCG, u = W w,
device -> host, every step.  Inputs are seeded synthetic data of the
BASELINE config's shape and distribution (no dataset exists).

--impl reference times the reference's CPU algorithm -- the oracle port in
oracle/ (C + OpenMP over all host cores; the reference itself is Python +
numba and cannot travel to the GPU box) -- one PCG iteration per step.

N > 1 (torchrun): the workload is partitioned in time slabs across the N
GPUs (paper_2009_08875_b200/distributed.py, SURVEY §8e design (a)): NCCL
halo rows for the temporal bands and wavelet stages, an allgather of the
coarse wavelet levels and of the dot partials; "scaling": "strong" (total
work fixed).  --slab runs the same distributed path at N = 1.

--config 5 (L-shaped domain, N = 6.4e9 dofs, quoted "across 8 B200"): one
GPU cannot hold it, so N GPUs run the per-GPU share of the 8-GPU problem --
the same spatial mesh (N_x = 3,141,633, K = 11 mapped) with J = 8 + log2 N
(N_t = 257 at N = 1; the full cfg 5, J = 11, at N = 8); "scaling": "weak".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2009_08875_b200 import inputs  # noqa: E402
from paper_2009_08875_b200 import discretization as disc  # noqa: E402

METRIC = "space-time DoFs x PCG iters/sec (rtol 1e-6)"
UNIT = "DoF*it/s"


def model_bytes_per_iteration(d, J, K, nu=3, cycles=2):
    """SURVEY.md §8d streaming byte model for one PCG iteration (8 B/word)."""
    n_t = 2 ** J + 1
    sizes = [(2 ** l - 1) ** d for l in range(1, K + 1)]
    n_x = sizes[-1]
    N = n_t * n_x
    wav = 2 * sum(2 ** j + 1 for j in range(1, J + 1)) * n_x
    words = 2 * wav + 3 * N + 3 * N + 2 * N + 13 * N
    mg = 0
    for cyc in range(cycles):
        for l in range(K, 1, -1):
            n, nc = sizes[l - 1], sizes[l - 2]
            zero = (l < K) or cyc == 0
            mg += 3 * nu * n - (n if zero else 0) + 3 * n + (n + nc) + (2 * n + nc) + 3 * nu * n
        mg += 2 * sizes[0]
    words += 4 * n_t * mg
    return 8.0 * words


def impl_bytes_per_iteration(d, J, K, cycles=2):  # grid layout (the L moves its zero quadrant)
    """Algorithmic HBM bytes this implementation moves per PCG iteration
    (no recomputation step): every kernel's compulsory reads + writes, 8 B
    words.  DESIGN.md §5 lists the terms; ncu confirms DRAM traffic = these
    bytes for the dominant kernels (profiles/ncu_traffic_cfg4.json)."""
    n_t = 2 ** J + 1
    size = [(2 ** l - 1) ** d for l in range(0, K + 1)]
    n_x = size[K]
    N = n_t * n_x
    # W: stage j reads 2^(j-1)+1 coarse + 2^(j-1) wavelet rows, writes 2^j + 1;
    # W^T: stage j reads 2^j + 1 rows, writes 2^(j-1)+1 + 2^(j-1).  The top two
    # stages run as one pass (hw_wavelet.cu: the stage J-1 prefix stays in
    # registers), so stage J-1's 2 (2^(J-1) + 1) rows are not moved
    fused_top = J >= 2
    wav = sum(2 * (2 ** j + 1) for j in range(1, J + 1) if not (fused_top and j == J - 1)) * n_x

    def mg_words_per_row():
        if d == 1:
            return 2 * n_x                              # mg1d: read b, write x once
        w = 0
        for cyc in range(cycles):
            for l in range(K, 5, -1):                   # streamed levels, DOWN + UP
                n2, m2 = size[l], size[l - 1]
                zero = l < K or cyc == 0
                w += (2 * n2 + m2) + (0 if zero else n2)   # DOWN: b, x_out, b_c (+ x_in)
                w += 3 * n2 + m2                           # UP: b, x_in, x_c, x_out
            w += 2 * size[min(K, 5)]                    # levels <= 5: read b, write x
        return w

    mg = mg_words_per_row()
    schur = wav + 3 * N + 2 * n_t * mg + 3 * N + wav     # W, B-side, K_x batch, B^T-side, W^T
    kx = 2 * n_t * mg + 2 * N + N                        # C A C (A_x: read, write) + fused r.z
    vec = 2 * N + 3 * N + 5 * N                          # p.q, r -= a q, (w += a p; p = z + b p)
    return 8.0 * (schur + kx + vec)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(cfg, world=1):
    d, J, K, dist, u0 = inputs.recipe(cfg)
    if cfg == 5:                       # per-GPU share of the 8-GPU problem (weak scaling)
        J = 8 + (world.bit_length() - 1)
    n_t = 2 ** J + 1
    n_x = disc.lshape_dofs(K) if domain_of(cfg) == "L" else (2 ** K - 1) ** d
    return d, J, K, dist, u0, n_t, n_x


def domain_of(cfg):
    return inputs.CONFIGS[cfg].get("domain", "square")


def diffusion_of(cfg, d):
    """D of the config (the L is mapped to [0,1]^2 minus [1/2,1]^2: D = I/4)."""
    return 0.25 * np.eye(2) if domain_of(cfg) == "L" else np.eye(d)


def dof_fraction(cfg, d, K, n_x):
    """Algorithmic bytes count the dofs: the L-shaped domain's kernels run on
    the embedded (2^K-1)^2 grid, whose removed quadrant (1/4) carries no
    information -- scale the grid-based byte counts by N_x / (2^K-1)^2."""
    return n_x / (2 ** K - 1) ** d if domain_of(cfg) == "L" else 1.0


def workload_label(cfg, d, J, K, n_t, n_x, world=1):
    if cfg == 5:
        return (f"cfg5: 2D L-shaped heat (mapped, D=I/4), J={J} (N_t={n_t}), K={K} "
                f"(N_x={n_x}), PCG to rtol 1e-6 -- the per-GPU share of cfg 5 on 8 GPUs "
                f"(full cfg 5 is J=11 at N=8)")
    return (f"cfg{cfg}: {d}D heat, J={J} (N_t={n_t}), K={K} (N_x={n_x}), PCG to rtol 1e-6")


def config_dict(cfg, world=1, slab=False):
    """The `config` object of the JSON line -- identical for both arms (the
    reference arm times a bounded sample of this workload, described in its
    cpu_baseline.sample)."""
    d, J, K, dist, u0, n_t, n_x = workload(cfg, world)
    par = "1 GPU" if world == 1 and not slab else (
        f"time slabs x{world} (NCCL halos + allgather)" if world > 1 or slab else "1 GPU")
    return {"workload": workload_label(cfg, d, J, K, n_t, n_x, world), "dofs": n_t * n_x,
            "parallelism": par,
            "l2": "inputs larger than L2 (each solve streams >100 arrays of "
                  f"{8 * n_t * n_x / 1e6:.0f} MB)"}


# --------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference)
# --------------------------------------------------------------------------
def oracle_setup(cfg, fhat=None, max_dofs=4.5e7):
    """Oracle system for the workload (or a reduced-N_t twin with the same
    N_x when the full config does not fit host RAM), its f-hat, and a label."""
    from oracle import heatwave_oracle as O
    d, J, K, dist, u0, n_t, n_x = workload(cfg)
    Jo = J
    while (2 ** Jo + 1) * n_x > max_dofs and Jo > 2:
        Jo -= 1
    system = O.assemble(d, Jo, K, D=diffusion_of(cfg, d), domain=domain_of(cfg))
    nto = 2 ** Jo + 1
    if fhat is not None and Jo == J:
        f = np.ascontiguousarray(fhat)
    else:
        f = system.rhs(inputs.forcing(dist, nto, n_x), u0)
    label = (f"cfg{cfg} full size" if Jo == J else
             f"reduced-N_t twin of cfg{cfg}: J={Jo} (N_t={nto}), same N_x={n_x}")
    return O, system, f, label


def oracle_iterations(O, system, f, iters):
    """Time `iters` PCG iterations of the oracle (solver.py:212-256 body),
    after an untimed setup (r = f, z = K r, p = z)."""
    r = f.copy()
    z = system.kx(r)
    rho = O.dot(r, z)
    p = z.copy()
    w = np.zeros_like(f)
    q = np.empty_like(f)
    times = []
    for _ in range(iters):
        t0 = time.perf_counter()
        q[...] = system.schur(p)
        alpha = rho / O.dot(p, q)
        O.axpy(alpha, p, w)
        O.axpy(-alpha, q, r)
        system.kx(r, z)
        rho_new = O.dot(r, z)
        beta, rho = rho_new / rho, rho_new
        O.xpay(beta, z, p)
        times.append(time.perf_counter() - t0)
    return times


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    from oracle import heatwave_oracle as O
    threads = O.lib().or_num_threads()
    O_, system, f, label = oracle_setup(args.config)
    n = f.size
    oracle_iterations(O_, system, f, args.warmup)
    times = oracle_iterations(O_, system, f, args.steps)
    t = sum(times)
    value = n * args.steps / t
    d, J, K, *_ = workload(args.config)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.config == 5 else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded BASELINE cfg{args.config} recipe)",
        "config": config_dict(args.config, max(args.gpus, 1)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"one step = one PCG iteration of the oracle (oracle/ C+OpenMP, "
                                   f"{threads} threads) on a bounded sample of the workload: "
                                   f"{label} (throughput per DoF is flat in N_t, SURVEY §8d); "
                                   f"{args.steps} timed steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# GPU leg
# --------------------------------------------------------------------------
def run_ours(args):
    import torch
    import paper_2009_08875_b200 as hw

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    d, J, K, dist_name, u0, n_t, n_x = workload(args.config)
    N = n_t * n_x
    problem = hw.ProblemData(D=diffusion_of(args.config, d), c=0.0, u0=u0)
    F = inputs.forcing(dist_name, n_t, n_x)
    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    asm = hw.assemble_system(problem, J, K, hw.SolveConfig(device=local), forcing=F,
                             host_rhs=False, domain=domain_of(args.config))
    torch.cuda.synchronize()
    # assemble_system (solver.py:353-386): context, tables, workspaces, and the
    # GPU right-hand side from the host forcing array (its H2D copy included)
    setup_s = {"assemble_system": time.perf_counter() - t_setup,
               "includes": "ctx/tables/workspaces + H2D of the nodal forcing + GPU f-hat"}
    del F
    ctx = asm.ctx
    f = asm.rhs.f_hat.array
    w = torch.empty_like(f)
    st = torch.cuda.current_stream(dev)

    def solve():
        stats, rc = ctx.pcg(f, w, 0.0, 1e-6, 200, 50)
        if rc != 0:
            raise RuntimeError(f"PCG failed with code {rc}")
        return stats

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    its = None
    for _ in range(args.warmup):
        its = solve()["iterations"]
    torch.cuda.synchronize()
    barrier()
    launches0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier()
        e0.record(st)
        its_list = [solve()["iterations"] for _ in range(args.steps)]
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = ctx.launches - launches0
    # per-kernel-class device times for the roofline: one more (untimed)
    # solve with CUDA events around every multigrid launch (the events cost
    # ~4 % at cfg 2, so they stay out of the timed region above)
    ctx.profile_enable(True)
    prof_its = solve()["iterations"]
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    barrier()
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_max = float(t.item())
    total_its = sum(its_list)
    value = N * total_its * world / (ms_max / 1e3)

    # roofline of the dominant kernel class (from the profiled solve)
    peak, peak_src = measured_peaks()
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dname, (dms, dbytes, dn) = dom
    dof_frac = dof_fraction(args.config, d, K, n_x)
    dbytes *= dof_frac
    achieved = dbytes / (dms / 1e3) / 1e9 if dms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            rec = json.load(fh).get(dname)
        if rec:   # measured dram bytes / algorithmic bytes, scaled to this run's launches
            traffic = rec["traffic_over_algorithmic"] * dbytes / max(dn, 1)
    model = model_bytes_per_iteration(d, J, K) * dof_frac
    impl_b = impl_bytes_per_iteration(d, J, K) * dof_frac
    it_s = (ms_max / 1e3) / total_its

    # end-to-end through the C ABI with host buffers
    fh = torch.empty((n_t, n_x), dtype=torch.float64, pin_memory=True)
    fh.copy_(f)
    uh = torch.empty((n_t, n_x), dtype=torch.float64, pin_memory=True)
    fh_np, uh_np = fh.numpy(), uh.numpy()
    ctx.solve_host(fh_np, uh_np, 0.0, 1e-6)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    e2e_its = 0
    for _ in range(args.steps):
        s, rc = ctx.solve_host(fh_np, uh_np, 0.0, 1e-6)
        if rc != 0:
            raise RuntimeError(f"solve_host failed with code {rc}")
        e2e_its += s["iterations"]
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = N * e2e_its * world / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import heatwave_oracle as O
        O_, system, fo, label = oracle_setup(args.config, fhat=f.cpu().numpy())
        n_iter = args.cpu_iterations
        times = oracle_iterations(O_, system, fo, n_iter)
        cpu = {"value": fo.size * n_iter / sum(times), "unit": UNIT,
               "cores": O.lib().or_num_threads(), "kind": "port",
               "sample": f"{n_iter} PCG iterations of the oracle (oracle/ C+OpenMP), {label}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak" if args.config == 5 else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded BASELINE cfg{args.config} recipe: {dist_name} nodal "
                    "forcing, blockwise-seeded)",
            "config": config_dict(args.config, world),
            "iterations_per_solve": its_list[0],
            "time_to_solve_s": ms_max / 1e3 / args.steps,
            "setup_s": setup_s,
            "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "launches": dn, "bytes_per_launch": dbytes / max(dn, 1),
                         "peak_source": peak_src,
                         **({"note": "mg1d is FP64-issue/latency-bound, not HBM-bound: ncu has the FP64 "
                                     "pipe 45 % busy and DRAM 14 % (profiles/r02/ncu_mg1d_rrp.txt); its "
                                     "16 B/point of traffic is the compulsory minimum"}
                            if dname == "mg1d" else {})},
            "roofline_iteration": {"bytes_per_iteration": impl_b, "s_per_iteration": it_s,
                                   "achieved_GBs": impl_b / it_s / 1e9, "peak": peak,
                                   "frac": impl_b / it_s / 1e9 / peak,
                                   "frac_vs_nominal_8TBs": impl_b / it_s / 8e12,
                                   "source": "algorithmic bytes of this implementation's "
                                             "kernels per PCG iteration (bench.impl_bytes_per_iteration)"},
            "roofline_model": {"bytes_per_iteration": model, "s_per_iteration": it_s,
                               "achieved_GBs": model / it_s / 1e9,
                               "frac": model / it_s / 1e9 / peak,
                               "source": "SURVEY.md §8d streaming model (one pass per smoothing "
                                         "sweep; the kernels here fuse sweeps, so frac > 1)"},
            "kernel_classes_ms": {k: v[0] for k, v in prof.items()},
            "kernel_classes_source": f"one extra profiled solve ({prof_its} iterations), "
                                     "CUDA events around every multigrid launch",
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * N,
                    "d2h_bytes_per_step": 8 * N, "time_to_solve_s": e2e_s / args.steps},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_slab(args):
    """Time-slab distributed solve over N GPUs (strong scaling)."""
    import torch
    import torch.distributed as tdist
    from paper_2009_08875_b200 import distributed as D
    from paper_2009_08875_b200 import discretization as disc

    rank, world, local = dist_env()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tdist.init_process_group("nccl", device_id=dev)
    d, J, K, dist_name, u0, n_t, n_x = workload(args.config, world)
    N = n_t * n_x
    domain = domain_of(args.config)
    torch.cuda.synchronize()
    t_setup0 = time.perf_counter()
    states = D.make_states(d, J, K, world, [rank], lambda p: dev, D=diffusion_of(args.config, d),
                           domain=domain)
    system = D.SlabSystem(states, D.TorchComm())
    st = states[0]
    lay = st.lay

    def frows(a, b):
        return torch.from_numpy(inputs.forcing_rows(dist_name, n_t, n_x, a, b)).to(dev)

    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    u0p = torch.from_numpy(disc.project_initial(disc.FineMesh(d, K, domain), u0)).to(dev)
    F = D.rhs(system, frows, u0p)
    torch.cuda.synchronize()
    setup_s = {"assemble_system": time.perf_counter() - t_setup0, "rhs": time.perf_counter() - t_setup,
               "includes": "rank contexts + forcing rows generated on the host + H2D + "
                           "distributed GPU f-hat"}
    W = [torch.empty_like(F[0])]

    def solve():
        return D.pcg(system, F, W, rtol=1e-6).iterations

    for _ in range(args.warmup):
        solve()
    ctx = st.k.ctx
    torch.cuda.synchronize()
    tdist.barrier()
    launches0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        tdist.barrier()
        e0.record()
        its_list = [solve() for _ in range(args.steps)]
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = ctx.launches - launches0
    ctx.profile_enable(True)                 # per-class times: one extra, untimed solve
    solve()
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    t = torch.tensor([ms], device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_its = sum(its_list)
    value = N * total_its / (ms_max / 1e3)

    # e2e: pinned host f-hat rows in, u rows out, every step
    Fd = D.from_grid(st, F[0])                       # the user-facing (dof-layout) f-hat rows
    fh = [torch.empty(Fd.shape, dtype=torch.float64, pin_memory=True)]
    fh[0].copy_(Fd)
    uh = [torch.empty((lay.n_out, n_x), dtype=torch.float64, pin_memory=True)]
    D.solve_host(system, fh, uh)
    tdist.barrier()
    t0 = time.perf_counter()
    e2e_its = 0
    for _ in range(args.steps):
        e2e_its += D.solve_host(system, fh, uh).iterations
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    e2e_s = float(t.item())

    peak, peak_src = measured_peaks()
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dname, (dms, dbytes, dn) = dom
    dof_frac = dof_fraction(args.config, d, K, n_x)
    dbytes *= dof_frac
    achieved = dbytes / (dms / 1e3) / 1e9 if dms > 0 else 0.0
    model = model_bytes_per_iteration(d, J, K) * dof_frac
    impl_b = impl_bytes_per_iteration(d, J, K) * dof_frac
    it_s = (ms_max / 1e3) / total_its
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak" if args.config == 5 else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE recipe, blockwise-seeded forcing rows)",
            "config": config_dict(args.config, world, slab=True),
            "iterations_per_solve": its_list[0],
            "time_to_solve_s": ms_max / 1e3 / args.steps,
            "setup_s": setup_s,
            "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                         "launches": dn, "bytes_per_launch": dbytes / max(dn, 1),
                         "peak_source": peak_src, "rank": 0},
            "roofline_iteration": {"bytes_per_iteration": impl_b, "s_per_iteration": it_s,
                                   "achieved_GBs": impl_b / it_s / 1e9, "peak": peak * world,
                                   "frac": impl_b / it_s / 1e9 / (peak * world),
                                   "frac_vs_nominal_8TBs": impl_b / it_s / (8e12 * world),
                                   "source": "algorithmic bytes per PCG iteration, aggregate "
                                             "over GPUs"},
            "roofline_model": {"bytes_per_iteration": model, "s_per_iteration": it_s,
                               "achieved_GBs": model / it_s / 1e9,
                               "frac": model / it_s / 1e9 / (peak * world),
                               "source": "SURVEY.md §8d streaming model, aggregate over GPUs"},
            "kernel_classes_ms": {k: v[0] for k, v in prof.items()},
            "e2e": {"value": N * e2e_its / e2e_s, "unit": UNIT, "h2d_bytes_per_step":
                    8 * n_x * sum(D.slab_layout(J, world, q).n_w for q in range(world)),
                    "d2h_bytes_per_step": 8 * N, "time_to_solve_s": e2e_s / args.steps},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    tdist.barrier()
    tdist.destroy_process_group()
    return 0


def launcher_command(argv, n, port):
    """torchrun command that re-runs this script as n ranks (one per GPU)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__), *argv]


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=(1, 2, 3, 4, 5))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--cpu-iterations", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slab", action="store_true", help="time-slab path even at N = 1")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "0")) or None
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference(args)            # rank 0 only; other ranks exit 0
    if world is None and args.gpus > 1:
        # one process per GPU: re-launch this script under torchrun
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) "
                  "are visible", file=sys.stderr)
            return 2
        return subprocess.call(launcher_command(sys.argv[1:], args.gpus, _free_port()))
    if world is not None and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.slab or (world or 1) > 1:
        return run_slab(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
