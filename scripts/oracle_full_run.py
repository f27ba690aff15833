"""One-off full-size parity run: the CPU oracle (C + OpenMP, pinned bit-exact
to the reference's own fixtures) solves a BASELINE config at FULL size on the
GPU box's host (16 threads, 196 GB RAM), then the GPU solves the same seeded
problem and the two are compared on the FULL arrays.

    python scripts/oracle_full_run.py --config 4 --out gpurun_out/cfg4full

Writes <out>.json (iterations, residual history, CG scalars, norms, the
full-array GPU-vs-oracle differences) and <out>.npz (65,536 seeded sample
positions of f-hat, w, u) -- committed as tests/golden/cfg4full.* and checked
by tests/test_gpu_parity.py::test_bench_config_against_full_oracle_run.

The reference itself cannot run here (it needs ~185 GB at 1.07e9 dofs and
does not travel to the box); the oracle restates it in the same arithmetic
order and is pinned to reference fixtures at every kernel (SURVEY.md §7
"oracle reach").  Test infrastructure: nothing here is on the product path.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2009_08875_b200 import inputs  # noqa: E402

NSAMPLE = 65536
SAMPLE_SEED = 7


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def oracle_solve(d, J, K, dist, u0, D=None, domain="square"):
    from oracle import heatwave_oracle as O
    O.build()
    system = O.assemble(d, J, K, D=D, domain=domain)
    n_t, n_x = system.shape
    log(f"oracle assembled: n_t={n_t} n_x={n_x} threads={O.lib().or_num_threads()}")
    t0 = time.perf_counter()
    F = inputs.forcing(dist, n_t, n_x)
    f = system.rhs(F, u0)
    del F
    gc.collect()
    log(f"oracle f-hat: {time.perf_counter() - t0:.1f} s")
    t1 = time.perf_counter()
    z = system.kx(f)
    rho0 = O.dot(f, z)
    del z
    eps = 1e-6 * np.sqrt(rho0)
    log(f"oracle rho0={rho0!r} eps={eps!r}")

    # the oracle's pcg with per-iteration progress (same body as O.pcg)
    import math
    w = np.zeros_like(f)
    r = f.copy()
    z = system.kx(r)
    rho = O.dot(r, z)
    hist = [math.sqrt(max(rho, 0.0))]
    alphas, betas = [], []
    p = z.copy()
    q = np.empty_like(f)
    its = 0
    for k in range(1, 201):
        q[...] = system.schur(p)
        pq = O.dot(p, q)
        alpha = rho / pq
        O.axpy(alpha, p, w)
        O.axpy(-alpha, q, r)                 # recompute_every = 50 > iterations here
        system.kx(r, z)
        rho_new = O.dot(r, z)
        beta = rho_new / rho
        alphas.append(alpha)
        betas.append(beta)
        rho = rho_new
        hist.append(math.sqrt(max(rho, 0.0)))
        its = k
        log(f"oracle it {k}: sqrt(rho)={hist[-1]:.6e} ({time.perf_counter() - t1:.0f} s)")
        if rho <= eps ** 2:
            break
        O.xpay(beta, z, p)
    secs = time.perf_counter() - t1
    del r, z, p, q
    system.bufs.clear()
    gc.collect()
    u = system.wavelet.apply(w)
    return dict(f=f, w=w, u=u, its=its, hist=hist, alphas=alphas, betas=betas, eps=eps,
                rho0=rho0, seconds=secs, threads=O.lib().or_num_threads())


def gpu_solve_and_compare(cfg, d, J, K, dist, u0, ref, D=None, domain="square"):
    import torch
    import paper_2009_08875_b200 as hw
    n_t = 2 ** J + 1
    F = inputs.forcing(dist, n_t, ref["f"].shape[1])
    prob = hw.ProblemData(D=np.eye(d) if D is None else D, c=0.0, u0=u0)
    asm = hw.assemble_system(prob, J, K, hw.SolveConfig(), forcing=F, host_rhs=False,
                             domain=domain)
    del F
    gc.collect()
    f = asm.rhs.f_hat.array

    def rel_full(dev, host):
        h = torch.from_numpy(host).to(dev.device)
        rel = float(torch.linalg.norm(dev - h) / torch.linalg.norm(h))
        del h
        torch.cuda.empty_cache()
        return rel

    out = {"rel_l2_fhat_full": rel_full(f, ref["f"])}
    res = hw.pcg(asm.S, asm.K_X, hw.SpaceTimeVector(f), 0.0, rtol=1e-6)
    out["gpu_iterations"] = res.iterations
    out["gpu_residual_norms"] = list(map(float, res.residual_norms))
    w = res.w.array
    out["rel_l2_w_full"] = rel_full(w, ref["w"])
    u = asm.wavelet.apply_array(w)
    out["rel_l2_u_full"] = rel_full(u, ref["u"])
    h = np.array(ref["hist"])
    g = np.array(out["gpu_residual_norms"])
    if len(g) == len(h):
        out["residual_history_max_rel_diff"] = float(np.abs(g - h).max() / h.max())
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--out", default="gpurun_out/cfg4full")
    ap.add_argument("--no-gpu", action="store_true")
    ap.add_argument("--J", type=int, default=None, help="override J (cfg 5: the per-GPU share)")
    args = ap.parse_args()
    d, J, K, dist, u0 = inputs.recipe(args.config)
    if args.J is not None:
        J = args.J
    domain = inputs.CONFIGS[args.config].get("domain", "square")
    D = 0.25 * np.eye(2) if domain == "L" else None       # the mapped L (discretization.lshape_problem)
    t0 = time.time()
    ref = oracle_solve(d, J, K, dist, u0, D=D, domain=domain)
    n_t, n_x = ref["f"].shape
    log(f"oracle done: {ref['its']} iterations, {ref['seconds']:.0f} s")
    idx = np.sort(np.random.default_rng(SAMPLE_SEED).choice(n_t * n_x, min(NSAMPLE, n_t * n_x), replace=False))
    meta = dict(name=os.path.basename(args.out), config=args.config, d=d, J=J, K=K, dist=dist,
                domain=domain, D=(np.eye(d) if D is None else D).tolist(),
                n_t=n_t, n_x=n_x, seed_f=inputs.SEED_F, sample_seed=SAMPLE_SEED,
                iterations=ref["its"], eps=ref["eps"], rho0=ref["rho0"],
                residual_norms=ref["hist"], cg_alphas=ref["alphas"], cg_betas=ref["betas"],
                fhat_norm=float(np.linalg.norm(ref["f"])), w_norm=float(np.linalg.norm(ref["w"])),
                u_norm=float(np.linalg.norm(ref["u"])),
                u_last_row_norm=float(np.linalg.norm(ref["u"][-1])),
                oracle_seconds=ref["seconds"], oracle_threads=ref["threads"],
                source="oracle/ C+OpenMP restatement of the reference (pinned bit-exact to "
                       "reference-generated fixtures), full size, scripts/oracle_full_run.py")
    np.savez_compressed(args.out + ".npz", sample_idx=idx,
                        fhat_sample=ref["f"].reshape(-1)[idx], w_sample=ref["w"].reshape(-1)[idx],
                        u_sample=ref["u"].reshape(-1)[idx])
    with open(args.out + ".json", "w") as fh:
        json.dump(meta, fh, indent=1)
    if not args.no_gpu:
        cmp = gpu_solve_and_compare(args.config, d, J, K, dist, u0, ref, D=D, domain=domain)
        meta["gpu_comparison"] = cmp
        log(f"gpu: {cmp}")
        with open(args.out + ".json", "w") as fh:
            json.dump(meta, fh, indent=1)
    meta["wall_s"] = time.time() - t0
    with open(args.out + ".json", "w") as fh:
        json.dump(meta, fh, indent=1)
    print(json.dumps({k: meta[k] for k in ("iterations", "u_norm", "wall_s")} |
                     meta.get("gpu_comparison", {})))


if __name__ == "__main__":
    main()
