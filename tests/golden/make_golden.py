"""Generate the golden fixtures in this directory from the REFERENCE package.

Run here (not on the GPU box; /root/reference does not travel):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [case ...]

Every array below is produced by the reference's own public functions
(``heatwave.assemble_system``, ``SchurOperator.apply_array``,
``PreconditionerKX.apply_array``, ``WaveletTransform.*``,
``MultigridSolver.apply_rows``, ``pcg``).  The forcing part of f-hat follows
``assemble_rhs`` (/root/reference/pkg/src/heatwave/system.py:295-324) with the
load ``(N (x) M_x) F`` of the P1 x P1 interpolant of the nodal forcing F
(SURVEY.md §8d); ``check_interpolant_load`` pins that identity against
``assemble_load`` (spatial.py:269-300) with an interpolating callable.

Inputs come from ``paper_2009_08875_b200.inputs`` (seeded, blockwise), so the
GPU box regenerates them bit-for-bit and only outputs are stored.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import heatwave as hw  # noqa: E402  (the reference)
from heatwave import system as hw_system  # noqa: E402
from heatwave.solver import _dot, ParallelPlan  # noqa: E402

from paper_2009_08875_b200 import inputs  # noqa: E402

PROBE_SEED = 7


def problem_for(d, dist, D=None, c=0.0, u0=None):
    if u0 is None:
        u0 = inputs.u0_for(dist)
    return hw.ProblemData(D=np.eye(d) if D is None else np.asarray(D, dtype=float), c=c, u0=u0)


def lshape_hierarchy(K):
    """Reference ``Mesh`` / ``MeshHierarchy`` objects of the mapped L-shaped
    domain [0,1]^2 minus [1/2,1]^2, levels 2..K.

    The reference builds only the cube (spatial.py:98-137); this is its
    square mesh (same vertex list, same element order) with the cells of the
    removed quadrant dropped and the closed quadrant's vertices on the
    boundary.  Everything downstream -- assemble_spatial, _build_prolongation,
    make_solver (dense inverse of the 5-dof level 2), the Schur operator,
    K_X, assemble_rhs, pcg -- is the reference's own code."""
    from heatwave.spatial import Mesh, MeshHierarchy, _build_prolongation
    levels = []
    for k in range(2, K + 1):
        m = 2 ** k
        g = np.arange(m + 1)
        X, Y = np.meshgrid(g, g, indexing="ij")
        verts = np.stack([X.ravel(), Y.ravel()], axis=1).astype(float) / m
        i, j = (a.ravel() for a in np.meshgrid(g[:-1], g[:-1], indexing="ij"))
        keep = ~((i >= m // 2) & (j >= m // 2))
        i, j = i[keep], j[keep]
        vid = lambda a, b: a * (m + 1) + b  # noqa: E731
        t1 = np.stack([vid(i, j), vid(i + 1, j), vid(i + 1, j + 1)], axis=1)
        t2 = np.stack([vid(i, j), vid(i + 1, j + 1), vid(i, j + 1)], axis=1)
        grid = np.rint(verts * m).astype(int)
        inner = np.all((grid > 0) & (grid < m), axis=1) & ~np.all(grid >= m // 2, axis=1)
        interior = np.where(inner)[0]
        index = np.full(len(verts), -1, dtype=np.int64)
        index[interior] = np.arange(len(interior))
        levels.append(Mesh(d=2, level=k, vertices=verts, elements=np.concatenate([t1, t2]),
                           interior=interior, interior_index=index))
    prols = [_build_prolongation(levels[q - 1], levels[q]) for q in range(1, len(levels))]
    return MeshHierarchy(d=2, K=len(levels), levels=levels, prolongations=prols)


def assemble_reference(problem, J, K, domain="square"):
    """hw.assemble_system; for the L-shaped domain the reference's own
    assemble_system runs with build_mesh_hierarchy swapped for
    lshape_hierarchy (its only mesh-dependent call, solver.py:360)."""
    if domain == "square":
        return hw.assemble_system(problem, J, K, hw.SolveConfig())
    import heatwave.solver as hws
    orig = hws.build_mesh_hierarchy
    hws.build_mesh_hierarchy = lambda d, k: lshape_hierarchy(k)
    try:
        return hw.assemble_system(problem, J, K, hw.SolveConfig())
    finally:
        hws.build_mesh_hierarchy = orig


def stencil_table(asm, problem):
    """Per-level (A, M) stencil values read from the reference's CSR."""
    out = []
    for ops in hw.assemble_level_operators(asm.hierarchy, problem.D, problem.c):
        A = ops.A_x.to_scipy().tocsr()
        M = ops.M_x.to_scipy().tocsr()
        n = A.shape[0]
        r = n // 2
        out.append(dict(n=n,
                        A_off=(A[r].indices - r).tolist(), A=A[r].data.tolist(),
                        M_off=(M[r].indices - r).tolist(), M=M[r].data.tolist()))
    return out


def forcing_part(asm, F):
    """g-part of f-hat from nodal forcing F via the reference's functions."""
    n_t, n_x = F.shape
    y = np.empty((asm.test.N.rows, n_x))
    tmp = np.empty_like(y)
    hw_system._spatial(asm.spatial.M_x, F, tmp[:n_t], None)
    hw_system._temporal(asm.test.N, tmp[:n_t], y, None)
    ky = hw.apply_KY(asm.spatial, asm.test, asm.K_x, hw.SpaceTimeVector(y)).array
    w1 = np.empty((n_t, n_x))
    w2 = np.empty((n_t, n_x))
    hw_system._temporal(asm.test.T.T, ky, w1, None)
    hw_system._spatial(asm.spatial.M_x, w1, w2, None)
    g_ss = w2.copy()
    hw_system._temporal(asm.test.N.T, ky, w1, None)
    hw_system._spatial(asm.spatial.A_x, w1, w2, None)
    g_ss += w2
    return y, ky, g_ss, asm.wavelet.transpose_apply_array(g_ss)


def u0_name(u0):
    return {inputs.u0_sines: "sines", inputs.u0_zero: "zero"}.get(u0, "modes")


LEAN_DROP = ("load", "ky", "g_ss", "g_hat", "u0_hat", "MxP", "AxP", "WP")


def run_case(name, d, J, K, dist, full=True, workers=8, lean=False, D=None, c=0.0,
             domain="square", u0=None, nsample=4096):
    t0 = time.time()
    problem = problem_for(d, dist, D, c, u0)
    asm = assemble_reference(problem, J, K, domain)
    n_t, n_x = asm.S.n_t, asm.S.n_x
    F = inputs.forcing(dist, n_t, n_x)
    y, ky, g_ss, g_hat = forcing_part(asm, F)
    u0_hat = asm.rhs.u0_part.array
    fhat = g_hat + u0_hat
    u0proj = hw.project_initial(asm.hierarchy.finest, problem.u0)

    plan = ParallelPlan.create(workers, n_t) if workers > 1 else None
    pool = hw.WorkerPool(workers) if workers > 1 else None
    z = asm.K_X.apply_array(fhat, pool)
    rho0 = _dot(fhat, z, np.empty(n_t), pool)
    eps = 1e-6 * np.sqrt(rho0)
    res = hw.pcg(asm.S, asm.K_X, hw.SpaceTimeVector(fhat), eps, plan)
    u = asm.wavelet.apply_array(res.w.array)
    meta = dict(name=name, d=d, J=J, K=K, dist=dist, n_t=n_t, n_x=n_x, domain=domain,
                u0=u0_name(problem.u0),
                D=np.asarray(problem.D, dtype=float).tolist(), c=float(problem.c),
                seed_f=inputs.SEED_F, probe_seed=PROBE_SEED,
                iterations=res.iterations, eps=eps, rho0=rho0,
                kappa=res.kappa_estimate,
                residual_norms=list(map(float, res.residual_norms)),
                cg_alphas=list(map(float, res.cg_alphas)),
                cg_betas=list(map(float, res.cg_betas)),
                F_sum=float(F.sum()), fhat_norm=float(np.linalg.norm(fhat)),
                u_norm=float(np.linalg.norm(u)),
                w_norm=float(np.linalg.norm(res.w.array)),
                stencils=stencil_table(asm, problem))
    arrays = dict(u0proj=u0proj) if nsample <= 4096 else {}   # large twins: K = 10 rows are 8 MB
    rng = np.random.default_rng(PROBE_SEED)
    idx = np.sort(rng.choice(n_t * n_x, size=min(nsample, n_t * n_x), replace=False))
    arrays["sample_idx"] = idx
    arrays["u_sample"] = u.reshape(-1)[idx]
    arrays["fhat_sample"] = fhat.reshape(-1)[idx]
    if nsample > 4096:                   # large twins: also w, and u's final-time row norm
        arrays["w_sample"] = res.w.array.reshape(-1)[idx]
        meta["u_last_row_norm"] = float(np.linalg.norm(u[-1]))
    if full:
        P = np.random.default_rng(PROBE_SEED).standard_normal((n_t, n_x))
        arrays.update(fhat=fhat, load=y, ky=ky, g_ss=g_ss, g_hat=g_hat,
                      u0_hat=u0_hat, w=res.w.array, u=u)
        arrays["WP"] = asm.wavelet.apply_array(P)
        arrays["WtP"] = asm.wavelet.transpose_apply_array(P)
        arrays["SP"] = asm.S.apply_array(P)
        arrays["KXP"] = asm.K_X.apply_array(P)
        mx = np.empty_like(P)
        ax = np.empty_like(P)
        hw_system._spatial(asm.spatial.M_x, P, mx, None)
        hw_system._spatial(asm.spatial.A_x, P, ax, None)
        arrays["MxP"], arrays["AxP"] = mx, ax
        kx = np.empty_like(P)
        asm.K_x.apply_rows(P, kx, 0, n_t)
        arrays["KxP"] = kx
        cj = np.empty_like(P)
        lv = asm.wavelet.levels.level_of
        for r in range(n_t):
            cj[r] = asm.K_X.blocks[int(lv[r])].apply(P[r])
        arrays["CjP"] = cj
        if lean:
            for key in LEAN_DROP:
                arrays.pop(key)
    if pool is not None:
        pool.close()
    meta["seconds"] = time.time() - t0
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{name}: its={res.iterations} kappa={res.kappa_estimate} "
          f"{meta['seconds']:.1f}s", flush=True)


def mg_rows_case(name, d, K, rows=1, domain="square", D=None, nsample=0):
    """Full outputs of K_x (alpha=1, mu=0) and C_j (alpha=0.3, mu=2^j) MG
    applies on seeded rows at a larger K (streaming-kernel sizes).
    ``nsample`` > 0: store only that many seeded sample positions per row
    plus the row norms (K = 10 rows are 8.4 MB each)."""
    hier = hw.build_mesh_hierarchy(d, K) if domain == "square" else lshape_hierarchy(K)
    ops = hw.assemble_level_operators(hier, D)
    n = ops[-1].A_x.rows
    B = np.random.default_rng(PROBE_SEED).standard_normal((rows, n))
    arrays = dict()
    meta = dict(name=name, d=d, K=K, n=n, rows=rows, probe_seed=PROBE_SEED,
                solvers=[], domain=domain,
                D=None if D is None else np.asarray(D, dtype=float).tolist())
    for (alpha, mu) in ((1.0, 0.0), (0.3, 2.0 ** 5), (0.3, 2.0 ** 10)):
        mg = hw.make_solver(hier, alpha, mu, 2, 3, level_operators=ops)
        X = np.empty_like(B)
        mg.apply_rows(B, X, 0, rows)
        key = f"a{alpha:g}_mu{mu:g}"
        if nsample:
            idx = np.sort(np.random.default_rng(PROBE_SEED + 1).choice(n, nsample, replace=False))
            arrays["sample_idx"] = idx
            arrays[key] = X[:, idx]
            meta.setdefault("row_norms", {})[key] = np.linalg.norm(X, axis=1).tolist()
        else:
            arrays[key] = X
        meta["solvers"].append(dict(key=key, alpha=alpha, mu=mu))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{name}: done", flush=True)


def wavelet_case(name, J, cols):
    lv = hw.build_wavelet(J)
    wt = hw.WaveletTransform(lv)
    P = np.random.default_rng(PROBE_SEED).standard_normal((2 ** J + 1, cols))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                        W=wt.apply_array(P), Wt=wt.transpose_apply_array(P))
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(dict(name=name, J=J, cols=cols, probe_seed=PROBE_SEED), fh)
    print(f"{name}: done", flush=True)


def test_space_case(name, d, J, K, dist, domain="square", D=None):
    """The reference's Lemma-1 (test-space) Schur form on a probe, the
    five-term form on the same probe, and its Lanczos condition estimate
    (solver.py:266-300) with default arguments."""
    problem = problem_for(d, dist, D)
    asm = assemble_reference(problem, J, K, domain)
    n_t, n_x = asm.S.n_t, asm.S.n_x
    St = hw.SchurOperator(temporal=asm.temporal, spatial=asm.spatial, K_x=asm.K_x,
                          wavelet=asm.wavelet, form="test_space", test=asm.test)
    P = np.random.default_rng(PROBE_SEED).standard_normal((n_t, n_x))
    kappa, k = hw.lanczos_condition(asm.S, asm.K_X)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), STP=St.apply_array(P),
                        SP=asm.S.apply_array(P))
    meta = dict(name=name, d=d, J=J, K=K, dist=dist, n_t=n_t, n_x=n_x, domain=domain,
                D=np.asarray(problem.D, dtype=float).tolist(), probe_seed=PROBE_SEED,
                lanczos_kappa=float(kappa), lanczos_iterations=int(k))
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{name}: lanczos kappa={kappa} k={k}", flush=True)


def check_interpolant_load():
    """(N (x) M_x) F == assemble_load of the P1 x P1 interpolant of F."""
    for d, J, K in ((1, 3, 4), (2, 2, 3)):
        hier = hw.build_mesh_hierarchy(d, K)
        mesh = hier.finest
        test = hw.assemble_temporal_test(J)
        ops = hw.assemble_level_operators(hier)[-1]
        n_t, n_x = 2 ** J + 1, ops.M_x.rows
        F = np.random.default_rng(3).uniform(-1, 1, (n_t, n_x))
        npts = 2 ** K

        def g(t, pts):
            # hat interpolation in time, P1 in space (quadrature points are
            # element midpoints/Gauss points -> use barycentric evaluation)
            k = min(int(t * 2 ** J), 2 ** J - 1)
            s = t * 2 ** J - k
            row = (1 - s) * F[k] + s * F[k + 1]
            full = np.zeros(len(mesh.vertices))
            full[mesh.interior] = row
            from scipy.interpolate import LinearNDInterpolator, interp1d
            if d == 1:
                f = interp1d(mesh.vertices[:, 0], full)
                return f(pts[:, 0])
            # the mesh's triangles, not Delaunay's: evaluate per element
            out = np.empty(len(pts))
            gi = pts * npts
            for q, p in enumerate(gi):
                i0, j0 = np.floor(p).astype(int)
                i0, j0 = min(i0, npts - 1), min(j0, npts - 1)
                fx, fy = p[0] - i0, p[1] - j0
                v = lambda a, b: full[(i0 + a) * (npts + 1) + (j0 + b)]
                if fx >= fy:   # triangle (i,j),(i+1,j),(i+1,j+1)
                    out[q] = v(0, 0) + fx * (v(1, 0) - v(0, 0)) + fy * (v(1, 1) - v(1, 0))
                else:          # triangle (i,j),(i+1,j+1),(i,j+1)
                    out[q] = v(0, 0) + fy * (v(0, 1) - v(0, 0)) + fx * (v(1, 1) - v(0, 1))
            return out

        load = hw.assemble_load(mesh, J, g).array
        tmp = np.empty((n_t, n_x))
        y = np.empty((test.N.rows, n_x))
        hw_system._spatial(ops.M_x, F, tmp, None)
        hw_system._temporal(test.N, tmp, y, None)
        rel = np.abs(load - y).max() / np.abs(y).max()
        print(f"interpolant load d={d}: rel diff {rel:.2e}")
        assert rel < 1e-13


def struct_case(name="struct"):
    """The reference's host-side containers on small problems: temporal
    trial/test matrices, meshes, prolongations, level operators (also with
    anisotropic D and reaction), wavelet two-scale matrices -- every CSR as
    (row_offsets, col_indices, values)."""
    from heatwave.multigrid import assemble_level_operators
    arrays, meta = {}, dict(name=name, cases=[])

    def put(key, m):
        arrays[key + ".ip"], arrays[key + ".ix"] = m.row_offsets, m.col_indices
        arrays[key + ".v"] = m.values
        arrays[key + ".shape"] = np.array([m.rows, m.cols])

    for J in (0, 1, 3):
        tr, te = hw.assemble_temporal_trial(J), hw.assemble_temporal_test(J)
        for f in ("M_t", "A_t", "L", "Gamma0"):
            put(f"J{J}.{f}", getattr(tr, f))
        arrays[f"J{J}.phi0"], arrays[f"J{J}.phiT"] = tr.phi_at_0, tr.phi_at_T
        for f in ("O", "T", "N"):
            put(f"J{J}.{f}", getattr(te, f))
        lv = hw.build_wavelet(J)
        arrays[f"J{J}.level_of"] = lv.level_of
        for j, (P, Q) in enumerate(lv.two_scale, start=1):
            put(f"J{J}.P{j}", P), put(f"J{J}.Q{j}", Q)
            put(f"J{J}.M{j}", lv.stage_mats[j - 1][0]), put(f"J{J}.MT{j}", lv.stage_mats[j - 1][1])
    for d, K, D, c in ((1, 4, None, 0.0), (2, 3, None, 0.0), (2, 4, [[1.0, 0.0], [0.0, 6.0]], 0.5)):
        tag = f"d{d}K{K}" + ("a" if D is not None else "")
        meta["cases"].append(dict(tag=tag, d=d, K=K, D=D, c=c))
        hier = hw.build_mesh_hierarchy(d, K)
        for k, m in enumerate(hier.levels, start=1):
            arrays[f"{tag}.mesh{k}.vertices"] = m.vertices
            arrays[f"{tag}.mesh{k}.elements"] = m.elements
            arrays[f"{tag}.mesh{k}.interior"] = m.interior
            arrays[f"{tag}.mesh{k}.interior_index"] = m.interior_index
        for k in range(2, K + 1):
            put(f"{tag}.P{k}", hier.prolongation(k))
        for k, ops in enumerate(assemble_level_operators(hier, D, c), start=1):
            put(f"{tag}.M{k}", ops.M_x), put(f"{tag}.A{k}", ops.A_x)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{name}: {len(arrays)} arrays", flush=True)


CASES = {
    "c1": lambda: run_case("c1", 2, 4, 4, "uniform"),
    "d1": lambda: run_case("d1", 1, 6, 6, "normal"),
    "c2s": lambda: run_case("c2s", 2, 3, 6, "uniform", lean=True),
    # anisotropic diffusion + reaction: |beta| = 0.43 along y > kRegBetaMax,
    # so the GPU multigrid takes the shared-ring (exact-scan) fallback
    "a1": lambda: run_case("a1", 2, 3, 6, "uniform", lean=True, D=[[1.0, 0.0], [0.0, 6.0]], c=0.5),
    # mapped L-shaped domain (BASELINE cfg 5 recipe: D = I/4 after the map
    # [-1,1]^2 -> [0,1]^2, F = 1 + U[-0.1, 0.1]); L1 also projects a
    # non-zero u0, L2 uses cfg 5's u0 = 0 at register-kernel sizes
    "L1": lambda: run_case("L1", 2, 3, 5, "lshape", D=0.25 * np.eye(2), domain="L",
                           u0=inputs.u0_sines),
    "L2": lambda: run_case("L2", 2, 4, 7, "lshape", lean=True, D=0.25 * np.eye(2), domain="L"),
    "mgL8": lambda: mg_rows_case("mgL8", 2, 8, rows=2, domain="L", D=0.25 * np.eye(2)),
    "ts1": lambda: test_space_case("ts1", 2, 4, 4, "uniform"),
    "ts2": lambda: test_space_case("ts2", 2, 3, 7, "lshape", domain="L", D=0.25 * np.eye(2)),
    "d2": lambda: run_case("d2", 1, 10, 10, "normal", full=False),
    "cfg2": lambda: run_case("cfg2", 2, 8, 8, "uniform", full=False),
    "mg8": lambda: mg_rows_case("mg8", 2, 8),
    "mg1d10": lambda: mg_rows_case("mg1d10", 1, 10, rows=4),
    "wav10": lambda: wavelet_case("wav10", 10, 3),
    # round 2: pins at the benched configs' shapes (the reference cannot hold
    # cfg 3/4 in this container's 62 GB: SURVEY §7 "oracle reach")
    # K = 10 MG rows: the n = 1023 finest-level kernels cfg 4 runs
    "mg10": lambda: mg_rows_case("mg10", 2, 10, rows=2, nsample=65536),
    # J = 4, K = 10: a full PCG through every cfg 4 kernel variant (5-point
    # K_x batch, zero-start DOWN, fused r.z UP at n = 1023)
    "c410": lambda: run_case("c410", 2, 4, 10, "uniform", full=False, nsample=65536),
    # J = 10 (cfg 4's N_t and wavelet levels), K = 8
    "t10k8": lambda: run_case("t10k8", 2, 10, 8, "uniform", full=False, nsample=65536),
    # 1D J = 16, K = 10 (cfg 3's N_x, 65,537 temporal rows)
    "d16": lambda: run_case("d16", 1, 16, 10, "normal", full=False, nsample=65536),
    "load": check_interpolant_load,
    "struct": struct_case,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
