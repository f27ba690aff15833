"""CPU-only checks: the C ABI library, host setup, inputs, bench helpers."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_2009_08875_b200 import _lib, discretization as disc, inputs
from paper_2009_08875_b200 import api


def _header_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        names |= set(re.findall(r"\b(hwg_[a-z_]+)\s*\(", src))
    return names


def test_library_exports_every_header_symbol():
    from paper_2009_08875_b200 import build
    build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 15
    for name in sorted(syms):
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) == syms
    L = _lib.load()
    assert L.hwg_version() == 5


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", ["c1", "c2s", "d1", "a1"])
def test_stencils_bit_identical_to_reference(name):
    meta, _ = golden(name)
    d = meta["d"]
    D, c = meta.get("D"), meta.get("c", 0.0)
    for lvl, st in enumerate(meta["stencils"], start=1):
        M, A = disc.level_stencils(d, lvl, D, c)
        m = 2 ** lvl - 1
        keymap = {0: "c0", 1: "cy"} if d == 1 else {0: "c0", 1: "cy", m: "cx", m + 1: "cd"}
        for ours, offs, vals in ((A, st["A_off"], st["A"]), (M, st["M_off"], st["M"])):
            ref = {keymap[o]: v for o, v in zip(offs, vals) if o >= 0 and o in keymap}
            for k, v in ref.items():
                assert ours[k] == v, (name, lvl, k)
            for k, v in ours.items():
                assert ref.get(k, 0.0) == v, (name, lvl, k)


def test_coef_table_matches_scipy_sum():
    import scipy.sparse as sp
    from oracle import heatwave_oracle as O
    d, J, K, alpha = 2, 3, 4, 0.3
    tab = disc.coef_table(d, J, K, alpha)
    levels = [O.mesh(d, k) for k in range(1, K + 1)]
    for l, lv in enumerate(levels, start=1):
        M, A = O.assemble_p1(lv)
        for o, (a, mu) in enumerate(disc.operator_list(J, alpha)):
            S = (a * A + mu * M).tocsr()
            r = S.shape[0] // 2
            row = dict(zip((S[r].indices - r).tolist(), S[r].data.tolist()))
            m = 2 ** l - 1
            assert tab[o, l, 0] == row[0]
            if l >= 2:
                assert tab[o, l, 2] == row.get(1, 0.0)
                assert tab[o, l, 1] == row.get(m, 0.0)
                assert tab[o, l, 3] == row.get(m + 1, 0.0)


def test_temporal_values_and_levels():
    t = disc.temporal_values(3)
    h = 1 / 8
    assert t[0] == h / 6 and t[1] == 2 * h / 3 and t[4] == 2.0 / h
    assert np.array_equal(disc.level_of(3), [0, 0, 1, 2, 2, 3, 3, 3, 3])
    assert disc.wavelet_scales(2)[1] == 2.0


def test_project_initial_matches_golden():
    for name in ("c1", "d1"):
        meta, g = golden(name)
        mesh = disc.FineMesh(meta["d"], meta["K"])
        u0 = inputs.u0_sines if meta["dist"] == "uniform" else inputs.u0_modes()
        assert np.array_equal(disc.project_initial(mesh, u0), g["u0proj"])


def test_forcing_is_split_invariant():
    full = inputs.forcing("uniform", 200, 7)
    parts = np.concatenate([inputs.forcing_rows("uniform", 200, 7, a, b)
                            for a, b in ((0, 37), (37, 130), (130, 200))])
    assert np.array_equal(full, parts)
    assert inputs.forcing("normal", 5, 3).shape == (5, 3)


def test_host_api_helpers():
    v = np.random.default_rng(0).standard_normal(129)
    assert abs(api.tree_reduce(v) - v.sum()) < 1e-12
    assert api.split_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    plan = api.ParallelPlan.create(3, 10)
    plan.validate()
    with pytest.raises(ValueError):
        api.ParallelPlan(2, ((0, 4), (5, 10)), 1).validate()
    d, e = api.lanczos_tridiagonal([1.0, 0.5], [0.25, 0.1])
    assert d[0] == 1.0 and d[1] == 2.0 + 0.25


def test_problem_data_validation():
    with pytest.raises(ValueError):
        disc.ProblemData(D=np.array([[1.0, 2.0], [0.0, 1.0]]), c=0.0, u0=lambda x: x[:, 0])
    with pytest.raises(ValueError):
        disc.ProblemData(D=np.eye(2), c=-1.0, u0=lambda x: x[:, 0])


def test_bench_model_bytes_match_survey():
    import bench
    per = {1: 2149.6, 2: 2261.6, 3: 3319.0, 4: 2267.4}
    for cfg, want in per.items():
        d, J, K, *_ = inputs.recipe(cfg)
        N = (2 ** J + 1) * (2 ** K - 1) ** d
        assert abs(bench.model_bytes_per_iteration(d, J, K) / N - want) < 0.05


def test_no_oracle_import_in_product():
    for path in glob.glob(os.path.join(ROOT, "paper_2009_08875_b200", "**", "*.py"), recursive=True):
        src = open(path).read()
        assert "oracle" not in src.replace("oracle/", ""), path


def test_library_has_no_undefined_internal_symbols():
    """Every hw:: function the translation units reference is defined in the
    shared library (a missing definition would only fail at dlopen on the
    GPU box)."""
    import shutil
    import subprocess

    from paper_2009_08875_b200 import _lib

    so = _lib.library_path() if hasattr(_lib, "library_path") else None
    if so is None:
        import paper_2009_08875_b200 as pkg
        so = os.path.join(os.path.dirname(pkg.__file__), "libhwgpu.so")
    if not os.path.exists(so) or shutil.which("nm") is None:
        pytest.skip("library not built / nm missing")
    out = subprocess.run(["nm", "-D", "--undefined-only", so], capture_output=True, text=True).stdout
    missing = [ln.split()[-1] for ln in out.splitlines() if "_ZN2hw" in ln]
    assert not missing, missing


def test_bench_implementation_byte_model():
    """Per-iteration algorithmic bytes of this implementation (bench.py
    roofline_iteration): 2D K = 10 streams ~88 words per DoF, dominated by
    the three batched multigrid applications; 1D streams 33 (the fused top
    two wavelet stages move one array less per transform)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    N4 = (2 ** 10 + 1) * (2 ** 10 - 1) ** 2
    w4 = bench.impl_bytes_per_iteration(2, 10, 10) / 8 / N4
    assert 85 < w4 < 95, w4
    N3 = (2 ** 20 + 1) * (2 ** 10 - 1)
    assert abs(bench.impl_bytes_per_iteration(1, 20, 10) / 8 / N3 - 33.0) < 0.01


def test_lshape_host_setup_matches_oracle():
    """L-shaped domain (BASELINE cfg 5, mapped): dof count, finest mesh, and
    the level-2 dense inverses the GPU coarse kernel applies are bit-identical
    to the oracle's (which the L1/L2/mgL8 fixtures pin to the reference)."""
    from oracle import heatwave_oracle as O

    D = 0.25 * np.eye(2)
    for K in (2, 3, 5, 11):
        assert disc.lshape_dofs(K) == (2 ** K - 1) ** 2 - 4 ** (K - 1)
    assert disc.lshape_dofs(11) == 3141633          # BASELINE cfg 5: ~3.1e6 interior dofs
    fm = disc.FineMesh(2, 5, "L")
    lv = O.mesh(2, 5, "L")
    assert np.array_equal(fm.interior, lv.interior)
    assert np.array_equal(fm.elements, lv.elems)
    system = O.assemble(2, 3, 4, D=D, domain="L")
    ci = disc.lshape_coarse_inverses(disc.operator_list(3, 0.3), D)
    assert np.array_equal(system.Kx._keep[-1].ravel(), ci[0])
    for j in range(4):
        assert np.array_equal(system.blocks[j]._keep[-1].ravel(), ci[1 + j])
    # interior stencils of the L equal the square's with the same D
    M, A = disc.level_stencils(2, 4, D)
    lv4 = O.mesh(2, 4, "L")
    Mo, Ao = O.assemble_p1(lv4, D)
    r = int(np.nonzero(np.all(np.rint(lv4.verts[lv4.interior] * 16) == [4, 4], axis=1))[0][0])
    assert sorted(Ao.tocsr()[r].data.tolist()) == sorted([A["c0"]] + [A["cx"]] * 2 + [A["cy"]] * 2)
    assert inputs.CONFIGS[5]["domain"] == "L"


def test_bench_config5_workload_and_dof_bytes():
    """bench.py --config 5: the per-GPU share of the 8-GPU L-shaped problem
    (J = 8 + log2 N, mapped K = 11, D = I/4), with the algorithmic bytes
    counted on the L's dofs (3/4 of the embedded grid)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    d, J, K, dist, u0, n_t, n_x = bench.workload(5)
    assert (d, J, K, dist, n_t, n_x) == (2, 8, 11, "lshape", 257, 3141633)
    assert bench.workload(5, 8)[1] == 11                # the full cfg 5 on 8 GPUs
    assert bench.domain_of(5) == "L" and bench.domain_of(4) == "square"
    assert np.array_equal(bench.diffusion_of(5, 2), 0.25 * np.eye(2))
    frac = bench.dof_fraction(5, 2, 11, n_x)
    assert abs(frac - 3141633 / 2047 ** 2) < 1e-15 and 0.74 < frac < 0.76
    assert bench.dof_fraction(4, 2, 10, 1023 ** 2) == 1.0
    assert "per-GPU share" in bench.workload_label(5, d, J, K, n_t, n_x)


def test_bench_launcher_command():
    """bench.py --gpus N (no WORLD_SIZE) re-runs itself as N torchrun ranks
    on 127.0.0.1 with the same arguments."""
    import bench
    cmd = bench.launcher_command(["--gpus", "8", "--steps", "2"], 8, 29501)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd
    i = cmd.index("--master-addr")
    assert cmd[i + 1] == "127.0.0.1" and "--master-port=29501" in cmd
    assert cmd[-5:] == [os.path.abspath(bench.__file__), "--gpus", "8", "--steps", "2"]


def test_bench_configs_match_between_arms():
    """Both arms print the same `config` object (the reference arm's bounded
    sample is described in its cpu_baseline.sample)."""
    import bench
    for cfg in (1, 2, 3, 4):
        assert bench.config_dict(cfg, 1)["dofs"] == (2 ** bench.workload(cfg)[1] + 1) * \
            bench.workload(cfg)[6]
    assert bench.config_dict(4, 8)["parallelism"].startswith("time slabs x8")
    assert bench.config_dict(4, 1)["parallelism"] == "1 GPU"
