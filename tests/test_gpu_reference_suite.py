"""The reference's own solver / multigrid / acceptance tests, restated on the
GPU package (tests/test_solver.py, test_multigrid.py, test_acceptance.py of
/root/reference/pkg; cited per test).  Tests that need the CPU-only
exact-inverse mode (ExactSolver, sparse LU) or 3D meshes are not restated:
both are outside the GPU hot path.  The oracle (tests only)
supplies the P1 mass matrix where a reference test assembles one."""
import dataclasses

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from conftest import relative_diff

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2009_08875_b200 as hw  # noqa: E402
from paper_2009_08875_b200 import discretization as disc  # noqa: E402


@pytest.fixture(scope="module")
def small2d():
    return hw.assemble_system(hw.decaying_heat(2), 3, 3, hw.SolveConfig())


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


# ---- test_solver.py: TestPcg ------------------------------------------------
def test_zero_rhs_returns_immediately(small2d):                 # test_solver.py:53-57
    rhs = hw.SpaceTimeVector(np.zeros((small2d.S.n_t, small2d.S.n_x)))
    res = hw.pcg(small2d.S, small2d.K_X, rhs, 1e-6)
    assert res.iterations == 0
    assert not np.any(res.w.array)


def test_solves_system(small2d):                                # test_solver.py:59-63
    res = hw.pcg(small2d.S, small2d.K_X, small2d.rhs, 1e-8)
    r = small2d.rhs.f_hat.array - small2d.S.apply_array(res.w.array.copy())
    z = small2d.K_X.apply_array(r.copy())
    assert np.sqrt((r * z).sum()) <= 1e-8


def test_residual_history_monotone_head_and_final(small2d):     # test_solver.py:65-68
    res = hw.pcg(small2d.S, small2d.K_X, small2d.rhs, 1e-6)
    assert res.residual_norms[-1] <= 1e-6
    assert res.residual_norms[0] > res.residual_norms[-1]


def test_iteration_cap_carries_history(small2d):                # test_solver.py:70-73
    with pytest.raises(hw.IterationLimitError) as err:
        hw.pcg(small2d.S, small2d.K_X, small2d.rhs, 1e-6, max_iterations=2)
    assert len(err.value.residual_norms) == 3


def test_invalid_tolerance(small2d):                            # test_solver.py:75-77
    with pytest.raises(ValueError):
        hw.pcg(small2d.S, small2d.K_X, small2d.rhs, 0.0)


def test_true_residual_recompute_matches_recurrence(small2d):   # test_solver.py:79-83
    few = hw.pcg(small2d.S, small2d.K_X, small2d.rhs, 1e-8, recompute_every=3)
    ref = hw.pcg(small2d.S, small2d.K_X, small2d.rhs, 1e-8)
    assert few.iterations == ref.iterations
    assert np.abs(few.w.array - ref.w.array).max() <= 1e-9


def test_condition_estimate_requires_iterations(small2d):       # test_solver.py:85-93
    res = hw.pcg(small2d.S, small2d.K_X, small2d.rhs, 1e-1)
    if res.iterations < 5:
        with pytest.raises(ValueError):
            hw.estimate_condition(res)
    full = hw.pcg(small2d.S, small2d.K_X, small2d.rhs, 1e-8)
    est = hw.estimate_condition(full)
    assert est == full.kappa_estimate and est > 1.0


# ---- test_solver.py: TestSolveHeat -----------------------------------------
def test_zero_data_zero_solution():                             # test_solver.py:154-159
    problem = hw.ProblemData(D=np.eye(1), c=0.0, u0=lambda x: np.zeros(len(x)))
    res, sol = hw.solve_heat(problem, 2, 2)
    assert res.iterations == 0
    assert not np.any(sol.coefficients.numpy())


def test_decaying_2d_solution_quality():                        # test_solver.py:161-175
    from oracle import heatwave_oracle as O
    problem = hw.decaying_heat(2)
    for lvl in (3, 4):
        res, sol = hw.solve_heat(problem, lvl, lvl)
        assert res.iterations <= 20
        err0 = hw.measure_error(sol, problem.exact_solution, 0.0)
        mesh = sol.mesh
        M, _ = O.assemble_p1(O.mesh(2, lvl))
        proj = spla.spsolve(M.tocsc(), disc.project_initial(mesh, problem.u0))
        proj_err = disc.l2_error_on_mesh(mesh, proj, lambda x: problem.exact_solution(0.0, x))
        assert err0 <= 16.0 * proj_err


def test_1d_smoke_within_budget():                              # test_solver.py:188-193
    import time
    hw.solve_heat(hw.forced_heat(1), 3, 3)                      # library / context warm-up
    t0 = time.perf_counter()
    res, _ = hw.solve_heat(hw.forced_heat(1), 6, 6)
    assert time.perf_counter() - t0 < 10.0
    assert res.iterations <= 30


def test_error_rate_under_joint_refinement():                   # test_solver.py:195-203,
    problem = hw.forced_heat(2)                                 # test_acceptance.py:276-289
    errs = []
    for lvl in (2, 3, 4):
        _, sol = hw.solve_heat(problem, lvl, lvl, hw.SolveConfig(epsilon=1e-9))
        errs.append(hw.measure_error(sol, problem.exact_solution, 1.0))
    rates = [np.log2(a / b) for a, b in zip(errs, errs[1:])]
    assert min(rates) >= 1.7


def test_interpolant_roundtrip_gives_interpolation_error():     # test_solver.py:205-217
    problem = hw.forced_heat(2)
    _, sol = hw.solve_heat(problem, 2, 3)
    mesh = sol.mesh
    nodes = mesh.vertices[mesh.interior]
    exact = problem.exact_solution
    X = np.array([exact(t, nodes) for t in np.linspace(0, 1, sol.temporal.N_t)])
    fake = hw.HeatSolution(coefficients=hw.SpaceTimeVector(X), mesh=mesh,
                           temporal=sol.temporal, algebraic_error=0.0)
    got = hw.measure_error(fake, exact, 1.0)
    want = disc.l2_error_on_mesh(mesh, exact(1.0, nodes), lambda x: exact(1.0, x))
    assert got == want


def test_trace_times_validated():                               # test_solver.py:219-225
    problem = hw.decaying_heat(1)
    _, sol = hw.solve_heat(problem, 2, 2)
    with pytest.raises(ValueError):
        hw.measure_error(sol, problem.exact_solution, 1.5)
    for t in (0.0, 0.3, 1.0):
        assert hw.measure_error(sol, problem.exact_solution, t) >= 0.0


# ---- test_multigrid.py: TestBasics (square and the L-shaped domain) ---------
@pytest.fixture(scope="module", params=["square", "L"])
def hier2d(request):
    return hw.build_mesh_hierarchy(2, 5, request.param)


def _D(h):
    return 0.25 * np.eye(2) if h.domain == "L" else None


def test_single_level_equals_direct_solve(rng):                 # test_multigrid.py:18-24
    mg = hw.make_solver(hw.build_mesh_hierarchy(2, 1), 1.0, 0.0)
    A = np.array([[4.0]])
    b = rng.standard_normal(1)
    assert np.allclose(mg.apply(b), np.linalg.solve(A, b), atol=1e-14)


def test_zero_rhs_and_dimension_mismatch(hier2d):              # test_multigrid.py:26-35
    mg = hw.make_solver(hier2d, 1.0, 0.0, D=_D(hier2d))
    assert not np.any(mg.apply(np.zeros(mg.n)))
    with pytest.raises(ValueError):
        mg.apply(np.zeros(mg.n + 1))


def test_invalid_coefficients_and_defaults(hier2d):            # test_multigrid.py:37-45
    with pytest.raises(ValueError):
        hw.make_solver(hier2d, 0.0, 0.0)
    mg = hw.make_solver(hier2d, 1.0, 0.0, D=_D(hier2d))
    assert mg.n_vcycles == 2 and mg.n_smooth == 3


def test_linearity(hier2d, rng):                               # test_multigrid.py:47-54
    mg = hw.make_solver(hier2d, 0.3, 4.0, D=_D(hier2d))
    x = rng.standard_normal(mg.n)
    y = rng.standard_normal(mg.n)
    lhs = mg.apply(2.0 * x + 3.0 * y)
    rhs = 2.0 * mg.apply(x) + 3.0 * mg.apply(y)
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(lhs).max()


def test_symmetry(hier2d, rng):                                # test_multigrid.py:56-64
    mg = hw.make_solver(hier2d, 1.0, 0.0, D=_D(hier2d))
    B1 = rng.standard_normal((50, mg.n))
    B2 = rng.standard_normal((50, mg.n))
    X1, X2 = np.empty_like(B1), np.empty_like(B2)
    mg.apply_rows(B1, X1, 0, 50)
    mg.apply_rows(B2, X2, 0, 50)
    for k in range(50):
        d1, d2 = X1[k] @ B2[k], B1[k] @ X2[k]
        assert abs(d1 - d2) <= 1e-12 * max(abs(d1), 1.0)


# ---- test_acceptance.py: criterion 2 (Schur forms agree) --------------------
def test_forms_agree_on_random_vectors(rng):                    # test_acceptance.py:85-98
    asm = hw.assemble_system(hw.decaying_heat(2), 3, 3, hw.SolveConfig())
    S1 = dataclasses.replace(asm.S, form="test_space")
    worst = 0.0
    for _ in range(100):
        v = hw.SpaceTimeVector(rng.standard_normal((9, 49)))
        a = S1.apply(v).array
        b = asm.S.apply(v).array
        worst = max(worst, np.abs(a - b).max() / np.abs(b).max())
    assert worst <= 1e-12


def test_lshape_decaying_mode_is_resolved():
    """L-shaped domain (mapped, D = I/4): u0 = the first sine mode of the
    lower-left unit square, which the L contains in the mapped coordinates
    ([0,1/2]^2) -- a smooth initial datum on the L.  The solution must decay
    in time and the trace at t = 0 must be as accurate as the L2 projection
    of u0 up to the reference's factor 16 (test_solver.py:161-175)."""
    from oracle import heatwave_oracle as O
    u0 = lambda p: np.where((p[:, 0] <= 0.5) & (p[:, 1] <= 0.5),  # noqa: E731
                            np.sin(2 * np.pi * p[:, 0]) * np.sin(2 * np.pi * p[:, 1]), 0.0)
    prob = hw.lshape_problem(u0=u0)
    res, sol = hw.solve_heat(prob, 5, 5, domain="L")          # matched resolution, as there
    assert res.iterations <= 25
    mesh = sol.mesh
    M, _ = O.assemble_p1(O.mesh(2, 5, "L"))
    proj = spla.spsolve(M.tocsc(), disc.project_initial(mesh, u0))
    err_proj = disc.l2_error_on_mesh(mesh, proj, u0)
    err0 = hw.measure_error(sol, lambda t, x: u0(x), 0.0)
    assert err0 <= 16.0 * err_proj
    c = sol.coefficients.numpy()
    assert np.linalg.norm(c[-1]) < 0.5 * np.linalg.norm(c[0])
