"""B200-native space-time PCG for the heat equation (arXiv 2009.08875).

A drop-in for the hot path of the reference package ``heatwave``: the same
public names (``assemble_system``, ``pcg``, ``solve_heat``, ``SchurOperator``,
``PreconditionerKX``, ``WaveletTransform``, ``MultigridSolver`` ...) backed by
hand-written sm_100a kernels in ``libhwgpu.so`` (C ABI:
``include/heatwave_b200.h``).  See DESIGN.md.
"""

from .discretization import ProblemData, lshape_problem
from ._lib import IterationLimitError
from .api import (SolveConfig, SpaceTimeVector, TemporalDiscretization, MeshHierarchy,
                  build_mesh_hierarchy, WaveletTransform, MultigridSolver, make_solver,
                  SchurOperator, PreconditionerKX, RightHandSide, ProblemAssembly,
                  assemble_system, assemble_rhs, PCGResult, pcg, solve_heat, HeatSolution,
                  measure_error, estimate_condition, lanczos_tridiagonal, lanczos_condition, ParallelPlan,
                  split_ranges, tree_reduce, project_initial, decaying_heat, forced_heat,
                  PROBLEMS, build_prolongation, schur_apply, apply_KY, apply_KX, wavelet_apply,
                  wavelet_transpose_apply, WorkerPool, parallel_execute)
from .structures import (SparseMatrix, TemporalMatrices, TestMatrices, SpatialMatrices,
                         WaveletLevels, csr_matvec, dense_materialize, assemble_temporal_trial,
                         assemble_temporal_test, evaluate_trace, assemble_spatial,
                         assemble_level_operators, build_wavelet)
from .api import assemble_load

__version__ = "0.1.0"
