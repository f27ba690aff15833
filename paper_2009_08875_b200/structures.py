"""Host-side containers of the reference's public API (setup only).

The reference exposes its discretisation as plain CSR containers and
dataclasses (``SparseMatrix`` sparse.py:50-117, ``TemporalMatrices`` /
``TestMatrices`` temporal.py:53-79, ``SpatialMatrices`` / ``Mesh`` /
``MeshHierarchy`` spatial.py:49-95, ``WaveletLevels`` wavelet.py:31-53).
Code written against ``heatwave`` reads ``asm.temporal.M_t``,
``asm.spatial.A_x``, ``asm.test.N``, ``hierarchy.levels`` or
``hierarchy.prolongation(k)``; this module provides the same objects with
the same values so that such code keeps working against the GPU package.

None of it is on the hot path: the GPU kernels carry the same operators as
compile-time stencils and band triples.  The matrices are
built on first use (the finest-level CSR at K = 10 is ~7e6 entries).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import discretization as disc


# --------------------------------------------------------------------------
# CSR container (sparse.py:50-117)
# --------------------------------------------------------------------------
@dataclass
class SparseMatrix:
    """Compressed-row matrix with int64 indices and sorted columns."""

    rows: int
    cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    symmetric: bool = False

    @classmethod
    def from_scipy(cls, m, symmetric=False):
        m = sp.csr_matrix(m)
        m.sort_indices()
        return cls(m.shape[0], m.shape[1], m.indptr.astype(np.int64),
                   m.indices.astype(np.int64), m.data.astype(np.float64), symmetric)

    @classmethod
    def identity(cls, n):
        return cls.from_scipy(sp.identity(n, format="csr"), symmetric=True)

    @classmethod
    def from_diagonal(cls, d):
        return cls.from_scipy(sp.diags(np.asarray(d, dtype=float)).tocsr(), symmetric=True)

    def to_scipy(self):
        return sp.csr_matrix((self.values, self.col_indices, self.row_offsets),
                             shape=(self.rows, self.cols))

    def to_dense(self):
        return self.to_scipy().toarray()

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def nnz(self):
        return len(self.values)

    @property
    def T(self):
        return SparseMatrix.from_scipy(self.to_scipy().T.tocsr(), self.symmetric)

    def diagonal(self):
        return self.to_scipy().diagonal()

    def check_symmetric(self, tol=1e-12):
        if self.rows != self.cols:
            return False
        a = self.to_scipy()
        scale = abs(a).max() if a.nnz else 1.0
        return abs(a - a.T).max() <= tol * max(scale, 1.0)

    def validate(self):
        if len(self.row_offsets) != self.rows + 1:
            raise ValueError("row_offsets must have rows+1 entries")
        if np.any(np.diff(self.row_offsets) < 0):
            raise ValueError("row_offsets must be nondecreasing")
        if self.nnz and (self.col_indices.min() < 0 or self.col_indices.max() >= self.cols):
            raise ValueError("col_indices out of range")
        if not np.all(np.isfinite(self.values)):
            raise ValueError("values must be finite")
        if self.symmetric and not self.check_symmetric():
            raise ValueError("matrix flagged symmetric is not")
        return self


def csr_matvec(A: SparseMatrix, x):
    """y = A x on the host, each row summed left to right (sparse.py:120-130)."""
    x = np.asarray(x, dtype=float)
    if x.shape != (A.cols,):
        raise ValueError(f"dimension mismatch: matrix is {A.rows}x{A.cols}, "
                         f"vector has shape {x.shape}")
    return A.to_scipy() @ x


def dense_materialize(op, n, m=None):
    """Dense matrix of a linear map x -> op(x) of R^n (columns op(e_i))."""
    m = n if m is None else m
    out = np.zeros((m, n))
    e = np.zeros(n)
    for i in range(n):
        e[i] = 1.0
        out[:, i] = np.asarray(op(e.copy())).reshape(-1)
        e[i] = 0.0
    return out


# --------------------------------------------------------------------------
# temporal matrices (temporal.py:53-158)
# --------------------------------------------------------------------------
@dataclass
class TemporalMatrices:
    M_t: SparseMatrix
    A_t: SparseMatrix
    L: SparseMatrix
    Gamma0: SparseMatrix
    phi_at_0: np.ndarray
    phi_at_T: np.ndarray


@dataclass
class TestMatrices:
    O: SparseMatrix
    T: SparseMatrix
    N: SparseMatrix

    __test__ = False          # not a pytest class


def _tridiag(lo, main, hi):
    n = len(main)
    return sp.diags([np.full(n - 1, lo), main, np.full(n - 1, hi)], [-1, 0, 1], format="csr")


def assemble_temporal_trial(J: int) -> TemporalMatrices:
    """M_t, A_t, L, Gamma0 on the hat basis of 2^J uniform elements; the
    band values are disc.temporal_values (the ones the GPU bands use)."""
    if J < 0:
        raise ValueError("refinement level J must be >= 0")
    n = 2 ** J + 1
    t = disc.temporal_values(J)
    ends = np.zeros(n, dtype=bool)
    ends[[0, -1]] = True
    M_t = _tridiag(t[0], np.where(ends, t[2], t[1]), t[0])
    A_t = _tridiag(t[3], np.where(ends, t[5], t[4]), t[3])
    main = np.zeros(n)
    main[0], main[-1] = -t[7], t[7]
    L = _tridiag(-t[6], main, t[6])
    e0 = np.zeros(n)
    e0[0] = 1.0
    eT = np.zeros(n)
    eT[-1] = 1.0
    G0 = sp.csr_matrix(([1.0], ([0], [0])), shape=(n, n))
    return TemporalMatrices(SparseMatrix.from_scipy(M_t, True), SparseMatrix.from_scipy(A_t, True),
                            SparseMatrix.from_scipy(L), SparseMatrix.from_scipy(G0, True), e0, eT)


def assemble_temporal_test(J: int) -> TestMatrices:
    """O = I, T and N against the per-element Legendre test basis (rows
    2k: degree 0, 2k+1: degree 1 of element k)."""
    if J < 0:
        raise ValueError("refinement level J must be >= 0")
    ne = 2 ** J
    t = disc.temporal_values(J)
    k = np.arange(ne)
    rows = np.stack([2 * k, 2 * k, 2 * k + 1, 2 * k + 1], axis=1).ravel()
    cols = np.stack([k, k + 1, k, k + 1], axis=1).ravel()
    tv = np.tile([-t[8], t[8], 0.0, 0.0], ne)
    nv = np.tile([t[9], t[9], -t[10], t[10]], ne)
    shape = (2 * ne, ne + 1)
    T = sp.csr_matrix((tv, (rows, cols)), shape=shape)
    T.eliminate_zeros()
    N = sp.csr_matrix((nv, (rows, cols)), shape=shape)
    return TestMatrices(SparseMatrix.from_scipy(sp.identity(2 * ne, format="csr"), True),
                        SparseMatrix.from_scipy(T), SparseMatrix.from_scipy(N))


def evaluate_trace(J: int, t: float) -> np.ndarray:
    """Hat-basis values at t = 0 or t = T = 1 (temporal.py:147-158)."""
    out = np.zeros(2 ** J + 1)
    if t == 0.0:
        out[0] = 1.0
    elif t == 1.0:
        out[-1] = 1.0
    else:
        raise ValueError("trace evaluation only defined at t = 0 or t = T = 1")
    return out


# --------------------------------------------------------------------------
# spatial matrices, level operators, prolongations (spatial.py:140-229,
# multigrid.py:26-28)
# --------------------------------------------------------------------------
@dataclass
class SpatialMatrices:
    M_x: SparseMatrix
    A_x: SparseMatrix


class LazySpatialMatrices:
    """SpatialMatrices of a mesh, assembled on first access (the finest
    level of a cfg 4 problem is 1e6 rows; the GPU path never needs it)."""

    def __init__(self, mesh, D=None, c=0.0):
        self._args = (mesh, D, c)
        self._m = None

    def _get(self):
        if self._m is None:
            self._m = assemble_spatial(*self._args)
        return self._m

    @property
    def M_x(self):
        return self._get().M_x

    @property
    def A_x(self):
        return self._get().A_x


class LazyMatrix:
    """Stands for ``getattr(owner, name)`` (a SparseMatrix) and builds it on
    first attribute access."""

    def __init__(self, owner, name):
        self._owner, self._name = owner, name

    def __getattr__(self, attr):
        return getattr(getattr(self._owner, self._name), attr)


def assemble_spatial(mesh, D=None, c=0.0) -> SpatialMatrices:
    """P1 mass and stiffness (+ c mass) on the mesh's interior vertices,
    symmetrised like the reference (A = (A + A^T)/2)."""
    d = mesh.d
    D = np.eye(d) if D is None else np.atleast_2d(np.asarray(D, dtype=float))
    if not np.allclose(D, D.T) or np.any(np.linalg.eigvalsh(D) <= 0):
        raise ValueError("diffusion matrix must be symmetric positive definite")
    locM, locA = disc._element_matrices(mesh.vertices, mesh.elements, d, D, c)
    inner = mesh.interior
    out = []
    for loc in (locM, locA):
        A = disc._assembled(mesh.vertices, mesh.elements, loc)[inner][:, inner].tocsr()
        out.append(SparseMatrix.from_scipy((A + A.T) / 2, symmetric=True))
    return SpatialMatrices(*out)


def prolongation_between(coarse, fine) -> SparseMatrix:
    """Interpolation from the coarse level's interior dofs to the fine
    level's: a fine vertex on a coarse vertex copies it; any other is the
    mean of the two ends of the coarse edge along its odd grid directions
    (the (+1, +1) diagonal orientation makes that an edge).  Coarse ends on
    the boundary (or in the L's removed quadrant) contribute nothing."""
    nf, nc = 2 ** fine.level, 2 ** coarse.level
    g = np.rint(fine.vertices[fine.interior] * nf).astype(np.int64)
    par = g % 2
    rows = np.arange(len(g))
    cidx = coarse.interior_index

    def coarse_ids(gc):
        ok = np.all((gc > 0) & (gc < nc), axis=1)
        flat = gc[:, 0] if fine.d == 1 else gc[:, 0] * (nc + 1) + gc[:, 1]
        cid = np.where(ok, cidx[np.where(ok, flat, 0)], -1)
        return cid

    on = ~par.any(axis=1)
    r_all, c_all, v_all = [], [], []
    cid = coarse_ids(g // 2)
    m = on & (cid >= 0)
    r_all.append(rows[m]), c_all.append(cid[m]), v_all.append(np.full(m.sum(), 1.0))
    for end in ((g - par) // 2, (g + par) // 2):
        cid = coarse_ids(end)
        m = ~on & (cid >= 0)
        r_all.append(rows[m]), c_all.append(cid[m]), v_all.append(np.full(m.sum(), 0.5))
    P = sp.csr_matrix((np.concatenate(v_all), (np.concatenate(r_all), np.concatenate(c_all))),
                      shape=(fine.n_interior, coarse.n_interior))
    return SparseMatrix.from_scipy(P)


def assemble_level_operators(hierarchy, D=None, c=0.0):
    """SpatialMatrices of every level, coarse to fine (multigrid.py:26-28)."""
    return [assemble_spatial(m, D, c) for m in hierarchy.levels]


# --------------------------------------------------------------------------
# wavelet levels (wavelet.py:31-96)
# --------------------------------------------------------------------------
@dataclass
class WaveletLevels:
    """Level map and two-scale matrices of the three-point wavelet basis:
    two_scale[j-1] = (P_j, Q_j), stage_mats[j-1] = (M_j, M_j^T) with
    M_j = [P_j | Q_j] on the length-(2^j+1) prefix."""

    J: int
    level_of: np.ndarray
    dims: np.ndarray
    two_scale: list
    stage_mats: list

    @property
    def n_t(self):
        return 2 ** self.J + 1

    def scaling_weights(self):
        return 2.0 ** self.level_of.astype(float)


def _two_scale(j):
    nc, nf, nw = 2 ** (j - 1) + 1, 2 ** j + 1, 2 ** (j - 1)
    i = np.arange(nc)
    pr = np.concatenate([2 * i, 2 * i[:-1] + 1, 2 * i[1:] - 1])
    pc = np.concatenate([i, i[:-1], i[1:]])
    pv = np.concatenate([np.ones(nc), np.full(nc - 1, 0.5), np.full(nc - 1, 0.5)])
    P = sp.csr_matrix((pv, (pr, pc)), shape=(nf, nc))
    s = 2.0 ** (j / 2.0)
    k = np.arange(nw)
    a = np.where(k == 0, -1.0, -0.5)
    b = np.where(k == nw - 1, -1.0, -0.5)
    qr = np.concatenate([2 * k, 2 * k + 1, 2 * k + 2])
    qc = np.concatenate([k, k, k])
    qv = np.concatenate([s * a, np.full(nw, s), s * b])
    Q = sp.csr_matrix((qv, (qr, qc)), shape=(nf, nw))
    M = sp.hstack([P, Q]).tocsr()
    return (SparseMatrix.from_scipy(P), SparseMatrix.from_scipy(Q)), \
        (SparseMatrix.from_scipy(M), SparseMatrix.from_scipy(M.T.tocsr()))


def build_wavelet(J: int) -> WaveletLevels:
    if J < 0:
        raise ValueError("refinement level J must be >= 0")
    pairs = [_two_scale(j) for j in range(1, J + 1)]
    return WaveletLevels(J, disc.level_of(J), np.array([2 ** j + 1 for j in range(J + 1)]),
                         [p[0] for p in pairs], [p[1] for p in pairs])


def dense_transform(levels: WaveletLevels) -> np.ndarray:
    """Dense W_J by the two-scale recursion W_j = [P_j W_{j-1} | Q_j]."""
    W = np.eye(2)
    for j in range(1, levels.J + 1):
        P, Q = levels.two_scale[j - 1]
        W = np.hstack([P.to_dense() @ W, Q.to_dense()])
    return W
