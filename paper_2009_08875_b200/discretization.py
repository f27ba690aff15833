"""Host-side setup: the numbers the GPU kernels are parameterised with.

Everything here is one-time setup on small arrays (no per-iteration work):

* per-level P1 stencils of M_x and A_x -- the reference assembles global CSR
  matrices (spatial.py:202-229); on the uniform nested meshes every interior
  row of a level carries the same values, so we assemble a 4x4-cell patch
  with the reference's element formulas and read its centre row (this
  reproduces the reference's values bit for bit, pinned by
  tests/test_discretization.py against reference-generated tables);
* the multigrid coefficient table alpha*A_l + mu*M_l for K_x (alpha=1,
  mu=0) and the blocks C_j (alpha, mu=2^j) -- multigrid.py:87-91,
  solver.py:372-377;
* temporal band values -- temporal.py:82-144;
* wavelet stage scales 2^(j/2) and the level map -- wavelet.py:56-96;
* quadrature moments <u0, phi_i> and the test-space load of a callable
  forcing -- spatial.py:232-300 (needed by assemble_rhs for general data).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import scipy.sparse as sp

COEF_STRIDE = 8


@dataclass
class ProblemData:
    """Coefficients and data of u_t - div(D grad u) + c u = g (spatial.py:29-46)."""

    D: np.ndarray
    c: float
    u0: Callable
    g: Optional[Callable] = None
    exact_solution: Optional[Callable] = None

    def __post_init__(self):
        self.D = np.atleast_2d(np.asarray(self.D, dtype=float))
        if not np.allclose(self.D, self.D.T):
            raise ValueError("diffusion matrix must be symmetric")
        if np.any(np.linalg.eigvalsh(self.D) <= 0):
            raise ValueError("diffusion matrix must be positive definite")
        if self.c < 0:
            raise ValueError("reaction coefficient must be >= 0")


# --------------------------------------------------------------------------
# uniform simplicial meshes of [0,1]^d (the reference's orientation:
# x-index slow, y-index fast; every square split along the (+1,+1) diagonal)
# --------------------------------------------------------------------------
def _grid_mesh(d, cells, h):
    """Vertices (npts^d, d) at integer multiples of h, and the elements."""
    npts = cells + 1
    g = np.arange(npts)
    if d == 1:
        verts = g[:, None].astype(float) * h
        elems = np.stack([g[:-1], g[1:]], axis=1)
        return verts, elems
    I, Jg = np.meshgrid(g, g, indexing="ij")
    verts = np.stack([I.ravel(), Jg.ravel()], axis=1).astype(float) * h
    a, b = (t.ravel() for t in np.meshgrid(g[:-1], g[:-1], indexing="ij"))
    vid = lambda i, j: i * npts + j  # noqa: E731
    first = np.stack([vid(a, b), vid(a + 1, b), vid(a + 1, b + 1)], axis=1)
    second = np.stack([vid(a, b), vid(a + 1, b + 1), vid(a, b + 1)], axis=1)
    return verts, np.concatenate([first, second])


def _lshape_filter(elems, cells):
    """Drop the elements of the removed quadrant [1/2,1]^2 from a square
    mesh of ``cells`` x ``cells`` cells (element order otherwise kept: the
    first half are the (i,j),(i+1,j),(i+1,j+1) triangles, the second half
    the (i,j),(i+1,j+1),(i,j+1) ones, both over cells (a, b) in ij order)."""
    g = np.arange(cells)
    a, b = (t.ravel() for t in np.meshgrid(g, g, indexing="ij"))
    keep = ~((a >= cells // 2) & (b >= cells // 2))
    return np.concatenate([elems[: cells * cells][keep], elems[cells * cells:][keep]])


def lshape_interior(gi, n):
    """Interior vertices of the mapped L (grid coordinates gi, n cells)."""
    return np.all((gi > 0) & (gi < n), axis=1) & ~np.all(gi >= n // 2, axis=1)


def lshape_dofs(K):
    """N_x of the mapped L at level K: (2^K-1)^2 - 4^(K-1)."""
    return (2 ** K - 1) ** 2 - 4 ** (K - 1)


def lshape_coarse_inverses(ops, D=None, c=0.0):
    """[(len(ops)), 25]: scipy.linalg.inv of alpha*A_2 + mu*M_2 on the L's
    5-dof level 2, per operator (alpha, mu) -- make_solver's coarse_inv
    (multigrid.py:98-118) for the reference hierarchy of the L, assembled
    like assemble_spatial (spatial.py:202-229)."""
    import scipy.linalg as sla
    D = np.eye(2) if D is None else np.atleast_2d(np.asarray(D, dtype=float))
    verts, elems = _grid_mesh(2, 4, 0.25)
    elems = _lshape_filter(elems, 4)
    locM, locA = _element_matrices(verts, elems, 2, D, c)
    gi = np.rint(verts * 4).astype(int)
    inner = np.nonzero(lshape_interior(gi, 4))[0]
    mats = []
    for loc in (locM, locA):
        A = _assembled(verts, elems, loc)[inner][:, inner].tocsr()
        mats.append(((A + A.T) / 2).tocsr())
    Mx, Ax = mats
    out = np.zeros((len(ops), 25))
    for o, (a, mu) in enumerate(ops):
        S = a * Ax + mu * Mx
        S.sort_indices()
        out[o] = np.ascontiguousarray(sla.inv(S.tocsr().toarray())).ravel()
    return out


def _element_matrices(verts, elems, d, D, c):
    v = verts[elems]
    E = v[:, 1:, :] - v[:, :1, :]
    vol = np.abs(np.linalg.det(E)) / math.factorial(d)
    G = np.swapaxes(np.linalg.inv(E), 1, 2)
    grads = np.concatenate([-G.sum(axis=1, keepdims=True), G], axis=1)
    DG = np.einsum("ij,ekj->eki", D, grads)
    locA = np.einsum("eki,eli->ekl", grads, DG) * vol[:, None, None]
    locM = (np.ones((d + 1, d + 1)) + np.eye(d + 1)) / ((d + 1) * (d + 2))
    locM = locM[None] * vol[:, None, None]
    if c:
        locA = locA + c * locM
    return locM, locA


def _assembled(verts, elems, loc):
    d1 = elems.shape[1]
    rows = np.repeat(elems, d1, axis=1).ravel()
    cols = np.tile(elems, (1, d1)).ravel()
    nv = len(verts)
    A = sp.coo_matrix((loc.ravel(), (rows, cols)), shape=(nv, nv)).tocsr()
    return A


def level_stencils(d, level, D=None, c=0.0):
    """Centre-row values of (M, A) on level ``level`` (h = 2^-level).

    2D returns dicts with keys c0 (centre), cx ((i+-1, j)), cy ((i, j+-1)),
    cd ((i+1, j+1) / (i-1, j-1)); 1D uses c0 and cy (the two neighbours).
    A missing CSR entry is reported as 0.0.
    """
    D = np.eye(d) if D is None else np.atleast_2d(np.asarray(D, dtype=float))
    h = 2.0 ** -level
    cells = min(4, 2 ** level)
    verts, elems = _grid_mesh(d, cells, h)
    locM, locA = _element_matrices(verts, elems, d, D, c)
    npts = cells + 1
    ctr = cells // 2
    if d == 1:
        inner = np.arange(1, npts - 1)
        center = ctr
        nb = {"cy": center + 1}
    else:
        gi, gj = np.meshgrid(np.arange(npts), np.arange(npts), indexing="ij")
        inner = np.nonzero(((gi > 0) & (gi < npts - 1) & (gj > 0) & (gj < npts - 1)).ravel())[0]
        center = ctr * npts + ctr
        nb = {"cx": center + npts, "cy": center + 1, "cd": center + npts + 1}
    out = []
    for loc in (locM, locA):
        A = _assembled(verts, elems, loc)
        A = A[inner][:, inner].tocsr()
        A = ((A + A.T) / 2).tocsr()
        pos = {v: k for k, v in enumerate(inner)}
        row = A[pos[center]]
        vals = dict(zip(row.indices.tolist(), row.data.tolist()))
        st = {"c0": vals.get(pos[center], 0.0)}
        for key, v in nb.items():
            st[key] = vals.get(pos[v], 0.0) if v in pos else 0.0
        out.append(st)
    return out[0], out[1]


def stencil_vector(st, d):
    """[centre, x, y, diagonal] as the C ABI expects it."""
    if d == 1:
        return np.array([st["c0"], 0.0, st.get("cy", 0.0), 0.0])
    return np.array([st["c0"], st.get("cx", 0.0), st.get("cy", 0.0), st.get("cd", 0.0)])


def operator_list(J, alpha):
    """(alpha, mu) of operator 0 = K_x and 1 + j = C_j (solver.py:372-377)."""
    return [(1.0, 0.0)] + [(alpha, 2.0 ** j) for j in range(J + 1)]


def coef_table(d, J, K, alpha, D=None, c=0.0):
    """[(J+2), K+1, 8] coefficients of alpha*A_l + mu*M_l per operator/level."""
    table = np.zeros((J + 2, K + 1, COEF_STRIDE))
    sts = [level_stencils(d, l, D, c) for l in range(1, K + 1)]
    for o, (a, mu) in enumerate(operator_list(J, alpha)):
        for l, (M, A) in enumerate(sts, start=1):
            # scipy's alpha*A + mu*M: an entry missing from one operand
            # contributes an exact 0.0 to the sum
            vals = {key: a * A.get(key, 0.0) + mu * M.get(key, 0.0)
                    for key in ("c0", "cx", "cy", "cd")}
            c0 = vals["c0"]
            table[o, l, :6] = [c0, vals["cx"], vals["cy"], vals["cd"], 1.0 / c0,
                               1.0 / c0 if l == 1 else 0.0]
    return table


def temporal_values(J):
    """The 11 band values of hwg_desc.temporal (temporal.py:82-144)."""
    h = 2.0 ** -J
    sq = np.sqrt(h)
    return np.array([h / 6, 2 * h / 3, h / 3,
                     -1.0 / h, 2.0 / h, 1.0 / h,
                     0.5, 0.5,
                     1.0 / sq, sq / 2, np.sqrt(3 * h) / 6])


def wavelet_scales(J):
    return np.array([2.0 ** (j / 2.0) for j in range(1, J + 1)])


def level_of(J):
    """Wavelet level of every temporal coordinate (wavelet.py:83-85)."""
    lv = np.zeros(2 ** J + 1, dtype=np.int64)
    for j in range(1, J + 1):
        lv[2 ** (j - 1) + 1: 2 ** j + 1] = j
    return lv


# --------------------------------------------------------------------------
# data moments on the finest mesh (spatial.py:232-300)
# --------------------------------------------------------------------------
_QUAD = {
    1: (np.array([[0.5 + 0.5 / np.sqrt(3), 0.5 - 0.5 / np.sqrt(3)],
                  [0.5 - 0.5 / np.sqrt(3), 0.5 + 0.5 / np.sqrt(3)]]),
        np.array([0.5, 0.5])),
    2: (np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5]]),
        np.array([1 / 3, 1 / 3, 1 / 3])),
}


class FineMesh:
    """The finest level's mesh with its interior numbering.

    ``domain="L"``: the mapped L-shaped domain [0,1]^2 minus [1/2,1]^2 (the
    square's vertices and element order, removed-quadrant cells dropped)."""

    def __init__(self, d, K, domain="square"):
        if d not in (1, 2):
            raise ValueError("the GPU path supports d = 1, 2")
        if domain not in ("square", "L") or (domain == "L" and d != 2):
            raise ValueError("domain must be 'square' or (2D) 'L'")
        self.d, self.K, self.domain = d, K, domain
        n = 2 ** K
        verts, elems = _grid_mesh(d, n, 1.0)
        self.vertices = verts / n
        gi = np.rint(self.vertices * n).astype(int)
        if domain == "L":
            self.elements = _lshape_filter(elems, n)
            self.interior = np.nonzero(lshape_interior(gi, n))[0]
        else:
            self.elements = elems
            self.interior = np.nonzero(np.all((gi > 0) & (gi < n), axis=1))[0]
        self.interior_index = np.full(len(self.vertices), -1, dtype=np.int64)
        self.interior_index[self.interior] = np.arange(len(self.interior))

    @property
    def level(self):          # the reference's Mesh.level (spatial.py:49-64)
        return self.K

    @property
    def h(self):
        return 2.0 ** -self.K

    @property
    def n_interior(self):
        return len(self.interior)

    def quadrature(self):
        bary, w = _QUAD[self.d]
        v = self.vertices[self.elements]
        pts = np.einsum("qk,ekd->eqd", bary, v)
        E = v[:, 1:, :] - v[:, :1, :]
        vol = np.abs(np.linalg.det(E)) / math.factorial(self.d)
        return pts, bary, w, vol


def project_initial(mesh: FineMesh, u0) -> np.ndarray:
    """<u0, phi_i> on interior P1 hats by the degree-2 element rule."""
    pts, bary, w, vol = mesh.quadrature()
    vals = np.asarray(u0(pts.reshape(-1, mesh.d))).reshape(pts.shape[:2])
    loc = np.einsum("eq,ql,q->el", vals, bary, w) * vol[:, None]
    out = np.zeros(len(mesh.vertices))
    np.add.at(out, mesh.elements.ravel(), loc.ravel())
    return out[mesh.interior]


def assemble_load(mesh: FineMesh, J: int, g) -> np.ndarray:
    """<g, xi_i (x) phi_j> against the per-element Legendre test basis
    (2-point Gauss in time, degree-2 rule in space); rows = 2*2^J."""
    n = 2 ** J
    ht = 1.0 / n
    pts, bary, w, vol = mesh.quadrature()
    nq = len(w)
    flat = pts.reshape(-1, mesh.d)
    nv = len(mesh.vertices)
    gp = 0.5 / np.sqrt(3)
    tq = np.array([0.5 - gp, 0.5 + gp])
    tw = np.array([0.5, 0.5])
    out = np.zeros((2 * n, mesh.n_interior))
    for k in range(n):
        for q in range(2):
            t = (k + tq[q]) * ht
            gv = np.asarray(g(t, flat)).reshape(-1, nq)
            loc = np.einsum("eq,ql,q->el", gv, bary, w) * vol[:, None]
            sv = np.zeros(nv)
            np.add.at(sv, mesh.elements.ravel(), loc.ravel())
            sv = sv[mesh.interior]
            wt = tw[q] * ht
            out[2 * k] += wt * (1.0 / np.sqrt(ht)) * sv
            out[2 * k + 1] += wt * (np.sqrt(3.0 / ht) * (2 * tq[q] - 1)) * sv
    return out


def l2_error_on_mesh(mesh: FineMesh, coeffs, exact) -> float:
    """L2(Omega) distance of a P1 interior field to a callable (spatial.py:303-313)."""
    pts, bary, w, vol = mesh.quadrature()
    full = np.zeros(len(mesh.vertices))
    full[mesh.interior] = coeffs
    nodal = full[mesh.elements]
    uh = np.einsum("el,ql->eq", nodal, bary)
    ue = np.asarray(exact(pts.reshape(-1, mesh.d))).reshape(uh.shape)
    err2 = np.einsum("eq,q->e", (uh - ue) ** 2, w) * vol
    return float(np.sqrt(err2.sum()))


def lshape_problem(u0=None, g=None, c=0.0):
    """BASELINE cfg 5 in the mapped coordinates the GPU path uses.

    u_t - Laplace u = f on [-1,1]^2 minus [0,1]^2 becomes, under x -> (x+1)/2,
    u_t - div(D grad u) = f on [0,1]^2 minus [1/2,1]^2 with D = I/4.  In 2D
    the mapped M_x is 1/4 of the original and A_x (D = I/4) too, so the
    mapped S-hat and f-hat are 1/4 and K_X 4x the original ones: PCG
    iterates, iteration counts and the rtol stopping rule are unchanged."""
    zero = lambda pts: np.zeros(len(pts))  # noqa: E731
    return ProblemData(D=0.25 * np.eye(2), c=c, u0=u0 if u0 is not None else zero, g=g)
