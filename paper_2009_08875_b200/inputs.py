"""Seeded synthetic inputs for the BASELINE configurations.

No public dataset is involved: BASELINE.json fixes only shapes and value
distributions, so every input here is generated from a seed.

* forcing ``F``: nodal values on the full ``(N_t, N_x)`` space-time grid of
  interior spatial vertices.  The forcing ``g`` is the P1(time) x P1(space)
  interpolant of ``F``; its test-space load is exactly ``(N (x) M_x) F``.
* ``u0``: a callable of spatial points ``(npts, d) -> (npts,)``.

Rows are generated in fixed blocks of ``ROW_BLOCK`` temporal rows, each from
its own ``SeedSequence([seed, block])``.  The array is therefore identical no
matter how the rows are later split between GPUs or host threads.
"""

from __future__ import annotations

import numpy as np

ROW_BLOCK = 64

#: BASELINE.json configs -> (d, J, K, forcing distribution)
CONFIGS = {
    1: dict(d=2, J=4, K=4, dist="uniform"),
    2: dict(d=2, J=8, K=8, dist="uniform"),
    3: dict(d=1, J=20, K=10, dist="normal"),
    4: dict(d=2, J=10, K=10, dist="uniform"),
    # L-shaped [-1,1]^2 \ [0,1]^2, h = 2^-10, mapped to [0,1]^2 minus
    # [1/2,1]^2 (K = 11 there) with D = I/4 (see discretization.lshape_problem)
    5: dict(d=2, J=11, K=11, dist="lshape", domain="L"),
}

SEED_F = 0
SEED_U0 = 1


def _block(dist, seed, b, rows, n_x):
    rng = np.random.default_rng(np.random.SeedSequence([seed, b]))
    if dist == "uniform":
        return rng.uniform(-1.0, 1.0, (rows, n_x))
    if dist == "normal":
        return rng.standard_normal((rows, n_x))
    if dist == "lshape":                      # BASELINE cfg 5: 1 + U[-0.1, 0.1]
        return 1.0 + rng.uniform(-0.1, 0.1, (rows, n_x))
    raise ValueError(f"unknown distribution {dist!r}")


def forcing_rows(dist: str, n_t: int, n_x: int, r0: int, r1: int,
                 seed: int = SEED_F, out=None) -> np.ndarray:
    """Rows [r0, r1) of the seeded nodal forcing F (blockwise-seeded)."""
    if not 0 <= r0 <= r1 <= n_t:
        raise ValueError("row range out of bounds")
    out = np.empty((r1 - r0, n_x)) if out is None else out
    b0, b1 = r0 // ROW_BLOCK, (r1 + ROW_BLOCK - 1) // ROW_BLOCK
    for b in range(b0, b1):
        lo = b * ROW_BLOCK
        hi = min(lo + ROW_BLOCK, n_t)
        blk = _block(dist, seed, b, hi - lo, n_x)
        a, z = max(lo, r0), min(hi, r1)
        out[a - r0:z - r0] = blk[a - lo:z - lo]
    return out


def forcing(dist: str, n_t: int, n_x: int, seed: int = SEED_F) -> np.ndarray:
    return forcing_rows(dist, n_t, n_x, 0, n_t, seed)


def u0_sines(pts):
    """u0 = prod_i sin(pi x_i) (BASELINE cfg 1/2/4)."""
    return np.prod(np.sin(np.pi * pts), axis=1)


def u0_modes(seed: int = SEED_U0, modes: int = 8):
    """u0 = sum_{m=1}^{modes} c_m sin(m pi x), c ~ U[-1,1] (BASELINE cfg 3)."""
    c = np.random.default_rng(seed).uniform(-1.0, 1.0, modes)

    def u0(pts):
        x = np.asarray(pts)[:, 0]
        return sum(c[m] * np.sin((m + 1) * np.pi * x) for m in range(modes))

    return u0


def u0_zero(pts):
    """u0 = 0 (BASELINE cfg 5)."""
    return np.zeros(len(pts))


def u0_for(dist: str):
    return {"uniform": u0_sines, "normal": None, "lshape": u0_zero}[dist] or u0_modes()


def recipe(cfg: int):
    """(d, J, K, dist, u0 callable) of a BASELINE config."""
    c = CONFIGS[cfg]
    return c["d"], c["J"], c["K"], c["dist"], u0_for(c["dist"])


def u0_by_name(name: str):
    """The u0 callable a fixture records by name ("sines", "modes", "zero")."""
    return {"sines": u0_sines, "zero": u0_zero}.get(name) or u0_modes()
