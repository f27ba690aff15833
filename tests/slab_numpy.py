"""Test double for the time-slab kernels: each local operation is computed by
embedding the rank's rows into a global-size array and applying the CPU
oracle's restatement of the reference (same arithmetic order), so the
distributed orchestration can be checked BIT-FOR-BIT against the oracle.
Test infrastructure only."""
import numpy as np
import scipy.sparse as sp

from oracle import heatwave_oracle as O


def _np(t):
    return t.detach().numpy()


class NumpyKernels:
    def __init__(self, system: "O.System"):
        self.s = system
        self.nt, self.nx = system.shape
        self.stage = {j + 1: st for j, st in enumerate(system.wavelet.stages)}

    # --- wavelet stages with offsets -------------------------------------
    def syn_stage(self, j, C, c0, Dw, d0, Y, f0, nf, Dh=None):
        C, Dw, Y = _np(C), _np(Dw), _np(Y)
        nc, nfl = 2 ** (j - 1) + 1, 2 ** j + 1
        Xg = np.zeros((nfl, self.nx))
        for r in range(C.shape[0]):
            if 0 <= c0 + r < nc:
                Xg[c0 + r] = C[r]
        if Dh is not None and 0 <= d0 - 1 < nfl - nc:
            Xg[nc + d0 - 1] = _np(Dh)
        for r in range(Dw.shape[0]):
            if 0 <= d0 + r < nfl - nc:
                Xg[nc + d0 + r] = Dw[r]
        out = O.temporal(self.stage[j][0], Xg, np.empty((nfl, self.nx)))
        Y[:nf] = out[f0:f0 + nf]

    def ana_stage(self, j, X, x0, C, c0, nc_out, Dw, d0, nd):
        X = _np(X)
        nc, nfl = 2 ** (j - 1) + 1, 2 ** j + 1
        Xg = np.zeros((nfl, self.nx))
        for r in range(X.shape[0]):
            if 0 <= x0 + r < nfl:
                Xg[x0 + r] = X[r]
        out = O.temporal(self.stage[j][1], Xg, np.empty((nfl, self.nx)))
        if nc_out:
            _np(C)[:nc_out] = out[c0:c0 + nc_out]
        if nd:
            _np(Dw)[:nd] = out[nc + d0:nc + d0 + nd]

    # --- five-term pieces --------------------------------------------------
    def bside_rows(self, U, u0, T1, T2, r0, nr, E0=None):
        U = _np(U)
        s = self.s
        Ug = np.zeros((self.nt, self.nx))
        for r in range(U.shape[0]):
            if 0 <= u0 + r < self.nt:
                Ug[u0 + r] = U[r]
        MxU = O.spatial(s.Mx, Ug, np.empty_like(Ug))
        AxU = O.spatial(s.Ax, Ug, np.empty_like(Ug))
        t1, t2 = np.empty_like(Ug), np.empty_like(Ug)
        O.temporal(s.At, MxU, t1)
        O.temporal(s.LT, AxU, t2)
        O.axpy(1.0, t2, t1)
        _np(T1)[:nr] = t1[r0:r0 + nr]
        O.temporal(s.Mt, AxU, t1)
        O.temporal(s.L, MxU, t2)
        O.axpy(1.0, t2, t1)
        _np(T2)[:nr] = t1[r0:r0 + nr]
        if r0 == 0 and E0 is not None:
            _np(E0)[:] = MxU[0]

    def bt_rows(self, G1, G2, E0, out):
        s = self.s
        G1, G2, o = np.ascontiguousarray(_np(G1)), np.ascontiguousarray(_np(G2)), _np(out)
        res = O.spatial(s.Mx, G1, np.empty_like(G1))
        t2 = O.spatial(s.Ax, G2, np.empty_like(G2))
        O.axpy(1.0, t2, res)
        if E0 is not None:
            res[0] += _np(E0)
        o[:] = res

    def mg_rows_dev(self, ops, B, X):
        ops, B, X = _np(ops), np.ascontiguousarray(_np(B)), _np(X)
        res = np.empty_like(B)
        for op in np.unique(ops):
            rows = np.nonzero(ops == op)[0]
            mg = self.s.Kx if op == 0 else self.s.blocks[int(op) - 1]
            mg.apply_rows(B, res, rows)
        X[:] = res

    def spatial(self, which, X, Y):
        A = self.s.Mx if which == 0 else self.s.Ax
        _np(Y)[:] = O.spatial(A, np.ascontiguousarray(_np(X)), np.empty(tuple(X.shape)))

    # --- vectors -----------------------------------------------------------
    def mg_rows_dev_dot(self, ops, B, X, Y, part):
        self.mg_rows_dev(ops, B, X)
        self.row_partials(Y, X, part)

    def row_partials(self, X, Y, part):
        x, y = np.ascontiguousarray(_np(X)), np.ascontiguousarray(_np(Y))
        p = np.empty(x.shape[0])
        O.lib().or_col_dots(O._p(x), O._p(y), O._p(p), x.shape[1], 0, x.shape[0])
        _np(part)[:] = p

    def tree_sum(self, part, n, res):
        v = np.ascontiguousarray(_np(part)[:n])
        _np(res)[0] = O.lib().or_tree_reduce(O._p(v), n, O._p(np.empty(n)))

    def axpy(self, a, X, Y):
        O.axpy(a, np.ascontiguousarray(_np(X)), _np(Y))

    def xpay(self, a, X, Y):
        O.xpay(a, np.ascontiguousarray(_np(X)), _np(Y))

    # --- device-scalar PCG steps (hwg_pcg_scalar / _update_wr / _update_wp)
    def pcg_scalar(self, step, scal):
        s = _np(scal)
        if step == 0:
            s[3] = s[0] / s[1]
        else:
            s[4] = s[2] / s[0]
            s[0] = s[2]

    def pcg_update_wr(self, w, r, p, q, scal, do_w, do_r):
        a = float(_np(scal)[3])
        if do_w:
            self.axpy(a, p, w)
        if do_r:
            self.axpy(-a, q, r)

    def pcg_update_wp(self, w, p, z, scal, do_w):
        s = _np(scal)
        if do_w:
            self.axpy(float(s[3]), p, w)
        self.xpay(float(s[4]), z, p)

    def sub(self, f, t, r):
        _np(r)[:] = _np(f) - _np(t)

    def any_nonzero(self, X, flag):
        _np(flag)[0] |= int(np.any(_np(X)))

    # --- temporal factor on a row range (distributed RHS) --------------------
    def temporal_rows(self, band, X, x0, Y, r0, nr):
        s = self.s
        B = {"Mt": s.Mt, "At": s.At, "L": s.L, "LT": s.LT, "T": s.T, "TT": s.T.T,
             "N": s.N, "NT": s.N.T}[band]
        X = _np(X)
        Xg = np.zeros((B.shape[1], self.nx))
        for r in range(X.shape[0]):
            if 0 <= x0 + r < B.shape[1]:
                Xg[x0 + r] = X[r]
        out = O.temporal(B, Xg, np.empty((B.shape[0], self.nx)))
        _np(Y)[:nr] = out[r0:r0 + nr]
