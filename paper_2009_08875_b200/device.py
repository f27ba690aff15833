"""One GPU context per assembled space-time system (the hwg_ctx handle).

torch is used only as plumbing: device buffers, the current CUDA stream and
host<->device copies.  All arithmetic happens in libhwgpu.so.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from . import discretization as disc


def _torch():
    import torch
    return torch


def require_cuda(device=0):
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2009_08875_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", device)


def as_device(X, device, dtype=None):
    """(contiguous fp64 CUDA tensor, was_host) for a numpy array or tensor."""
    torch = _torch()
    if isinstance(X, torch.Tensor):
        if X.device.type != "cuda":
            return X.to(device=device, dtype=torch.float64).contiguous(), True
        if X.dtype != torch.float64 or not X.is_contiguous():
            X = X.to(dtype=torch.float64).contiguous()
        return X, False
    arr = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
    return torch.from_numpy(arr).to(device), True


def ptr(t):
    return C.c_void_p(t.data_ptr())


def stream_handle(device):
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class GpuContext:
    """Owns one hwg_ctx: tables, workspaces and the launch counter."""

    def __init__(self, d, J, K, alpha=0.3, vcycles=2, smooth=3, D=None, c=0.0,
                 device=0, coef=None, rows_max=0, domain="square", coarse_inv=None):
        if domain not in ("square", "L"):
            raise ValueError("domain must be 'square' or 'L'")
        self.device = require_cuda(device)
        self.lib = _lib.load()
        self.d, self.J, self.K = d, J, K
        self.alpha = alpha
        self.domain = domain
        self.n_t = 2 ** J + 1
        self.m = 2 ** K - 1
        self.n_grid = self.m ** d                     # points per row of the grid layout
        self.n_x = disc.lshape_dofs(K) if domain == "L" else self.n_grid
        self.coef = np.ascontiguousarray(
            disc.coef_table(d, J, K, alpha, D, c) if coef is None else coef, dtype=np.float64)
        self.coarse_inv = None
        if domain == "L":
            self.coarse_inv = np.ascontiguousarray(
                disc.lshape_coarse_inverses(disc.operator_list(J, alpha), D, c)
                if coarse_inv is None else coarse_inv, dtype=np.float64)
        Mf, Af = disc.level_stencils(d, K, D, c)
        self.stencil_M = disc.stencil_vector(Mf, d)
        self.stencil_A = disc.stencil_vector(Af, d)
        self.temporal = disc.temporal_values(J)
        self.scales = disc.wavelet_scales(J)
        desc = _lib.HwgDesc(dim=d, J=J, K=K, vcycles=vcycles, smooth=smooth,
                            device=self.device.index or 0, alpha=alpha,
                            coef=self.coef.ctypes.data, stencil_M=self.stencil_M.ctypes.data,
                            stencil_A=self.stencil_A.ctypes.data,
                            temporal=self.temporal.ctypes.data,
                            wavelet_scale=self.scales.ctypes.data, rows_max=int(rows_max),
                            domain=1 if domain == "L" else 0,
                            coarse_inv=self.coarse_inv.ctypes.data if self.coarse_inv is not None else None)
        h = C.c_void_p()
        _lib.check(self.lib.hwg_create(C.byref(desc), C.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self.lib.hwg_destroy(h)
            self.handle = None

    # ---- raw entry points on CUDA tensors ---------------------------------
    def stream(self):
        return stream_handle(self.device)

    @property
    def launches(self):
        return int(self.lib.hwg_launch_count(self.handle))

    @property
    def workspace_bytes(self):
        return int(self.lib.hwg_workspace_bytes(self.handle))

    PROFILE_CLASSES = ("mg2d_down_finest", "mg2d_up_finest", "mg2d_down_coarser",
                       "mg2d_up_coarser", "mg2d_coarse", "mg1d")

    profiling = False

    def profile_enable(self, on=True):
        _lib.check(self.lib.hwg_profile_enable(self.handle, int(on)))
        self.profiling = bool(on)

    def profile_read(self):
        """{class: (ms, bytes, launches)} since profile_enable."""
        out = {}
        for k, name in enumerate(self.PROFILE_CLASSES):
            ms, by, n = C.c_double(), C.c_double(), C.c_int64()
            _lib.check(self.lib.hwg_profile_read(self.handle, k, C.byref(ms), C.byref(by),
                                                 C.byref(n)))
            out[name] = (ms.value, by.value, n.value)
        return out

    # ---- time-slab building blocks (distributed path) ----------------------
    def syn_stage(self, j, C, c0, Dw, d0, Y, f0, nf, Dh=None):
        _lib.check(self.lib.hwg_syn_stage(self.handle, j, ptr(C), c0, ptr(Dw), d0,
                                          ptr(Dh) if Dh is not None else None, ptr(Y), f0, nf,
                                          self.stream()))

    def ana_stage(self, j, X, x0, C, c0, nc, Dw, d0, nd):
        _lib.check(self.lib.hwg_ana_stage(self.handle, j, ptr(X), x0,
                                          ptr(C) if nc else None, c0, nc,
                                          ptr(Dw) if nd else None, d0, nd, self.stream()))

    def bside_rows(self, U, u0, T1, T2, r0, nr, E0=None):
        _lib.check(self.lib.hwg_bside_rows(self.handle, ptr(U), u0, U.shape[0], ptr(T1), ptr(T2),
                                           r0, nr, ptr(E0) if E0 is not None else None,
                                           self.stream()))

    def bt_rows(self, G1, G2, E0, out):
        _lib.check(self.lib.hwg_bt_rows(self.handle, ptr(G1), ptr(G2),
                                        ptr(E0) if E0 is not None else None, ptr(out),
                                        out.shape[0], self.stream()))

    BANDS = {"Mt": 0, "At": 1, "L": 2, "LT": 3, "T": 4, "TT": 5, "N": 6, "NT": 7}

    def temporal_rows(self, band, X, x0, Y, r0, nr):
        _lib.check(self.lib.hwg_temporal_rows(self.handle, self.BANDS[band], ptr(X), x0, ptr(Y),
                                              r0, nr, self.stream()))

    def set_schur_form(self, form):
        """"five_term" (default) or "test_space" for schur() and pcg()."""
        _lib.check(self.lib.hwg_set_schur_form(self.handle, {"five_term": 0, "test_space": 1}[form]))

    def grid_scatter(self, X, Y):
        """dof-layout rows X -> grid-layout rows Y (L-shaped domain)."""
        _lib.check(self.lib.hwg_grid_scatter(self.handle, ptr(X), ptr(Y), X.shape[0], self.stream()))

    def grid_gather(self, X, Y):
        """grid-layout rows X -> dof-layout rows Y."""
        _lib.check(self.lib.hwg_grid_gather(self.handle, ptr(X), ptr(Y), X.shape[0], self.stream()))

    def mg_rows_dev(self, ops, B, X):
        _lib.check(self.lib.hwg_mg_rows_dev(self.handle, ptr(ops), ptr(B), ptr(X), B.shape[0],
                                            self.stream()))

    def mg_rows_dev_dot(self, ops, B, X, Y, part):
        """X = MG(B) row-wise and part[r] = <Y[r], X[r]> (fused when possible)."""
        _lib.check(self.lib.hwg_mg_rows_dev_dot(self.handle, ptr(ops), ptr(B), ptr(X), B.shape[0],
                                                ptr(Y), ptr(part), self.stream()))

    def row_partials(self, X, Y, part):
        _lib.check(self.lib.hwg_row_partials(self.handle, ptr(X), ptr(Y), X.shape[0], ptr(part),
                                             self.stream()))

    def tree_sum(self, part, n, out):
        _lib.check(self.lib.hwg_tree_sum(self.handle, ptr(part), n, ptr(out), self.stream()))

    def axpy(self, a, X, Y):
        _lib.check(self.lib.hwg_axpy(self.handle, float(a), ptr(X), ptr(Y), X.numel(), self.stream()))

    def xpay(self, a, X, Y):
        _lib.check(self.lib.hwg_xpay(self.handle, float(a), ptr(X), ptr(Y), X.numel(), self.stream()))

    # device-resident PCG scalars (scal: [rho, pq, rho_new, alpha, beta, ...])
    def pcg_scalar(self, step, scal):
        _lib.check(self.lib.hwg_pcg_scalar(self.handle, int(step), ptr(scal), self.stream()))

    def pcg_update_wr(self, w, r, p, q, scal, do_w, do_r):
        _lib.check(self.lib.hwg_pcg_update_wr(self.handle, ptr(w), ptr(r), ptr(p), ptr(q), ptr(scal),
                                              p.numel(), int(do_w), int(do_r), self.stream()))

    def pcg_update_wp(self, w, p, z, scal, do_w):
        _lib.check(self.lib.hwg_pcg_update_wp(self.handle, ptr(w), ptr(p), ptr(z), ptr(scal),
                                              p.numel(), int(do_w), self.stream()))

    def sub(self, f, t, r):
        _lib.check(self.lib.hwg_sub(self.handle, ptr(f), ptr(t), ptr(r), f.numel(), self.stream()))

    def any_nonzero(self, X, flag):
        """flag (int32 device tensor) |= any(X != 0)."""
        _lib.check(self.lib.hwg_any_nonzero(self.handle, ptr(X), X.numel(), ptr(flag),
                                            self.stream()))

    def wavelet(self, X, Y, transpose):
        _lib.check(self.lib.hwg_wavelet(self.handle, ptr(X), ptr(Y), int(transpose), self.stream()))

    def spatial(self, which, X, Y):
        _lib.check(self.lib.hwg_spatial(self.handle, int(which), ptr(X), ptr(Y),
                                        X.shape[0], self.stream()))

    def schur(self, X, Y):
        _lib.check(self.lib.hwg_schur_apply(self.handle, ptr(X), ptr(Y), self.stream()))

    def kx(self, X, Y):
        _lib.check(self.lib.hwg_kx_apply(self.handle, ptr(X), ptr(Y), self.stream()))

    def mg_rows(self, op, B, X, ops_host=None):
        rows = B.shape[0]
        if ops_host is not None:
            ops_host = np.ascontiguousarray(ops_host, dtype=np.int32)
            if len(ops_host) != rows:
                raise ValueError("one operator id per row")
            op_ptr = C.c_void_p(ops_host.ctypes.data)
        else:
            op_ptr = None
        _lib.check(self.lib.hwg_mg_rows(self.handle, int(op), op_ptr, ptr(B), ptr(X), rows,
                                        self.stream()))

    def rhs(self, F, load, u0proj, fhat):
        _lib.check(self.lib.hwg_rhs(self.handle, ptr(F) if F is not None else None,
                                    ptr(load) if load is not None else None,
                                    ptr(u0proj) if u0proj is not None else None,
                                    ptr(fhat), self.stream()))

    def dot(self, X, Y):
        out = C.c_double()
        _lib.check(self.lib.hwg_dot(self.handle, ptr(X), ptr(Y), X.shape[0], C.byref(out),
                                    self.stream()))
        return out.value

    def _stats(self, max_iterations):
        cap = max_iterations + 1
        bufs = [np.zeros(cap), np.zeros(cap), np.zeros(cap)]
        st = _lib.HwgPcgStats(iterations=0, capacity=cap,
                              residual_norms=bufs[0].ctypes.data, alphas=bufs[1].ctypes.data,
                              betas=bufs[2].ctypes.data)
        return st, bufs

    def pcg(self, f, w, epsilon=0.0, rtol=0.0, max_iterations=200, recompute_every=50):
        """hwg_pcg; returns (stats dict, return code)."""
        st, bufs = self._stats(max_iterations)
        rc = self.lib.hwg_pcg(self.handle, ptr(f), ptr(w), float(epsilon), float(rtol),
                              int(max_iterations), int(recompute_every), C.byref(st),
                              self.stream())
        return self._unpack(st, bufs), rc

    def solve_host(self, fhat_host, u_host, epsilon=0.0, rtol=0.0, max_iterations=200,
                   recompute_every=50):
        """hwg_solve_host on host arrays (the end-to-end call)."""
        st, bufs = self._stats(max_iterations)
        rc = self.lib.hwg_solve_host(self.handle, C.c_void_p(fhat_host.ctypes.data),
                                     C.c_void_p(u_host.ctypes.data), float(epsilon),
                                     float(rtol), int(max_iterations), int(recompute_every),
                                     C.byref(st), self.stream())
        return self._unpack(st, bufs), rc

    @staticmethod
    def _unpack(st, bufs):
        k = st.iterations
        return dict(iterations=k, residual_norms=bufs[0][:k + 1].tolist(),
                    alphas=bufs[1][:k].tolist(), betas=bufs[2][:k].tolist(),
                    ms_schur=st.ms_schur, ms_precond=st.ms_precond, ms_vector=st.ms_vector,
                    ms_total=st.ms_total, epsilon=st.epsilon_used)
