"""The reference's own temporal / wavelet-construction tests
(/root/reference/pkg/tests/test_temporal.py, test_wavelet.py; cited per
test) run against the drop-in package's host containers, imported under the
reference's name (CPU only: these are the setup-side objects)."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2009_08875_b200 as heatwave
from paper_2009_08875_b200 import structures as st

hw = heatwave


def test_dimensions():                                               # test_temporal.py:8-15
    for J in range(0, 7):
        d = hw.TemporalDiscretization(J)
        assert d.N_t == 2 ** J + 1 and d.mesh_width == 2.0 ** -J
    with pytest.raises(ValueError):
        hw.TemporalDiscretization(-1)


def test_trial_single_element_literals():                            # test_temporal.py:18-25
    tm = hw.assemble_temporal_trial(0)
    assert np.allclose(tm.M_t.to_dense(), [[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    assert np.allclose(tm.A_t.to_dense(), [[1, -1], [-1, 1]])
    assert np.allclose(tm.L.to_dense(), [[-0.5, 0.5], [-0.5, 0.5]])
    assert np.array_equal(tm.Gamma0.to_dense(), [[1.0, 0.0], [0.0, 0.0]])


def test_mass_row_sums_and_stiffness_kernel():                        # test_temporal.py:27-41
    for J in (0, 2, 4):
        h = 2.0 ** -J
        M = hw.assemble_temporal_trial(J).M_t.to_dense()
        want = np.full(2 ** J + 1, h)
        want[0] = want[-1] = h / 2
        assert np.allclose(M.sum(axis=1), want, atol=1e-15)
        assert abs(M.sum() - 1.0) <= 1e-14
    for J in (0, 3, 5):
        A = hw.assemble_temporal_trial(J).A_t
        assert np.abs(A.to_scipy() @ np.ones(A.rows)).max() == 0.0


def test_integration_by_parts_and_spd():                              # test_temporal.py:43-58
    for J in range(0, 7):
        tm = hw.assemble_temporal_trial(J)
        L = tm.L.to_dense()
        gT, g0 = np.outer(tm.phi_at_T, tm.phi_at_T), np.outer(tm.phi_at_0, tm.phi_at_0)
        assert np.abs(L + L.T - (gT - g0)).max() <= 1e-14
    tm = hw.assemble_temporal_trial(4)
    assert np.linalg.eigvalsh(tm.M_t.to_dense()).min() > 0
    ev = np.linalg.eigvalsh(tm.A_t.to_dense())
    assert ev[0] >= -1e-13 and ev[1] > 0
    G0 = tm.Gamma0.to_scipy()
    assert G0.nnz == 1 and G0[0, 0] == 1.0


def test_test_matrices():                                             # test_temporal.py:61-101
    ts = hw.assemble_temporal_test(0)
    assert np.array_equal(ts.O.to_dense(), np.eye(2))
    assert np.allclose(ts.T.to_dense(), [[-1.0, 1.0], [0.0, 0.0]])
    s3 = np.sqrt(3) / 6
    assert np.allclose(ts.N.to_dense(), [[0.5, 0.5], [-s3, s3]])
    assert np.diff(hw.assemble_temporal_test(4).T.to_scipy().tocsc().indptr).max() <= 2
    for J in range(0, 7):
        tm, ts = hw.assemble_temporal_trial(J), hw.assemble_temporal_test(J)
        T, N, O = ts.T.to_dense(), ts.N.to_dense(), ts.O.to_dense()
        assert np.abs(O - np.eye(O.shape[0])).max() <= 1e-14
        Oi = np.linalg.inv(O)
        assert np.abs(T.T @ Oi @ N - tm.L.to_dense().T).max() <= 1e-13
        assert np.abs(N.T @ Oi @ N - tm.M_t.to_dense()).max() <= 1e-13
        assert np.abs(T.T @ Oi @ T - tm.A_t.to_dense()).max() <= 1e-13
        Mt, At = tm.M_t.to_dense(), tm.A_t.to_dense()
        for j in range(2 ** J + 1):
            assert abs(Mt[j, j] - (N[:, j] ** 2).sum()) <= 1e-13
            assert abs(At[j, j] - (T[:, j] ** 2).sum()) <= 1e-13


def test_trace():                                                     # test_temporal.py:104-117
    assert np.array_equal(hw.evaluate_trace(3, 0.0), np.eye(9)[0])
    assert np.array_equal(hw.evaluate_trace(3, 1.0), np.eye(9)[8])
    with pytest.raises(ValueError):
        hw.evaluate_trace(3, 0.5)
    v = hw.evaluate_trace(4, 0.0)
    assert np.array_equal(np.outer(v, v), hw.assemble_temporal_trial(4).Gamma0.to_dense())


def test_wavelet_construction():                                      # test_wavelet.py:14-58
    lv = hw.build_wavelet(3)
    assert np.array_equal(lv.level_of, [0, 0, 1, 2, 2, 3, 3, 3, 3])
    assert np.array_equal(lv.dims, [2, 3, 5, 9])
    assert np.array_equal(lv.scaling_weights(), 2.0 ** lv.level_of)
    sigmas = []
    for j in range(1, 9):
        P, Q = (m.to_scipy() for m in hw.build_wavelet(j).two_scale[j - 1])
        assert np.diff(Q.tocsc().indptr).max() <= 3 and np.diff(P.tocsc().indptr).max() <= 3
        assert np.diff(P.indptr).max() <= 2 and set(np.round(P.data, 12)) <= {0.5, 1.0}
        M = sp.hstack([P, Q]).toarray()
        assert M.shape == (2 ** j + 1, 2 ** j + 1)
        sigmas.append(np.linalg.svd(M, compute_uv=False)[-1])
    assert min(sigmas) >= 0.5
    for j in (1, 2, 4, 6):
        Q = hw.build_wavelet(j).two_scale[j - 1][1].to_scipy()
        Mt = hw.assemble_temporal_trial(j).M_t.to_scipy()
        assert np.abs(np.diag((Q.T @ Mt @ Q).toarray()) - 2.0 / 3.0).max() <= 1e-13
    for j in (1, 2, 3, 5):
        Q = hw.build_wavelet(j).two_scale[j - 1][1].to_dense()
        h = 2.0 ** -j
        w = np.full(2 ** j + 1, h)
        w[0] = w[-1] = h / 2
        assert np.abs(w @ Q).max() <= 1e-13


def test_riesz_stability():                                           # test_wavelet.py:118-140
    k2, kh = [], []
    for J in range(3, 9):
        lv = hw.build_wavelet(J)
        W = st.dense_transform(lv)
        tm = hw.assemble_temporal_trial(J)
        k2.append(np.linalg.cond(W.T @ tm.M_t.to_dense() @ W))
        G = W.T @ (tm.A_t.to_dense() + tm.M_t.to_dense()) @ W
        Dinv = np.diag(2.0 ** -lv.level_of.astype(float))
        kh.append(np.linalg.cond(Dinv @ G @ Dinv))
    assert max(k2) / min(k2) <= 1.3 and max(k2) <= 6.0
    assert max(kh) / min(kh) <= 1.3 and max(kh) <= 25.0
