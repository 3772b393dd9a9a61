"""lsb_ieskf_gain (host C++ in the product library) against the reference's
numpy algebra of one IESKF iteration (estimator.py:292-331), on random
well-conditioned and filter-like inputs; singular input raises."""
import ctypes

import numpy as np
import pytest


def _lib():
    from paper_2501_08672_b200 import _lib
    return _lib.load()


def _ref(cov, jinv, A6, b6, delta):
    Hj = np.eye(15)
    Hj[:3, :3] = jinv
    P = Hj @ cov @ Hj.T
    A = np.zeros((15, 15))
    A[:6, :6] = A6
    b = np.zeros(15)
    b[:6] = b6
    S_inv = np.linalg.inv(A + np.linalg.inv(P))
    K_H = S_inv @ A
    xi = -(S_inv @ b) - (np.eye(15) - K_H) @ (Hj @ delta)
    return xi, K_H, P


def _call(cov, jinv, A6, b6, delta):
    lib = _lib()
    p = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    args = [p(cov), p(jinv), p(A6), p(b6), p(delta)]
    xi, KH, P = np.empty(15), np.empty((15, 15)), np.empty((15, 15))
    rc = lib.lsb_ieskf_gain(*[a.ctypes.data_as(ctypes.c_void_p) for a in args + [xi, KH, P]])
    return rc, xi, KH, P


@pytest.mark.parametrize("seed,scale", [(0, 1.0), (1, 1e-6), (2, 1e-8)])
def test_gain_matches_numpy(seed, scale):
    rng = np.random.default_rng(seed)
    L = rng.normal(size=(15, 15))
    cov = scale * (L @ L.T + 15 * np.eye(15))
    th = rng.normal(size=3) * 0.01
    from paper_2501_08672_b200.geometry import so3_left_jacobian
    jinv = so3_left_jacobian(-th)
    Hr = rng.normal(size=(200, 6))
    A6 = Hr.T @ Hr * 100.0
    b6 = Hr.T @ rng.normal(size=200) * 100.0
    delta = rng.normal(size=15) * 1e-3
    rc, xi, KH, P = _call(cov, jinv, A6, b6, delta)
    assert rc == 0
    xr, KHr, Pr = _ref(cov, jinv, A6, b6, delta)
    assert np.abs(P - Pr).max() <= 1e-12 * np.abs(Pr).max()
    assert np.abs(KH - KHr).max() <= 1e-8 * max(np.abs(KHr).max(), 1.0)
    assert np.abs(xi - xr).max() <= 1e-8 * max(np.abs(xr).max(), 1e-12)


def test_singular_covariance_reports_error():
    rc, *_ = _call(np.zeros((15, 15)), np.eye(3), np.eye(6), np.zeros(6), np.zeros(15))
    assert rc != 0
    assert b"singular" in _lib().lsb_last_error()


@pytest.mark.parametrize("seed", range(4))
def test_iterate_matches_python_state_algebra(seed):
    """lsb_ieskf_iterate (boxminus, gain, boxplus on the state vectors) against
    the NavState / numpy restatement of one ieskf_update iteration."""
    from paper_2501_08672_b200.estimator import NavState, _pack, _unpack
    from paper_2501_08672_b200.geometry import SE3, so3_exp, so3_left_jacobian
    rng = np.random.default_rng(10 + seed)
    xb = NavState(SE3(so3_exp(rng.normal(size=3)), rng.normal(size=3)), rng.normal(size=3),
                  rng.uniform(-0.1, 0.1, 3), rng.uniform(-0.1, 0.1, 3))
    xh = xb.boxplus(rng.normal(size=15) * 1e-2)
    L = rng.normal(size=(15, 15))
    cov = 1e-4 * (L @ L.T + 15 * np.eye(15))
    Hr = rng.normal(size=(100, 6))
    A6, b6 = Hr.T @ Hr * 50.0, Hr.T @ rng.normal(size=100) * 5.0
    delta = xh.boxminus(xb)
    xr, KHr, Pr = _ref(cov, so3_left_jacobian(-delta[:3]), A6, b6, delta)
    ref = xh.boxplus(xr, bias_limit=0.5)
    lib = _lib()
    x_bar, x_hat = _pack(xb), _pack(xh)
    xi, KH, P = np.empty(15), np.empty((15, 15)), np.empty((15, 15))
    p = lambda a: np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(ctypes.c_void_p)
    assert lib.lsb_ieskf_iterate(p(cov), x_bar.ctypes.data_as(ctypes.c_void_p), x_hat.ctypes.data_as(ctypes.c_void_p),
                                 p(A6), p(b6), 0.5, xi.ctypes.data_as(ctypes.c_void_p),
                                 KH.ctypes.data_as(ctypes.c_void_p), P.ctypes.data_as(ctypes.c_void_p)) == 0
    assert np.abs(xi - xr).max() <= 1e-9 * max(np.abs(xr).max(), 1e-12)
    got = _unpack(x_hat)
    assert np.abs(got.T_WI.R - ref.T_WI.R).max() <= 1e-12
    assert np.abs(got.T_WI.t - ref.T_WI.t).max() <= 1e-12
    for a, b in ((got.velocity, ref.velocity), (got.bias_gyro, ref.bias_gyro), (got.bias_accel, ref.bias_accel)):
        assert np.abs(a - b).max() <= 1e-12
