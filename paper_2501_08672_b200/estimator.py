"""Visual (photometric) IESKF measurement on the B200 — drop-in for the
visual part of livsplat.estimator (estimator.py:241-331).

select_semi_dense_pixels, visual_measurement and Measurement keep the
reference's names, arguments and TooFewPixels behaviour.  The render, the
semi-dense mask, the residual gate and the pose rows run on the GPU; `hb()`
additionally reduces the pose block of H^T R^-1 H and H^T R^-1 z on the
device (the only products of the measurement the 15-dim filter update
needs).  The 15x15 filter algebra itself (ieskf_update) is tiny host math
and out of scope.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import NoAssociations, SingularGain, TooFewPixels
from .geometry import SE3, so3_exp, so3_log
from .raster import (_CAP_HINT, RasterSettings, RenderState, _as_arrays, _degree_used, _f32, _observed, pose_rows,
                     render)

DIM = 15


@dataclass
class FilterConfig:
    """estimator.FilterConfig (estimator.py:100-115): same fields, order and
    defaults, so a config loaded for the reference drives this package.  The
    IMU noise fields belong to imu_propagate (out of scope) and are carried
    for schema compatibility only."""

    gyro_noise: float = 1e-3
    accel_noise: float = 1e-2
    gyro_bias_rw: float = 1e-5
    accel_bias_rw: float = 1e-4
    lidar_sigma: float = 0.02
    photo_sigma: float = 0.1
    lidar_gate: float = 1.0
    pixel_budget: int = 1024
    grad_threshold: float = 0.05
    photo_gate: float = 0.15
    min_pixels: int = 50
    max_iter: int = 5
    visual_max_iter: int = 2
    step_tol: float = 1e-6
    bias_limit: float = 0.5
    coverage_max_transmittance: float = 0.9


@dataclass
class NavState:
    """Filter state (estimator.py:45-83): pose, velocity, biases; 15-dim
    error state (d_rho, d_tau, d_v, d_bg, d_ba) with the boxplus retraction."""

    T_WI: SE3 = field(default_factory=SE3.identity)
    velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))
    bias_gyro: np.ndarray = field(default_factory=lambda: np.zeros(3))
    bias_accel: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def clone(self) -> "NavState":
        return NavState(SE3(self.T_WI.R.copy(), self.T_WI.t.copy()), np.array(self.velocity, float).copy(),
                        np.array(self.bias_gyro, float).copy(), np.array(self.bias_accel, float).copy())

    def boxplus(self, xi, bias_limit: float = 0.5) -> "NavState":
        xi = np.asarray(xi, dtype=float)
        return NavState(SE3(self.T_WI.R @ so3_exp(xi[0:3]), self.T_WI.t + xi[3:6]), self.velocity + xi[6:9],
                        np.clip(self.bias_gyro + xi[9:12], -bias_limit, bias_limit),
                        np.clip(self.bias_accel + xi[12:15], -bias_limit, bias_limit))

    def boxminus(self, other: "NavState") -> np.ndarray:
        return np.concatenate([so3_log(other.T_WI.R.T @ self.T_WI.R), self.T_WI.t - other.T_WI.t,
                               self.velocity - other.velocity, self.bias_gyro - other.bias_gyro,
                               self.bias_accel - other.bias_accel])


class Measurement:
    """Stacked residuals with pose Jacobian rows padded to the full state
    (estimator.py:84-92).  The device measurements keep rows_dev (= -H[:, :6])
    and z_dev on the GPU; the numpy z / H / R_diag the reference exposes are
    materialised on first access, so an IESKF step that only needs hb() never
    copies the rows to the host."""

    def __init__(self, z=None, H=None, R_diag=None, rows_dev: torch.Tensor = None, z_dev: torch.Tensor = None,
                 sigma2: float = None, keep_dev: torch.Tensor = None, count: int = None):
        self._z = None if z is None else np.asarray(z, dtype=float).reshape(-1)
        self._H = None if H is None else np.asarray(H, dtype=float).reshape(-1, DIM)
        self._R = None if R_diag is None else np.asarray(R_diag, dtype=float).reshape(-1)
        self.rows_dev, self.z_dev, self.sigma2 = rows_dev, z_dev, sigma2
        # keep_dev: the device rows are every input point's, the kept ones
        # marked (dropped rows are zero, so hb() needs no compaction); z / H
        # are the kept rows in scan order
        self.keep_dev, self._count = keep_dev, count

    def __len__(self) -> int:
        if self._count is not None:
            return int(self._count)
        return int(self.z_dev.numel()) if self.z_dev is not None else len(self._z)

    def _kept(self, t: torch.Tensor) -> np.ndarray:
        a = t.cpu().numpy()
        return a if self.keep_dev is None else a[self.keep_dev.cpu().numpy().astype(bool)]

    @property
    def z(self) -> np.ndarray:
        if self._z is None:
            self._z = self._kept(self.z_dev)
        return self._z

    @property
    def H(self) -> np.ndarray:
        if self._H is None:
            H = np.zeros((len(self), DIM))
            H[:, :6] = -self._kept(self.rows_dev)
            self._H = H
        return self._H

    @property
    def R_diag(self) -> np.ndarray:
        if self._R is None:
            self._R = np.full(len(self), float(self.sigma2))
        return self._R

    def hb(self) -> tuple[np.ndarray, np.ndarray]:
        """(6x6 sum h h^T / sigma^2, 6 sum h z / sigma^2) for the pose block,
        reduced on the device (estimator.py:314-318 with H = -rows)."""
        m = int(self.z_dev.numel())          # (with keep_dev: every point's row, dropped ones zero)
        inv = 1.0 / (self.sigma2 if self.sigma2 is not None else float(self.R_diag[0])) if len(self) else 1.0
        lib = _lib.load()
        out = torch.empty(42, dtype=torch.float64, device=self.z_dev.device)
        scratch = torch.empty(lib.lsb_hb_scratch_doubles(), dtype=torch.float64, device=self.z_dev.device)
        _lib.check(lib.lsb_hb_reduce(ctypes.c_void_p(self.rows_dev.data_ptr()), ctypes.c_void_p(self.z_dev.data_ptr()),
                                     m, None, float(inv), ctypes.c_void_p(out.data_ptr()),
                                     ctypes.c_void_p(scratch.data_ptr()), _lib.stream_ptr()), "hb_reduce")
        o = out.cpu().numpy()
        return o[:36].reshape(6, 6), o[36:]


def select_semi_dense_pixels(observed, coverage_t, cfg: FilterConfig) -> np.ndarray:
    """High-gradient, covered pixels, uniformly subsampled to the budget
    (estimator.py:241-257).  Returns flat ids (numpy int64)."""
    _lib.require()
    dev = coverage_t.device if torch.is_tensor(coverage_t) and coverage_t.is_cuda else torch.device("cuda")
    h, w = int(np.shape(coverage_t)[0]), int(np.shape(coverage_t)[1])
    obs = _observed(observed, (h, w, 3), dev)
    tf = _f32(coverage_t, (h, w), dev)
    mask = torch.empty((h, w), dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().lsb_semidense_mask(ctypes.c_void_p(obs.data_ptr()), int(obs.dtype == torch.uint8),
                                              ctypes.c_void_p(tf.data_ptr()), w, h,
                                              float(cfg.grad_threshold), float(cfg.coverage_max_transmittance),
                                              ctypes.c_void_p(mask.data_ptr()), _lib.stream_ptr()), "semidense")
    ids = torch.nonzero(mask.view(-1)).view(-1).cpu().numpy()
    if len(ids) > cfg.pixel_budget:
        take = np.round(np.linspace(0, len(ids) - 1, cfg.pixel_budget)).astype(int)
        ids = ids[np.unique(take)]
    return ids


def visual_measurement(state, observed, window, cam, T_ic, cfg: FilterConfig,
                       settings: RasterSettings) -> Measurement:
    """Photometric residuals I(u) - I_hat(u) on semi-dense pixels
    (estimator.py:260-280)."""
    T_wc = state.T_WI @ T_ic
    # contributing-list binning when alpha_cut > 0: the same image, T and pose
    # rows (the dropped entries never composite), fewer tile entries
    out = render(window, T_wc, cam, settings, bin_mode=1 if settings.alpha_cut > 0 else 0)
    dev = out.image.device
    h, w = int(cam.height), int(cam.width)
    obs = _observed(observed, (h, w, 3), dev)
    u8 = int(obs.dtype == torch.uint8)
    # semi-dense mask, then selection + residual + gate in one device pass;
    # one small read-back for the counts the reference's exceptions need
    lib = _lib.load()
    npx = h * w
    mask = torch.empty(npx, dtype=torch.uint8, device=dev)
    _lib.check(lib.lsb_semidense_mask(ctypes.c_void_p(obs.data_ptr()), u8,
                                      ctypes.c_void_p(out.final_transmittance.data_ptr()), w, h,
                                      float(cfg.grad_threshold), float(cfg.coverage_max_transmittance),
                                      ctypes.c_void_p(mask.data_ptr()), _lib.stream_ptr()), "semidense")
    budget = int(cfg.pixel_budget)
    scratch = torch.empty(int(lib.lsb_visual_select_scratch_bytes(npx, budget)), dtype=torch.uint8, device=dev)
    ids = torch.empty(budget, dtype=torch.int32, device=dev)
    res = torch.empty(budget, dtype=torch.float64, device=dev)
    counts = torch.empty(3, dtype=torch.int64, device=dev)
    _lib.check(lib.lsb_visual_select(ctypes.c_void_p(mask.data_ptr()), ctypes.c_void_p(obs.data_ptr()), u8,
                                     ctypes.c_void_p(out.image.data_ptr()), npx, budget, float(cfg.photo_gate),
                                     ctypes.c_void_p(scratch.data_ptr()), ctypes.c_void_p(ids.data_ptr()),
                                     ctypes.c_void_p(res.data_ptr()), ctypes.c_void_p(counts.data_ptr()),
                                     _lib.stream_ptr()), "visual_select")
    _, n_sel, n_ok = (int(v) for v in counts.cpu())
    if n_sel < cfg.min_pixels:
        raise TooFewPixels(f"{n_sel} < {cfg.min_pixels}")
    if n_ok < cfg.min_pixels:
        raise TooFewPixels(f"{n_ok} < {cfg.min_pixels} after gating")
    idt = ids[:n_ok]
    res = res[:n_ok].contiguous()
    rows = pose_rows(out, idt, T_ic=T_ic, as_numpy=False)
    return Measurement(rows_dev=rows, z_dev=res, sigma2=cfg.photo_sigma ** 2)


def lidar_measurement(state: NavState, points_l, vmap, T_il, cfg: FilterConfig,
                      plane_cache: dict = None) -> Measurement:
    """Point-to-plane residuals against the map's local planes
    (estimator.py:190-238).  Every scan point is transformed, keyed, fitted
    (its leaf and 6 face neighbours, csrc/voxmap.cu) and gated on the device;
    rows keep the scan order.  plane_cache is accepted for the reference's
    signature; the device refits per call (the map does not change between
    the iterations of one update, so the fits are identical)."""
    _lib.require()
    dev = vmap.device
    pts = torch.as_tensor(np.atleast_2d(np.asarray(points_l, dtype=np.float64))) if not torch.is_tensor(points_l) \
        else points_l
    pts = pts.to(device=dev, dtype=torch.float64).reshape(-1, 3).contiguous()
    n = pts.shape[0]
    rows = torch.empty((max(n, 1), 6), dtype=torch.float64, device=dev)
    z = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    keep = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    c = lambda a, k: (ctypes.c_double * k)(*np.asarray(a, dtype=np.float64).ravel().tolist())
    m = vmap.struct()
    _lib.check(_lib.load().lsb_lidar_rows(ctypes.byref(m), ctypes.c_void_p(pts.data_ptr()), n, c(T_il.R, 9),
                                          c(T_il.t, 3), c(state.T_WI.R, 9), c(state.T_WI.t, 3),
                                          float(cfg.lidar_gate), ctypes.c_void_p(rows.data_ptr()),
                                          ctypes.c_void_p(z.data_ptr()), ctypes.c_void_p(keep.data_ptr()),
                                          _lib.stream_ptr()), "lidar_rows")
    # the rows of dropped points are zero (k_lidar_rows), so the H/b
    # reduction runs over all n rows without a compaction; z / H are
    # compacted to the kept rows (scan order) only if a caller reads them
    k = keep[:n]
    m_ok = int(k.sum(dtype=torch.int64).item())
    if m_ok == 0:
        raise NoAssociations("no scan point matched a plane (or all residuals gated out)")
    return Measurement(rows_dev=rows[:n], z_dev=z[:n], sigma2=cfg.lidar_sigma ** 2, keep_dev=k, count=m_ok)


class _VisualPass:
    """The device side of one visual IESKF iteration in ONE library call
    (lsb_visual_pass) and ONE host sync: render (contributing lists) ->
    semi-dense mask -> selection / residual / gate -> pose chain -> pose
    rows -> H/b, the kept count staying on the device; the counts, the
    intersection overflow flag and the 42 H/b numbers come back in one
    read.  Buffers persist across the iterations of an update.  Same kernels
    and the same bits as visual_measurement(...).hb() (tested)."""

    def __init__(self, window, observed, cam, cfg: FilterConfig, settings: RasterSettings):
        self.arrays = _as_arrays(window)
        self.cam, self.cfg, self.settings = cam, cfg, settings
        dev = self.arrays.device
        self.h, self.w = h, w = int(cam.height), int(cam.width)
        self.bin_mode = 1 if settings.alpha_cut > 0 else 0
        self.key = (len(self.arrays), w, h, float(settings.alpha_cut), self.bin_mode)
        self.cap = max(_CAP_HINT.get(self.key, 0), 1 << 16, 8 * len(self.arrays))
        self.set_observed(observed)
        self.image = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
        self.t_final = torch.empty((h, w), dtype=torch.float32, device=dev)
        self.n_contrib = torch.empty((h, w), dtype=torch.int32, device=dev)
        lib = _lib.load()
        npx, B = h * w, int(cfg.pixel_budget)
        self.mask = torch.empty(npx, dtype=torch.uint8, device=dev)
        self.scratch = torch.empty(int(lib.lsb_visual_select_scratch_bytes(npx, B)), dtype=torch.uint8, device=dev)
        self.ids = torch.empty(B, dtype=torch.int32, device=dev)
        self.res = torch.empty(B, dtype=torch.float64, device=dev)
        self.rows = torch.zeros((B, 6), dtype=torch.float64, device=dev)
        self.chain = torch.empty((max(len(self.arrays), 1), 48), dtype=torch.float32, device=dev)
        self.hb_scratch = torch.empty(lib.lsb_hb_scratch_doubles(), dtype=torch.float64, device=dev)
        # one device buffer read back per iteration: [L, selected, kept] + the
        # render counters [M, I, overflow] as int64, then the 42 H/b doubles
        self.dev_out = torch.empty(6 + 42, dtype=torch.float64, device=dev)
        self.host_out = torch.empty(6 + 42, dtype=torch.float64).pin_memory()
        self.state = None

    def set_observed(self, observed) -> None:
        self.obs = _observed(observed, (self.h, self.w, 3), self.arrays.device)
        self.u8 = int(self.obs.dtype == torch.uint8)

    def run(self, nav: NavState, T_ic):
        from .geometry import imu_camera_adjoint
        lib = _lib.load()
        T_cw = (nav.T_WI @ T_ic).inverse()
        cfg = self.cfg
        c = _lib.VisualCfg()
        c.budget, c.observed_u8 = int(cfg.pixel_budget), self.u8
        c.grad_thr, c.t_max = float(cfg.grad_threshold), float(cfg.coverage_max_transmittance)
        c.gate, c.inv_sigma2 = float(cfg.photo_gate), 1.0 / float(cfg.photo_sigma) ** 2
        c.A[:] = imu_camera_adjoint(T_cw.R, T_ic).ravel().tolist()
        while True:
            if self.state is None or self.state.dims.isect_cap != self.cap:
                self.state = RenderState(self.arrays, self.cam, T_cw.R, T_cw.t, self.settings, self.cap,
                                         self.bin_mode)
                self.bufs = _lib.VisualBufs(*(t.data_ptr() for t in (
                    self.mask, self.scratch, self.ids, self.res, self.chain, self.rows, self.hb_scratch,
                    self.dev_out)))
            else:
                self.state.set_pose(T_cw.R, T_cw.t)
            st = self.state
            c.sh_degree_used = _degree_used(st)
            p = st.arrays.params()
            _lib.check(lib.lsb_visual_pass(
                ctypes.byref(p), ctypes.byref(st.c_cam), ctypes.byref(st.c_pose), ctypes.byref(st.c_set), st._ws(),
                st.ws_bytes, ctypes.byref(st.dims), ctypes.c_void_p(self.image.data_ptr()),
                ctypes.c_void_p(self.t_final.data_ptr()), ctypes.c_void_p(self.n_contrib.data_ptr()),
                ctypes.c_void_p(self.obs.data_ptr()), ctypes.byref(c), ctypes.byref(self.bufs), _lib.stream_ptr()),
                "visual_pass")
            self.host_out.copy_(self.dev_out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            _, n_sel, n_ok, _, I, overflow = self.host_out[:6].view(torch.int64).tolist()
            if not overflow:
                break
            self.cap = int(I * 1.25) + 1024                  # grow and redo (rare)
        _CAP_HINT[self.key] = int(I * 1.25) + 1024
        if n_sel < cfg.min_pixels:
            raise TooFewPixels(f"{n_sel} < {cfg.min_pixels}")
        if n_ok < cfg.min_pixels:
            raise TooFewPixels(f"{n_ok} < {cfg.min_pixels} after gating")
        o = self.host_out[6:].numpy()
        return o[:36].reshape(6, 6).copy(), o[36:].copy()


def _pack(x: NavState) -> np.ndarray:
    return np.concatenate([np.asarray(x.T_WI.R, float).reshape(9), np.asarray(x.T_WI.t, float).reshape(3),
                           np.asarray(x.velocity, float).reshape(3), np.asarray(x.bias_gyro, float).reshape(3),
                           np.asarray(x.bias_accel, float).reshape(3)])


def _unpack(v: np.ndarray) -> NavState:
    return NavState(SE3(v[:9].reshape(3, 3).copy(), v[9:12].copy()), v[12:15].copy(), v[15:18].copy(),
                    v[18:21].copy())


_VIS_CACHE: dict = {}


def _visual_pass(window, observed, cam, cfg: FilterConfig, settings: RasterSettings) -> _VisualPass:
    """The update's _VisualPass, reused across updates on the same window /
    camera / configuration (its device buffers and pinned read-back buffer
    are allocated once); the observed frame is refreshed every update."""
    arrays = _as_arrays(window)
    # keyed on the parameter storage, not the wrapper object: a window's
    # as_gaussian_arrays() returns a new wrapper of the same tensors per call
    key = (arrays.means.data_ptr(), arrays.shs.data_ptr(), len(arrays), int(arrays.shs.shape[1]), int(cam.width),
           int(cam.height), float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy), repr(cfg), repr(settings))
    vis = _VIS_CACHE.get(key)
    if vis is None:
        if len(_VIS_CACHE) > 4:
            _VIS_CACHE.clear()
        vis = _VIS_CACHE[key] = _VisualPass(arrays, observed, cam, cfg, settings)
    else:
        vis.arrays = arrays
        vis.set_observed(observed)
    return vis


def _meas_len(meas) -> int:
    try:
        return len(meas)
    except TypeError:                     # a reference Measurement (numpy z)
        return int(np.asarray(meas.z).size)


def _pose_hb(meas):
    """(A6, b6) = the pose block of H^T R^-1 H and H^T R^-1 z of a
    measurement: reduced on the device when the measurement is this
    package's (Measurement.hb), else from its numpy H / z / R_diag."""
    if hasattr(meas, "hb"):
        return meas.hb()
    H = np.asarray(meas.H, dtype=float)
    if H.shape[1] > 6 and np.any(H[:, 6:] != 0.0):
        raise ValueError("ieskf_update: measurement rows beyond the pose block are not supported")
    HtRi = H[:, :6].T / np.asarray(meas.R_diag, dtype=float)[None, :]
    return HtRi @ H[:, :6], HtRi @ np.asarray(meas.z, dtype=float)


def ieskf_update(state: NavState, cov: np.ndarray, meas_fn, max_iter: int = 5, step_tol: float = 1e-6,
                 bias_limit: float = 0.5):
    """Iterated EKF update re-linearising meas_fn(state) -> Measurement about
    the running estimate (estimator.py:292-331), the reference's generic
    signature.  meas_fn may raise NoAssociations / TooFewPixels (callers
    skip the update) and SingularGain comes from a singular gain; an empty
    measurement keeps the prior.  The pose block of H^T R^-1 H / H^T R^-1 z
    comes from the measurement (reduced on the device for this package's
    measurements) and the 15x15 gain algebra runs in one host call per
    iteration (lsb_ieskf_iterate; K z = S^-1 b, K H = S^-1 A)."""
    lib = _lib.load()
    cov_c = np.ascontiguousarray(cov, dtype=np.float64)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    x_bar = _pack(state)
    x_hat = x_bar.copy()
    K_H = P = None
    xi, KH_buf, P_buf = np.empty(DIM), np.empty((DIM, DIM)), np.empty((DIM, DIM))
    for _ in range(max_iter):
        meas = meas_fn(_unpack(x_hat))
        if meas is None or _meas_len(meas) == 0:
            if K_H is None:
                return state.clone(), cov.copy()
            break
        A6, b6 = _pose_hb(meas)
        if lib.lsb_ieskf_iterate(ptr(cov_c), ptr(x_bar), ptr(x_hat), ptr(np.ascontiguousarray(A6, dtype=np.float64)),
                                 ptr(np.ascontiguousarray(b6, dtype=np.float64)), float(bias_limit), ptr(xi),
                                 ptr(KH_buf), ptr(P_buf)):
            raise SingularGain(lib.lsb_last_error().decode())
        K_H, P = KH_buf.copy(), P_buf.copy()
        if float(np.sqrt(xi @ xi)) < step_tol:
            break
    if K_H is None:
        return state.clone(), cov.copy()
    cov_post = (np.eye(DIM) - K_H) @ P
    return _unpack(x_hat), 0.5 * (cov_post + cov_post.T)


def ieskf_visual_update(state: NavState, cov: np.ndarray, observed, window, cam, T_ic, cfg: FilterConfig,
                        settings: RasterSettings, max_iter: int = 5, step_tol: float = 1e-6,
                        bias_limit: float = 0.5):
    """Iterated EKF update with the photometric measurement (estimator.py:
    292-331).  Each iteration re-renders the window at the running estimate
    and reduces the pose block of H^T R^-1 H and H^T R^-1 z on the GPU
    (Measurement.hb); only the 15x15 filter algebra runs on the host, using
    K z = S^-1 b and K H = S^-1 A (H is zero outside its 6 pose columns)."""
    K_H = P = None
    vis = _visual_pass(window, observed, cam, cfg, settings)
    lib = _lib.load()
    cov_c = np.ascontiguousarray(cov, dtype=np.float64)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    # the states as [R | t | v | b_g | b_a] vectors; one host C++ call per
    # iteration does boxminus, the 15x15 gain algebra and boxplus
    # (lsb_ieskf_iterate: estimator.py:292-331)
    x_bar = _pack(state)
    x_hat = x_bar.copy()
    xi, KH_buf, P_buf = np.empty(DIM), np.empty((DIM, DIM)), np.empty((DIM, DIM))
    for _ in range(max_iter):
        A6, b6 = vis.run(_unpack(x_hat), T_ic)
        if lib.lsb_ieskf_iterate(ptr(cov_c), ptr(x_bar), ptr(x_hat), ptr(np.ascontiguousarray(A6)),
                                 ptr(np.ascontiguousarray(b6)), float(bias_limit), ptr(xi), ptr(KH_buf),
                                 ptr(P_buf)):
            raise SingularGain(lib.lsb_last_error().decode())
        K_H, P = KH_buf, P_buf
        if float(np.sqrt(xi @ xi)) < step_tol:
            break
    x_hat = _unpack(x_hat)
    if K_H is None:
        return state.clone(), cov.copy()
    cov_post = (np.eye(DIM) - K_H) @ P
    return x_hat, 0.5 * (cov_post + cov_post.T)
