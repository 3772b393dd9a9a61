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
from .errors import TooFewPixels
from .geometry import SE3
from .raster import RasterSettings, _f32, pose_rows, render

DIM = 15


@dataclass
class FilterConfig:
    """The visual fields of estimator.FilterConfig (estimator.py:95-115)."""

    photo_sigma: float = 0.1
    pixel_budget: int = 1024
    grad_threshold: float = 0.05
    photo_gate: float = 0.15
    min_pixels: int = 50
    coverage_max_transmittance: float = 0.9


@dataclass
class NavState:
    T_WI: SE3 = field(default_factory=SE3.identity)


@dataclass
class Measurement:
    """Stacked residuals with pose Jacobian rows padded to the full state
    (estimator.py:84-92); numpy on the host, as the filter consumes it."""

    z: np.ndarray
    H: np.ndarray
    R_diag: np.ndarray
    rows_dev: torch.Tensor = field(default=None, repr=False)
    z_dev: torch.Tensor = field(default=None, repr=False)

    def hb(self) -> tuple[np.ndarray, np.ndarray]:
        """(6x6 sum h h^T / sigma^2, 6 sum h z / sigma^2) for the pose block,
        reduced on the device (estimator.py:314-318 with H = -rows)."""
        m = int(self.z_dev.numel())
        out = torch.empty(42, dtype=torch.float64, device=self.z_dev.device)
        _lib.check(_lib.load().lsb_hb_reduce(ctypes.c_void_p(self.rows_dev.data_ptr()),
                                             ctypes.c_void_p(self.z_dev.data_ptr()), m,
                                             float(1.0 / self.R_diag[0]) if m else 1.0,
                                             ctypes.c_void_p(out.data_ptr()), _lib.stream_ptr()), "hb_reduce")
        o = out.cpu().numpy()
        return o[:36].reshape(6, 6), o[36:]


def select_semi_dense_pixels(observed, coverage_t, cfg: FilterConfig) -> np.ndarray:
    """High-gradient, covered pixels, uniformly subsampled to the budget
    (estimator.py:241-257).  Returns flat ids (numpy int64)."""
    _lib.require()
    dev = coverage_t.device if torch.is_tensor(coverage_t) and coverage_t.is_cuda else torch.device("cuda")
    h, w = int(np.shape(coverage_t)[0]), int(np.shape(coverage_t)[1])
    obs = _f32(observed, (h, w, 3), dev)
    tf = _f32(coverage_t, (h, w), dev)
    mask = torch.empty((h, w), dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().lsb_semidense_mask(ctypes.c_void_p(obs.data_ptr()), ctypes.c_void_p(tf.data_ptr()), w, h,
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
    out = render(window, T_wc, cam, settings)
    dev = out.image.device
    h, w = int(cam.height), int(cam.width)
    obs = _f32(observed, (h, w, 3), dev)
    ids = select_semi_dense_pixels(obs, out.final_transmittance, cfg)
    if len(ids) < cfg.min_pixels:
        raise TooFewPixels(f"{len(ids)} < {cfg.min_pixels}")
    idt = torch.as_tensor(ids, device=dev)
    gray_obs = obs.view(-1, 3).to(torch.float64)[idt].sum(dim=1) / 3.0
    gray_hat = out.image.view(-1, 3).to(torch.float64)[idt].sum(dim=1) / 3.0
    res = gray_obs - gray_hat
    ok = res.abs() <= cfg.photo_gate
    n_ok = int(ok.sum().item())
    if n_ok < cfg.min_pixels:
        raise TooFewPixels(f"{n_ok} < {cfg.min_pixels} after gating")
    idt = idt[ok]
    res = res[ok].contiguous()
    rows = pose_rows(out, idt, T_ic=T_ic, as_numpy=False)
    rows_h = rows.cpu().numpy()
    H = np.zeros((n_ok, DIM))
    H[:, :6] = -rows_h
    return Measurement(z=res.cpu().numpy(), H=H, R_diag=np.full(n_ok, cfg.photo_sigma ** 2), rows_dev=rows,
                       z_dev=res)
