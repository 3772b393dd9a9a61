"""render / backward — drop-in for livsplat.raster on the B200.

Same entry points, argument meaning and error behaviour as the reference
(raster.py:212 render, :309 backward); the numba/numpy body is replaced by
libsplat_b200.so (include/lsb.h) working on HBM-resident torch tensors:

    K1 preprocess  (projection, EWA covariance, footprint, SH colour)   f64
    K2 binning     (tile histogram, scan, scatter, per-tile depth sort) int
    K3 blend fwd   (one CTA per 16x16 tile, smem-staged records)        f32
    K4 blend bwd   (forward-order recompute, warp reductions)           f32
    K5 chain       (per-splat chain rule, pose reduction)               f64

Outputs are device tensors (image (H,W,3) f32, final_transmittance (H,W),
contrib_count (H,W) int32) that numpy reads through np.asarray (a host copy,
HostReadable); `RenderOutput.numpy()` gives all of them as f64 / int64.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import MissingCache
from .geometry import SE3, as_se3, imu_camera_adjoint

TILE = 16


@dataclass
class RasterSettings:
    """raster.py:24-34 (identical fields and defaults)."""

    near: float = 0.01
    dilation: float = 0.3
    alpha_clamp: float = 0.99
    transmittance_min: float = 1e-4
    footprint_sigma: float = 6.0
    alpha_cut: float = 0.0
    max_footprint_px: float = 512.0
    background: tuple = (0.0, 0.0, 0.0)
    sh_degree: int = 0


def _dev(device=None):
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _as(x, shape, device, dtype=torch.float32):
    t = torch.as_tensor(x)
    if t.dtype != dtype or t.device != device:
        t = t.to(device=device, dtype=dtype)
    return t.reshape(shape).contiguous()


def _f32(x, shape, device):
    return _as(x, shape, device, torch.float32)


OBS_U8 = 0x100      # include/lsb.h LSB_OBS_U8


def _observed(x, shape, device):
    """An observed frame on the device: 8-bit frames (the camera's / the
    dataset's PPM bytes, raster.py:520-541) stay 8-bit — the kernels use
    u / 255.0 like read_ppm — anything else becomes float32."""
    t = torch.as_tensor(x)
    if t.dtype == torch.uint8:
        return _as(t, shape, device, torch.uint8)
    if t.dtype == torch.float64:
        # a frame read by read_ppm is u / 255.0 in f64: keep it as those
        # bytes (decoded exactly in the kernels) instead of rounding to f32,
        # which moves the Sobel magnitudes of quantised edges across the
        # gradient threshold (estimator.py:248-252)
        u = torch.round(t * 255.0)
        if bool(((u >= 0) & (u <= 255) & (u / 255.0 == t)).all()):
            return _as(u.to(torch.uint8), shape, device, torch.uint8)
    return _f32(t, shape, device)


def _obs_kind(observed, kind: int) -> int:
    if observed.dtype == torch.uint8:
        return int(kind) | OBS_U8
    if observed.dtype != torch.float32:
        raise ValueError("observed frames are float32 or uint8 (H, W, 3)")
    return int(kind)


class GaussianArrays:
    """Structure-of-arrays Gaussian parameters in HBM.  f32 by default (the
    window arena's storage type, window.py:51-55; the reference upcasts the
    same f32 values to f64 for its math, raster.py:47-52); f64 for the
    working copy that optimize_window steps (optimize.py:142-149)."""

    def __init__(self, means, rots, scales, opacities, shs, device=None, dtype=torch.float32):
        dev = _dev(device)
        if dtype not in (torch.float32, torch.float64):
            raise ValueError("GaussianArrays dtype must be float32 or float64")
        n = int(np.shape(means)[0]) if not torch.is_tensor(means) else int(means.shape[0])
        self.means = _as(means, (n, 3), dev, dtype)
        self.rots = _as(rots, (n, 3, 3), dev, dtype)
        self.scales = _as(scales, (n, 3), dev, dtype)
        self.opacities = _as(opacities, (n,), dev, dtype)
        k = (int(np.prod(np.shape(shs))) // (3 * n)) if n else 1
        self.shs = _as(shs, (n, max(k, 1), 3), dev, dtype)

    @property
    def dtype(self):
        return self.means.dtype

    def clone(self, dtype=None) -> "GaussianArrays":
        """A copy (new storage), optionally cast."""
        dt = dtype or self.dtype
        return GaussianArrays(*(t.to(dt).clone() for t in (self.means, self.rots, self.scales, self.opacities,
                                                           self.shs)), device=self.device, dtype=dt)

    def copy_from(self, other: "GaussianArrays") -> None:
        """In-place copy (with cast) of another arena's values."""
        for k in ("means", "rots", "scales", "opacities", "shs"):
            getattr(self, k).copy_(getattr(other, k))

    def __len__(self):
        return self.means.shape[0]

    @property
    def device(self):
        return self.means.device

    @staticmethod
    def from_gaussians(gaussians, device=None, dtype=torch.float32) -> "GaussianArrays":
        if not gaussians:
            return GaussianArrays(np.zeros((0, 3)), np.zeros((0, 3, 3)), np.zeros((0, 3)), np.zeros(0),
                                  np.zeros((0, 1, 3)), device, dtype)
        k = max(g.sh.shape[0] for g in gaussians)
        shs = np.zeros((len(gaussians), k, 3))
        for i, g in enumerate(gaussians):
            shs[i, : g.sh.shape[0]] = g.sh
        return GaussianArrays(np.stack([g.mean_w for g in gaussians]), np.stack([g.rot for g in gaussians]),
                              np.stack([g.scale for g in gaussians]),
                              np.array([g.opacity for g in gaussians], dtype=float), shs, device, dtype)

    def params(self) -> _lib.Params:
        return _lib.Params(self.means.data_ptr(), self.rots.data_ptr(), self.scales.data_ptr(),
                           self.opacities.data_ptr(), self.shs.data_ptr(), len(self),
                           int(self.shs.shape[1]), 1 if self.dtype == torch.float64 else 0)


@dataclass
class ParamGradients:
    """Per-Gaussian gradients aligned with the input arrays (raster.py:85-98);
    device tensors that are views of one flat f32 buffer (`flat`), so a
    multi-GPU step all-reduces a single contiguous allocation."""

    mean: torch.Tensor
    rot: torch.Tensor
    scale: torch.Tensor
    opacity: torch.Tensor
    sh: torch.Tensor
    flat: Optional[torch.Tensor] = field(default=None, repr=False)

    @staticmethod
    def zeros(n: int, k: int, device) -> "ParamGradients":
        return ParamGradients.from_flat(torch.zeros(n * (10 + 3 * k), dtype=torch.float32, device=device), n, k)

    @staticmethod
    def from_flat(flat: torch.Tensor, n: int, k: int) -> "ParamGradients":
        """Group views of an existing flat buffer (n * (10 + 3k) f32)."""
        o = 0
        views = []
        for size, shape in ((3 * n, (n, 3)), (3 * n, (n, 3)), (3 * n, (n, 3)), (n, (n,)), (3 * k * n, (n, k, 3))):
            views.append(flat[o:o + size].view(shape))
            o += size
        return ParamGradients(*views, flat=flat)

    def struct(self) -> _lib.Grads:
        return _lib.Grads(self.mean.data_ptr(), self.rot.data_ptr(), self.scale.data_ptr(),
                          self.opacity.data_ptr(), self.sh.data_ptr())

    def numpy(self) -> dict:
        return {k: getattr(self, k).detach().cpu().numpy().astype(np.float64)
                for k in ("mean", "rot", "scale", "opacity", "sh")}


class PoseGradient:
    """Loss gradient w.r.t. the rendering pose (raster.py:101-115).  The
    device computes the camera-tangent pieces; the 6x6 extrinsic chain runs
    on the host when first read (one 72-byte copy)."""

    def __init__(self, dev_vals: torch.Tensor, R_cw: np.ndarray, T_ic):
        self._dev = dev_vals
        self._R_cw = R_cw
        self._T_ic = T_ic
        self._host = None

    def _resolve(self):
        if self._host is None:
            v = self._dev.cpu().numpy()
            rho_cam = v[0:3].copy()
            tau_cam = v[3:6] - self._R_cw @ v[6:9]      # raster.py:380
            A = imu_camera_adjoint(self._R_cw, self._T_ic)
            imu = A.T @ np.concatenate([rho_cam, tau_cam])
            self._host = (imu[:3], imu[3:], rho_cam, tau_cam)
        return self._host

    rho = property(lambda self: self._resolve()[0])
    tau = property(lambda self: self._resolve()[1])
    camera_rho = property(lambda self: self._resolve()[2])
    camera_tau = property(lambda self: self._resolve()[3])

    def as_vector(self) -> np.ndarray:
        return np.concatenate([self.rho, self.tau])


class HostReadable(torch.Tensor):
    """A device tensor that numpy can read: np.asarray(x) (what the
    reference's consumers of a render call -- write_ppm, metrics.psnr,
    raster.py:511-517, metrics.py:12-22) copies it to the host.  Torch
    operations on it return plain tensors (no subclass dispatch)."""

    __torch_function__ = torch._C._disabled_torch_function_impl

    def __array__(self, dtype=None, copy=None):
        a = self.detach().cpu().as_subclass(torch.Tensor).numpy()
        return a if dtype is None else a.astype(dtype, copy=False)


def host_readable(t: Optional[torch.Tensor]) -> Optional[torch.Tensor]:
    return None if t is None else t.as_subclass(HostReadable)


@dataclass
class RenderOutput:
    image: torch.Tensor                 # (H, W, 3) f32, device
    final_transmittance: torch.Tensor   # (H, W) f32
    contrib_count: torch.Tensor         # (H, W) int32, splats processed per pixel
    cache: Optional["RenderState"] = field(default=None, repr=False)
    depth: Optional[torch.Tensor] = None

    def numpy(self) -> dict:
        out = {"image": self.image.cpu().numpy().astype(np.float64),
               "final_transmittance": self.final_transmittance.cpu().numpy().astype(np.float64),
               "contrib_count": self.contrib_count.cpu().numpy().astype(np.int64)}
        if self.depth is not None:
            out["depth"] = self.depth.cpu().numpy().astype(np.float64)
        return out


# capacity hints per (n, W, H): the intersection count seen last time
_CAP_HINT: dict = {}


class RenderState:
    """The render 'cache': the device workspace (records, tile lists,
    partials) plus the structs the backward needs.  Opaque to callers, like
    the reference's cache dict (raster.py:246-258)."""

    def __init__(self, arrays: GaussianArrays, cam, R_cw, t_cw, settings: RasterSettings,
                 isect_cap: int, bin_mode: int = 0):
        self.arrays = arrays
        self.cam = cam
        self.settings = settings
        self.bin_mode = bin_mode
        self.R_cw = np.asarray(R_cw, dtype=np.float64)
        self.t_cw = np.asarray(t_cw, dtype=np.float64)
        self.c_cam = _lib.make_camera(cam)
        self.c_set = _lib.make_settings(settings, bin_mode)
        self.c_pose = _lib.make_pose(self.R_cw, self.t_cw)
        self.dims = _lib.Dims(len(arrays), int(cam.width), int(cam.height), int(arrays.shs.shape[1]), TILE,
                              int(isect_cap))
        nb = ctypes.c_size_t()
        _lib.check(_lib.load().lsb_workspace_bytes(ctypes.byref(self.dims), ctypes.byref(nb)), "workspace")
        self.ws = torch.empty(nb.value, dtype=torch.uint8, device=arrays.device)
        self.sticky(clear=True)
        self.counts = None
        self._max_px = int(cam.width) * int(cam.height)

    @property
    def ws_bytes(self) -> int:
        return self.ws.numel()

    def set_pose(self, R_cw, t_cw) -> None:
        self.R_cw = np.asarray(R_cw, dtype=np.float64)
        self.t_cw = np.asarray(t_cw, dtype=np.float64)
        self.c_pose = _lib.make_pose(self.R_cw, self.t_cw)

    def set_camera(self, cam) -> None:
        """Render through another camera of at most the workspace's size (a
        row band of the full frame: crop_rows)."""
        if int(cam.width) * int(cam.height) > self._max_px:
            raise ValueError("camera larger than the workspace was sized for")
        self.cam = cam
        self.c_cam = _lib.make_camera(cam)
        self.dims.width, self.dims.height = int(cam.width), int(cam.height)

    def _ws(self):
        return ctypes.c_void_p(self.ws.data_ptr())

    def read_counts(self, stream=None):
        c = (ctypes.c_int64 * 4)()
        _lib.check(_lib.load().lsb_render_counts(ctypes.c_void_p(self.ws.data_ptr()), ctypes.byref(self.dims),
                                                 c, _lib.stream_ptr(stream)), "counts")
        self.counts = tuple(int(v) for v in c)
        return self.counts

    def sticky(self, clear: bool = False, read: bool = False, stream=None) -> Optional[bool]:
        """The workspace's sticky overflow flag: set by any render since the
        last clear (read: syncs `stream`; clear: stream-ordered reset)."""
        out = ctypes.c_int64(0) if read else None
        _lib.check(_lib.load().lsb_render_sticky(ctypes.c_void_p(self.ws.data_ptr()), ctypes.byref(self.dims),
                                                 ctypes.byref(out) if read else None, 1 if clear else 0,
                                                 _lib.stream_ptr(stream)), "sticky")
        return bool(out.value) if read else None

    def band_stats(self, stream=None):
        """(tiles re-blended, band pairs decided in f64, of them composited,
        max relative f32 alpha error over those pairs) of the last forward:
        the alpha_cut decisions the f32 alpha cannot take the reference's way
        by itself (_kernels.py:104), see csrc/blend.cu."""
        c = (ctypes.c_int64 * 4)()
        _lib.check(_lib.load().lsb_render_band_stats(ctypes.c_void_p(self.ws.data_ptr()), ctypes.byref(self.dims),
                                                     c, _lib.stream_ptr(stream)), "band_stats")
        err = float(np.frombuffer(np.uint32(c[3]).tobytes(), np.float32)[0])
        return int(c[0]), int(c[1]), int(c[2]), err

    def export(self, what: int, stream=None) -> np.ndarray:
        """Parity hooks: 0 ids, 1 bboxes, 2 tile ranges, 3 tile entry ids, 4 depth."""
        M, I = self.counts[0], self.counts[1]
        ntiles = ((self.dims.width + TILE - 1) // TILE) * ((self.dims.height + TILE - 1) // TILE)
        shape, dt = {0: ((M,), torch.int32), 1: ((M, 4), torch.int32), 2: ((ntiles, 2), torch.int32),
                     3: ((I,), torch.int32), 4: ((M,), torch.float64)}[what]
        dst = torch.empty(shape, dtype=dt, device=self.ws.device)
        if dst.numel():
            _lib.check(_lib.load().lsb_render_export(ctypes.c_void_p(self.ws.data_ptr()), ctypes.byref(self.dims),
                                                     what, ctypes.c_void_p(dst.data_ptr()),
                                                     _lib.stream_ptr(stream)), "export")
        return dst.cpu().numpy()


def crop_rows(cam, y0: int, y1: int):
    """The camera of rows [y0, y1) of `cam`'s frame (y0 a multiple of the
    16-pixel tile, so the band's tiles are the frame's tiles): same
    intrinsics with the principal point shifted up by y0."""
    from types import SimpleNamespace
    if y0 % TILE or not (0 <= y0 < y1 <= int(cam.height)):
        raise ValueError("band rows must start on a tile row and lie inside the frame")
    return SimpleNamespace(fx=float(cam.fx), fy=float(cam.fy), cx=float(cam.cx), cy=float(cam.cy) - y0,
                           width=int(cam.width), height=int(y1 - y0))


def _as_arrays(source) -> GaussianArrays:
    if isinstance(source, GaussianArrays):
        return source
    if hasattr(source, "as_gaussian_arrays"):
        a = source.as_gaussian_arrays()
        return a if isinstance(a, GaussianArrays) else GaussianArrays(a.means, a.rots, a.scales, a.opacities,
                                                                       a.shs)
    if all(hasattr(source, k) for k in ("means", "rots", "scales", "opacities", "shs")):
        return GaussianArrays(source.means, source.rots, source.scales, source.opacities, source.shs)
    raise TypeError(f"cannot render from {type(source)!r}")


def render_fwd(state: RenderState, image, t_final, n_contrib, depth=None, stream=None) -> None:
    """Launch K1-K3 into `state` (async, no host sync)."""
    p = state.arrays.params()
    _lib.check(_lib.load().lsb_render_fwd(
        ctypes.byref(p), ctypes.byref(state.c_cam), ctypes.byref(state.c_pose), ctypes.byref(state.c_set),
        ctypes.c_void_p(state.ws.data_ptr()), state.ws_bytes, ctypes.byref(state.dims),
        ctypes.c_void_p(image.data_ptr()), ctypes.c_void_p(t_final.data_ptr()),
        ctypes.c_void_p(n_contrib.data_ptr()), ctypes.c_void_p(depth.data_ptr()) if depth is not None else None,
        _lib.stream_ptr(stream)), "render")


def render_bin(state: RenderState, stream=None) -> None:
    """K1 preprocess + K2 binning/sort (async)."""
    p = state.arrays.params()
    _lib.check(_lib.load().lsb_render_bin(ctypes.byref(p), ctypes.byref(state.c_cam), ctypes.byref(state.c_pose),
                                          ctypes.byref(state.c_set), state._ws(), state.ws_bytes,
                                          ctypes.byref(state.dims), _lib.stream_ptr(stream)), "bin")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def render_blend(state: RenderState, image, t_final, n_contrib, depth=None, stream=None) -> None:
    """K3 blend forward (async).  n_contrib None: no entry count (include/lsb.h)."""
    _lib.check(_lib.load().lsb_render_blend(
        ctypes.byref(state.c_set), state._ws(), state.ws_bytes, ctypes.byref(state.dims),
        ctypes.c_void_p(image.data_ptr()), ctypes.c_void_p(t_final.data_ptr()),
        _ptr(n_contrib), _ptr(depth), _lib.stream_ptr(stream)), "blend")


def render_blend_loss(state: RenderState, image, t_final, n_contrib, observed, kind: int, grad_scale: float,
                      grad_out, loss_ptr, depth=None, stream=None) -> None:
    """K3 blend forward fused with the photometric loss (async)."""
    _lib.check(_lib.load().lsb_render_blend_loss(
        ctypes.byref(state.c_set), state._ws(), state.ws_bytes, ctypes.byref(state.dims),
        ctypes.c_void_p(image.data_ptr()), ctypes.c_void_p(t_final.data_ptr()),
        _ptr(n_contrib), _ptr(depth), ctypes.c_void_p(observed.data_ptr()), _obs_kind(observed, kind), float(grad_scale), ctypes.c_void_p(grad_out.data_ptr()),
        loss_ptr, _lib.stream_ptr(stream)), "blend_loss")


def render_blend_bwd(state: RenderState, image, n_contrib, grad_image, grad_scale: float = 1.0,
                     stream=None) -> None:
    """K4 blend backward into the per-intersection partials (async)."""
    _lib.check(_lib.load().lsb_render_blend_bwd(
        ctypes.byref(state.c_set), state._ws(), state.ws_bytes, ctypes.byref(state.dims),
        ctypes.c_void_p(image.data_ptr()), _ptr(n_contrib),
        ctypes.c_void_p(grad_image.data_ptr()), float(grad_scale), _lib.stream_ptr(stream)), "blend_bwd")


def render_blend_fused_loss(state: RenderState, observed, kind: int, grad_scale: float, loss_ptr,
                            stream=None) -> None:
    """K3 + loss + K4 in one kernel (the window engine's step; async)."""
    _lib.check(_lib.load().lsb_render_blend_fused_loss(
        ctypes.byref(state.c_set), state._ws(), state.ws_bytes, ctypes.byref(state.dims),
        ctypes.c_void_p(observed.data_ptr()), _obs_kind(observed, kind), float(grad_scale), loss_ptr,
        _lib.stream_ptr(stream)), "blend_fused_loss")


def render_blend_bwd_loss(state: RenderState, image, observed, kind: int, grad_scale: float, loss_ptr,
                          stream=None) -> None:
    """K4 blend backward with the photometric loss fused in: dL/dI formed per
    pixel from (image, observed), loss sums to loss_ptr (async)."""
    _lib.check(_lib.load().lsb_render_blend_bwd_loss(
        ctypes.byref(state.c_set), state._ws(), state.ws_bytes, ctypes.byref(state.dims),
        ctypes.c_void_p(image.data_ptr()), ctypes.c_void_p(observed.data_ptr()), _obs_kind(observed, kind),
        float(grad_scale), loss_ptr, _lib.stream_ptr(stream)), "blend_bwd_loss")


def render_chain(state: RenderState, grads: "ParamGradients", pose_dev=None, stream=None) -> None:
    """K5 chain rule; ACCUMULATES into grads (async)."""
    p = state.arrays.params()
    g = grads.struct()
    _lib.check(_lib.load().lsb_render_chain(
        ctypes.byref(p), ctypes.byref(state.c_cam), ctypes.byref(state.c_pose), ctypes.byref(state.c_set),
        state._ws(), state.ws_bytes, ctypes.byref(state.dims), ctypes.byref(g),
        ctypes.c_void_p(pose_dev.data_ptr()) if pose_dev is not None else None, _lib.stream_ptr(stream)),
        "chain")


def render_bwd(state: RenderState, out: "RenderOutput", grad_image: torch.Tensor, grad_scale: float,
               grads: ParamGradients, pose_dev: Optional[torch.Tensor], stream=None) -> None:
    """Launch K4-K5 (async): ACCUMULATES into `grads`."""
    p = state.arrays.params()
    g = grads.struct()
    _lib.check(_lib.load().lsb_render_bwd(
        ctypes.byref(p), ctypes.byref(state.c_cam), ctypes.byref(state.c_pose), ctypes.byref(state.c_set),
        ctypes.c_void_p(state.ws.data_ptr()), state.ws_bytes, ctypes.byref(state.dims),
        ctypes.c_void_p(out.image.data_ptr()), ctypes.c_void_p(out.final_transmittance.data_ptr()),
        ctypes.c_void_p(out.contrib_count.data_ptr()), ctypes.c_void_p(grad_image.data_ptr()),
        float(grad_scale), ctypes.byref(g),
        ctypes.c_void_p(pose_dev.data_ptr()) if pose_dev is not None else None,
        _lib.stream_ptr(stream)), "backward")


class Culled:
    """Normal outcome for a splat that cannot contribute to the image (raster.py:78-82)."""

    def __repr__(self):
        return "Culled()"


def splat_batch(source, T_cw, cam, settings: RasterSettings = RasterSettings()):
    """Per-Gaussian screen footprints of `source` on the device (lsb_splat):
    (visible (n,) bool, mu_i (n,2), cov_i (n,2,2), depth (n,), color (n,3)),
    device f64 tensors; the same projection, EWA covariance, footprint cull
    and SH colour as render()'s preprocess (raster.py:134-185, 232-238)."""
    _lib.require()
    arrays = _as_arrays(source)
    T_cw = as_se3(T_cw)
    n = len(arrays)
    dev = arrays.device
    geo = torch.zeros((max(n, 1), 7), dtype=torch.float64, device=dev)
    col = torch.zeros((max(n, 1), 3), dtype=torch.float64, device=dev)
    if n:
        p = arrays.params()
        _lib.check(_lib.load().lsb_splat(ctypes.byref(p), ctypes.byref(_lib.make_camera(cam)),
                                         ctypes.byref(_lib.make_pose(T_cw.R, T_cw.t)),
                                         ctypes.byref(_lib.make_settings(settings, 0)),
                                         ctypes.c_void_p(geo.data_ptr()), ctypes.c_void_p(col.data_ptr()),
                                         _lib.stream_ptr()), "splat")
    geo, col = geo[:n], col[:n]
    cov = torch.stack([geo[:, 3], geo[:, 4], geo[:, 4], geo[:, 5]], dim=1).reshape(n, 2, 2)
    return geo[:, 0] > 0.5, geo[:, 1:3], cov, geo[:, 6], col


def splat(g, T_cw, cam, settings: RasterSettings = RasterSettings()):
    """Project one Gaussian; returns a Gaussian2D or Culled (raster.py:188-205)."""
    from .geometry import Gaussian2D
    vis, mu, cov, depth, col = splat_batch(GaussianArrays.from_gaussians([g], dtype=torch.float64), T_cw, cam,
                                           settings)
    if not bool(vis[0]):
        return Culled()
    return Gaussian2D(mean_i=mu[0].cpu().numpy(), cov_i=cov[0].cpu().numpy(), depth=float(depth[0]),
                      color=col[0].cpu().numpy(), opacity=float(g.opacity))


def render(source, T_wc, cam, settings: RasterSettings = RasterSettings(), retain_cache: bool = True,
           with_depth: bool = False, bin_mode: int = 0) -> RenderOutput:
    """Splat, bin, depth-sort per tile and composite (raster.py:212-264).

    Synchronises once to size the intersection buffers (the reference API is
    synchronous too); the multi-view engine (optimize.WindowEngine) avoids
    that sync.  bin_mode 1 (alpha_cut > 0) bins into contributing tiles only
    (include/lsb.h): same image / T / depth / gradients, but contrib_count
    then counts contributing-list entries instead of the reference's."""
    _lib.require()
    arrays = _as_arrays(source)
    T_cw = as_se3(T_wc).inverse()
    dev = arrays.device
    h, w = int(cam.height), int(cam.width)
    key = (len(arrays), w, h, float(settings.alpha_cut), int(bin_mode))
    cap = max(_CAP_HINT.get(key, 0), 1 << 16, 8 * len(arrays))
    image = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
    t_final = torch.empty((h, w), dtype=torch.float32, device=dev)
    n_contrib = torch.empty((h, w), dtype=torch.int32, device=dev)
    depth = torch.empty((h, w), dtype=torch.float32, device=dev) if with_depth else None
    while True:
        state = RenderState(arrays, cam, T_cw.R, T_cw.t, settings, cap, bin_mode)
        render_fwd(state, image, t_final, n_contrib, depth)
        M, I, overflow, _ = state.read_counts()
        if not overflow:
            break
        cap = int(I * 1.25) + 1024
    _CAP_HINT[key] = int(I * 1.25) + 1024
    return RenderOutput(image=host_readable(image), final_transmittance=host_readable(t_final),
                        contrib_count=host_readable(n_contrib), cache=state if retain_cache else None,
                        depth=host_readable(depth))


def backward(out: RenderOutput, grad_image, T_ic=None):
    """Analytic gradients for image gradient `grad_image` (raster.py:309-399).

    Returns (ParamGradients on the device, PoseGradient)."""
    state = out.cache
    if state is None:
        raise MissingCache("render() must be called with retain_cache=True")
    T_ic = SE3.identity() if T_ic is None else T_ic
    dev = state.ws.device
    h, w = state.dims.height, state.dims.width
    g_img = _f32(grad_image, (h, w, 3), dev)
    grads = ParamGradients.zeros(len(state.arrays), int(state.arrays.shs.shape[1]), dev)
    pose_dev = torch.zeros(9, dtype=torch.float64, device=dev)
    render_bwd(state, out, g_img, 1.0, grads, pose_dev)
    return grads, PoseGradient(pose_dev, state.R_cw, T_ic)


def _degree_used(state: RenderState) -> int:
    K = int(state.arrays.shs.shape[1])
    stored = int(round(np.sqrt(K))) - 1
    return min(int(state.settings.sh_degree), stored)


def pose_rows(out: RenderOutput, pixel_ids, T_ic=None, as_numpy: bool = True):
    """IMU-tangent rows d gray(I_hat(u)) / d xi for selected pixels
    (raster.py:450-508).  pixel_ids are flat row-major indices; returns
    (m, 6) f64 with columns (rho, tau) — numpy by default, else a device
    tensor."""
    state = out.cache
    if state is None:
        raise MissingCache("render() must be called with retain_cache=True")
    T_ic = SE3.identity() if T_ic is None else T_ic
    dev = state.ws.device
    ids = torch.as_tensor(np.asarray(pixel_ids, dtype=np.int32) if not torch.is_tensor(pixel_ids) else pixel_ids)
    ids = ids.to(device=dev, dtype=torch.int32).contiguous()
    m = int(ids.numel())
    rows = torch.zeros((m, 6), dtype=torch.float64, device=dev)
    if m:
        M = state.counts[0] if state.counts is not None else state.read_counts()[0]
        chain = torch.empty((max(M, 1), 48), dtype=torch.float32, device=dev)
        p = state.arrays.params()
        lib = _lib.load()
        _lib.check(lib.lsb_pose_prepare(ctypes.byref(p), ctypes.byref(state.c_cam), ctypes.byref(state.c_pose),
                                        ctypes.byref(state.c_set), state._ws(), state.ws_bytes,
                                        ctypes.byref(state.dims), ctypes.c_void_p(chain.data_ptr()),
                                        _lib.stream_ptr()), "pose_prepare")
        A = imu_camera_adjoint(state.R_cw, T_ic)
        Ac = (ctypes.c_double * 36)(*A.ravel().tolist())
        Rc = (ctypes.c_double * 9)(*state.R_cw.ravel().tolist())
        _lib.check(lib.lsb_pose_rows(ctypes.byref(state.c_set), _degree_used(state), state._ws(), state.ws_bytes,
                                     ctypes.byref(state.dims), ctypes.c_void_p(out.image.data_ptr()),
                                     ctypes.c_void_p(out.contrib_count.data_ptr()), ctypes.c_void_p(chain.data_ptr()),
                                     ctypes.c_void_p(ids.data_ptr()), m, None, Ac, Rc,
                                     ctypes.c_void_p(rows.data_ptr()), _lib.stream_ptr()), "pose_rows")
    return rows.cpu().numpy() if as_numpy else rows
