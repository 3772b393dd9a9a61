"""ctypes binding of include/lsb.h (libsplat_b200.so, built in-tree).

This is the only way the package reaches its compute: there is no CPU or
PyTorch fallback.  If the library is missing or no CUDA device is present,
every entry point raises immediately (`require()`).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# LSB_SO selects a tuning variant built next to the default library
SO_PATH = os.environ.get("LSB_SO") or os.path.join(HERE, "libsplat_b200.so")

LSB_OK, LSB_EINVAL, LSB_ECAPACITY, LSB_ECUDA, LSB_EMISSING_CACHE = range(5)

_c = ctypes
_P = _c.c_void_p


class Camera(_c.Structure):
    _fields_ = [("fx", _c.c_double), ("fy", _c.c_double), ("cx", _c.c_double), ("cy", _c.c_double),
                ("width", _c.c_int32), ("height", _c.c_int32)]


class Settings(_c.Structure):
    _fields_ = [("near_plane", _c.c_double), ("dilation", _c.c_double), ("alpha_clamp", _c.c_double),
                ("transmittance_min", _c.c_double), ("footprint_sigma", _c.c_double),
                ("alpha_cut", _c.c_double), ("max_footprint_px", _c.c_double),
                ("background", _c.c_double * 3), ("sh_degree", _c.c_int32), ("bin_mode", _c.c_int32)]


class Pose(_c.Structure):
    _fields_ = [("R", _c.c_double * 9), ("t", _c.c_double * 3), ("cam_center", _c.c_double * 3)]


class Params(_c.Structure):
    _fields_ = [("means", _P), ("rots", _P), ("scales", _P), ("opacities", _P), ("shs", _P),
                ("n", _c.c_int64), ("sh_coeffs", _c.c_int32), ("dtype", _c.c_int32)]


class Grads(_c.Structure):
    _fields_ = [("mean", _P), ("rot", _P), ("scale", _P), ("opacity", _P), ("sh", _P)]


class Dims(_c.Structure):
    _fields_ = [("n", _c.c_int64), ("width", _c.c_int32), ("height", _c.c_int32),
                ("sh_coeffs", _c.c_int32), ("tile", _c.c_int32), ("isect_cap", _c.c_int64)]


class VoxMap(_c.Structure):
    _fields_ = [("keys", _P), ("count", _P), ("sum", _P), ("outer", _P), ("gslot", _P), ("claim", _P),
                ("n_used", _P), ("flags", _P), ("cap", _c.c_int64), ("root_len", _c.c_double),
                ("max_level", _c.c_int32), ("_pad", _c.c_int32), ("gkeys", _P), ("n_gkeys", _P)]


class AdamCfg(_c.Structure):
    _fields_ = [(k, _c.c_double) for k in ("lr_mean", "lr_rot", "lr_scale", "lr_opacity", "lr_sh", "beta1",
                                           "beta2", "eps", "scene_scale", "opacity_clip", "scale_floor")] + [
        ("step", _c.c_int64)]


class VisualCfg(_c.Structure):
    _fields_ = [("budget", _c.c_int32), ("observed_u8", _c.c_int32), ("sh_degree_used", _c.c_int32),
                ("_pad", _c.c_int32), ("grad_thr", _c.c_double), ("t_max", _c.c_double), ("gate", _c.c_double),
                ("inv_sigma2", _c.c_double), ("A", _c.c_double * 36)]


class VisualBufs(_c.Structure):
    _fields_ = [(k, _P) for k in ("mask", "select_scratch", "ids", "res", "chain", "rows", "hb_scratch", "out")]


# (name, restype, argtypes) for every symbol include/lsb.h declares
SIGNATURES = [
    ("lsb_abi_version", _c.c_int, []),
    ("lsb_last_error", _c.c_char_p, []),
    ("lsb_workspace_bytes", _c.c_int, [_c.POINTER(Dims), _c.POINTER(_c.c_size_t)]),
    ("lsb_voxmap_accumulate_temp_bytes", _c.c_int, [_c.c_int64, _c.POINTER(_c.c_size_t)]),
    ("lsb_voxmap_accumulate", _c.c_int, [_c.POINTER(VoxMap), _P, _c.c_int64, _P, _P, _c.c_size_t, _P]),
    ("lsb_sort_temp_bytes", _c.c_int, [_c.c_int64, _c.POINTER(_c.c_size_t)]),
    ("lsb_sort_pairs", _c.c_int, [_P, _P, _P, _P, _c.c_int64, _c.c_int, _P, _c.c_size_t, _P]),
    ("lsb_segments", _c.c_int, [_P, _c.c_int64, _P, _P, _P, _c.c_size_t, _P]),
    ("lsb_splat", _c.c_int, [_c.POINTER(Params), _c.POINTER(Camera), _c.POINTER(Pose), _c.POINTER(Settings),
                             _P, _P, _P]),
    ("lsb_render_fwd", _c.c_int, [_c.POINTER(Params), _c.POINTER(Camera), _c.POINTER(Pose),
                                  _c.POINTER(Settings), _P, _c.c_size_t, _c.POINTER(Dims),
                                  _P, _P, _P, _P, _P]),
    ("lsb_render_counts", _c.c_int, [_P, _c.POINTER(Dims), _c.POINTER(_c.c_int64), _P]),
    ("lsb_render_sticky", _c.c_int, [_P, _c.POINTER(Dims), _c.POINTER(_c.c_int64), _c.c_int, _P]),
    ("lsb_render_band_stats", _c.c_int, [_P, _c.POINTER(Dims), _c.POINTER(_c.c_int64), _P]),
    ("lsb_ieskf_gain", _c.c_int, [_P] * 8),
    ("lsb_ieskf_iterate", _c.c_int, [_P, _P, _P, _P, _P, _c.c_double, _P, _P, _P]),
    ("lsb_visual_pass", _c.c_int, [_c.POINTER(Params), _c.POINTER(Camera), _c.POINTER(Pose), _c.POINTER(Settings),
                                   _P, _c.c_size_t, _c.POINTER(Dims), _P, _P, _P, _P, _c.POINTER(VisualCfg),
                                   _c.POINTER(VisualBufs), _P]),
    ("lsb_render_export", _c.c_int, [_P, _c.POINTER(Dims), _c.c_int, _P, _P]),
    ("lsb_render_bwd", _c.c_int, [_c.POINTER(Params), _c.POINTER(Camera), _c.POINTER(Pose),
                                  _c.POINTER(Settings), _P, _c.c_size_t, _c.POINTER(Dims),
                                  _P, _P, _P, _P, _c.c_float, _c.POINTER(Grads), _P, _P]),
    ("lsb_render_bin", _c.c_int, [_c.POINTER(Params), _c.POINTER(Camera), _c.POINTER(Pose),
                                  _c.POINTER(Settings), _P, _c.c_size_t, _c.POINTER(Dims), _P]),
    ("lsb_render_blend", _c.c_int, [_c.POINTER(Settings), _P, _c.c_size_t, _c.POINTER(Dims), _P, _P, _P, _P,
                                    _P]),
    ("lsb_render_blend_loss", _c.c_int, [_c.POINTER(Settings), _P, _c.c_size_t, _c.POINTER(Dims), _P, _P, _P,
                                         _P, _P, _c.c_int, _c.c_float, _P, _P, _P]),
    ("lsb_render_blend_bwd", _c.c_int, [_c.POINTER(Settings), _P, _c.c_size_t, _c.POINTER(Dims), _P, _P, _P,
                                        _c.c_float, _P]),
    ("lsb_render_blend_fused_loss", _c.c_int, [_c.POINTER(Settings), _P, _c.c_size_t, _c.POINTER(Dims), _P,
                                               _c.c_int, _c.c_float, _P, _P]),
    ("lsb_render_blend_bwd_loss", _c.c_int, [_c.POINTER(Settings), _P, _c.c_size_t, _c.POINTER(Dims), _P, _P,
                                             _c.c_int, _c.c_float, _P, _P]),
    ("lsb_render_chain", _c.c_int, [_c.POINTER(Params), _c.POINTER(Camera), _c.POINTER(Pose),
                                    _c.POINTER(Settings), _P, _c.c_size_t, _c.POINTER(Dims),
                                    _c.POINTER(Grads), _P, _P]),
    ("lsb_adam_step", _c.c_int, [_c.POINTER(Params), _P, _P, _P, _P, _c.POINTER(AdamCfg), _P]),
    ("lsb_adam_step_dev", _c.c_int, [_c.POINTER(Params), _P, _P, _P, _P, _c.POINTER(AdamCfg), _P, _c.c_int64, _P,
                                     _P]),
    ("lsb_adam_step_dev_groups", _c.c_int, [_c.POINTER(Params), _P, _P, _P, _P, _c.POINTER(AdamCfg), _P,
                                            _c.c_int64, _P, _c.c_int32, _c.c_int32, _P]),
    ("lsb_adam_peer_step", _c.c_int, [_P, _c.c_int32, _c.c_int32, _P, _c.c_int64, _c.c_int64, _P, _P, _P,
                                      _c.POINTER(AdamCfg), _P, _c.c_int64, _P, _P]),
    ("lsb_copy_h2d", _c.c_int, [_P, _P, _c.c_size_t, _P]),
    ("lsb_orthonormalize", _c.c_int, [_P, _c.c_int32, _P, _c.c_int64, _P]),
    ("lsb_pose_prepare", _c.c_int, [_c.POINTER(Params), _c.POINTER(Camera), _c.POINTER(Pose),
                                    _c.POINTER(Settings), _P, _c.c_size_t, _c.POINTER(Dims), _P, _P]),
    ("lsb_pose_rows", _c.c_int, [_c.POINTER(Settings), _c.c_int, _P, _c.c_size_t, _c.POINTER(Dims), _P, _P, _P,
                                 _P, _c.c_int64, _P, _c.POINTER(_c.c_double), _c.POINTER(_c.c_double), _P, _P]),
    ("lsb_hb_scratch_doubles", _c.c_int, []),
    ("lsb_hb_reduce", _c.c_int, [_P, _P, _c.c_int64, _P, _c.c_double, _P, _P, _P]),
    ("lsb_visual_select_scratch_bytes", _c.c_int64, [_c.c_int64, _c.c_int32]),
    ("lsb_visual_select", _c.c_int, [_P, _P, _c.c_int32, _P, _c.c_int64, _c.c_int32, _c.c_double, _P, _P, _P, _P,
                                     _P]),
    ("lsb_semidense_mask", _c.c_int, [_P, _c.c_int32, _P, _c.c_int32, _c.c_int32, _c.c_double, _c.c_double, _P, _P]),
    ("lsb_voxmap_keys", _c.c_int, [_P, _c.c_int64, _c.c_double, _P, _P]),
    ("lsb_voxmap_insert_points", _c.c_int, [_c.POINTER(VoxMap), _P, _c.c_int64, _c.c_int32, _P, _P]),
    ("lsb_voxmap_try_insert", _c.c_int, [_c.POINTER(VoxMap), _P, _c.c_int64, _c.c_int32, _P, _P, _P]),
    ("lsb_voxmap_lookup", _c.c_int, [_c.POINTER(VoxMap), _P, _c.c_int64, _P, _P]),
    ("lsb_voxmap_fov", _c.c_int, [_c.POINTER(VoxMap), _P, _c.c_int64, _P, _c.c_int64, _P, _P, _c.c_int64, _P]),
    ("lsb_voxmap_dump", _c.c_int, [_c.POINTER(VoxMap), _P, _P, _P, _c.c_int64, _P]),
    ("lsb_voxmap_rehash", _c.c_int, [_c.POINTER(VoxMap), _c.POINTER(VoxMap), _P]),
    ("lsb_voxmap_fit_planes", _c.c_int, [_c.POINTER(VoxMap), _P, _c.c_int64, _c.POINTER(_c.c_double), _P, _P, _P,
                                         _P]),
    ("lsb_lidar_rows", _c.c_int, [_c.POINTER(VoxMap), _P, _c.c_int64, _c.POINTER(_c.c_double),
                                  _c.POINTER(_c.c_double), _c.POINTER(_c.c_double), _c.POINTER(_c.c_double),
                                  _c.c_double, _P, _P, _P, _P]),
    ("lsb_init_gaussians", _c.c_int, [_c.POINTER(VoxMap), _P, _P, _c.c_int64, _P, _c.c_int32, _c.c_int32,
                                      _c.POINTER(_c.c_double), _c.POINTER(_c.c_double), _c.POINTER(_c.c_double),
                                      _c.POINTER(_c.c_double), _c.c_double, _c.c_double, _c.c_double, _c.c_double,
                                      _c.c_int32, _P, _P, _P]),
    ("lsb_segment_mean", _c.c_int, [_P, _P, _P, _P, _c.c_int64, _P, _P]),
    ("lsb_window_mark", _c.c_int, [_P, _c.c_int64, _P, _P, _c.c_int64, _P, _c.c_int64, _P, _P, _P]),
    ("lsb_window_plan_tiles", _c.c_int64, [_c.c_int64]),
    ("lsb_window_append_tiles", _c.c_int64, [_c.c_int64]),
    ("lsb_window_plan", _c.c_int, [_P, _c.c_int64, _P, _P, _P, _P, _P]),
    ("lsb_window_compact", _c.c_int, [_c.POINTER(VoxMap), _c.POINTER(Params), _P, _P, _c.c_int64, _P, _c.c_int64,
                                      _c.c_int64, _P, _P]),
    ("lsb_window_leaf_gids", _c.c_int, [_c.POINTER(VoxMap), _P, _c.c_int64, _P, _P]),
    ("lsb_window_dist", _c.c_int, [_P, _c.c_int64, _c.c_double, _c.POINTER(_c.c_double), _P, _P]),
    ("lsb_window_append", _c.c_int, [_c.POINTER(Params), _P, _P, _P, _c.c_int64, _P, _c.c_int64, _P, _P, _P]),
    ("lsb_loss_scratch_doubles", _c.c_int, []),
    ("lsb_photometric_loss", _c.c_int, [_P, _P, _P, _c.c_int64, _c.c_int64, _c.c_int, _c.c_float,
                                        _P, _P, _P]),
]

_lib = None


def load(path: str = SO_PATH):
    """Load the shared library and bind every declared symbol (no GPU needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2501_08672_b200.build_ext` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def require():
    """The library, after checking a CUDA device is present (fail loudly)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2501_08672_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return load()


def check(rc: int, what: str) -> None:
    if rc == LSB_OK:
        return
    msg = f"{what}: {load().lsb_last_error().decode(errors='replace')}"
    if rc == LSB_EMISSING_CACHE:
        from .errors import MissingCache
        raise MissingCache(msg)
    if rc == LSB_EINVAL:
        raise ValueError(msg)
    if rc == LSB_ECAPACITY:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def ptr(t) -> int | None:
    """Device address of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def make_camera(cam) -> Camera:
    return Camera(float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy), int(cam.width),
                  int(cam.height))


def make_settings(s, bin_mode: int = 0) -> Settings:
    """RasterSettings -> lsb_settings.  bin_mode 1 (contributing tile lists)
    only takes effect with alpha_cut > 0 (include/lsb.h)."""
    bg = np.asarray(s.background, dtype=np.float64).reshape(3)
    return Settings(float(s.near), float(s.dilation), float(s.alpha_clamp), float(s.transmittance_min),
                    float(s.footprint_sigma), float(s.alpha_cut), float(s.max_footprint_px),
                    (ctypes.c_double * 3)(*bg.tolist()), int(s.sh_degree), int(bin_mode))


def make_pose(R_cw: np.ndarray, t_cw: np.ndarray) -> Pose:
    R = np.asarray(R_cw, dtype=np.float64).reshape(3, 3)
    t = np.asarray(t_cw, dtype=np.float64).reshape(3)
    cc = -R.T @ t               # raster.py:233 (same numpy expression, same bits)
    return Pose((ctypes.c_double * 9)(*R.ravel().tolist()), (ctypes.c_double * 3)(*t.tolist()),
                (ctypes.c_double * 3)(*cc.tolist()))
