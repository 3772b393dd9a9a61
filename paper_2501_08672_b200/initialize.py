"""Batched LiDAR-camera initialisation of new Gaussians on the B200 — the
per-leaf loop of pipeline._insert_new_gaussians with initialize.init_gaussian
(pipeline.py:99-137, initialize.py:22-124), SURVEY.md §8(f) rank 3.

One call per scan: the scan's world points are grouped by leaf (stable, so
each group keeps scan order and its centroid is numpy's axis-0 mean),
and one device thread per group (sorted key order, like the reference's
loop) skips leaves that already hold a Gaussian, applies the observability
pre-check, fits the plane normal (view-direction fallback), samples the
image bilinearly, and emits the slab-frame Gaussian row; the rows go into
the map's device store (`HashOctree.set_gaussians_dev`).  The grouping is
the library's own stable radix sort and run segmentation (csrc/sort.cu).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .geometry import as_se3
from .sort import segments, sort_pairs
from .voxmap import HashOctree, keys_of_points_dev
from .window import order_keys, unpack_order_keys


def insert_new_gaussians(vmap: HashOctree, points_w, image, T_wc, cam, sensor_origin, kappa: float = 0.5,
                         delta: float = 1e-3, opacity: float = 0.9, sh_coeffs: int = 1, near: float = 0.01,
                         accumulate: bool = True):
    """Create one Gaussian per newly observed leaf of this scan.

    points_w (n,3) world points of the scan (added to the leaf statistics
    first when `accumulate`, as pipeline.py:183-187 does), image (H,W,3) in
    [0,1], T_wc the camera pose.  Returns (keys (k,3), rows (k, 16+3K) f32,
    created (k,) bool) for the scan's leaf groups in sorted key order; the
    created rows are already stored in the map."""
    _lib.require()
    dev = vmap.device
    pts = torch.as_tensor(np.atleast_2d(np.asarray(points_w, dtype=np.float64))) if not torch.is_tensor(points_w) \
        else points_w
    pts = pts.to(device=dev, dtype=torch.float64).reshape(-1, 3).contiguous()
    if accumulate:
        vmap.accumulate_points_dev(pts)
    R = 16 + 3 * int(sh_coeffs)
    if pts.shape[0] == 0:
        return (torch.empty((0, 3), dtype=torch.int64, device=dev), torch.empty((0, R), device=dev),
                torch.empty(0, dtype=torch.bool, device=dev))
    keys = keys_of_points_dev(pts, vmap.leaf_len, dev)
    skeys, perm32 = sort_pairs(order_keys(keys), key_bits=63, signed=False)
    starts = segments(skeys)
    k = int(starts.numel())
    uniq = skeys[starts]
    counts = torch.diff(starts, append=torch.full((1,), skeys.numel(), dtype=torch.int64, device=dev))
    perm = perm32.to(torch.int64)
    cent = torch.empty((k, 3), dtype=torch.float64, device=dev)
    lib = _lib.load()
    _lib.check(lib.lsb_segment_mean(ctypes.c_void_p(pts.data_ptr()), ctypes.c_void_p(perm.data_ptr()),
                                    ctypes.c_void_p(starts.data_ptr()), ctypes.c_void_p(counts.data_ptr()), k,
                                    ctypes.c_void_p(cent.data_ptr()), _lib.stream_ptr()), "segment_mean")
    gkeys = unpack_order_keys(uniq).contiguous()
    img = torch.as_tensor(image, dtype=torch.float32).to(dev).contiguous()
    h, w = int(img.shape[0]), int(img.shape[1])
    T_cw = as_se3(T_wc).inverse()
    c = lambda a, n: (ctypes.c_double * n)(*np.asarray(a, dtype=np.float64).ravel().tolist())
    rows = torch.empty((k, R), dtype=torch.float32, device=dev)
    status = torch.empty(k, dtype=torch.uint8, device=dev)
    m = vmap.struct()
    _lib.check(lib.lsb_init_gaussians(ctypes.byref(m), ctypes.c_void_p(gkeys.data_ptr()),
                                      ctypes.c_void_p(cent.data_ptr()), k, ctypes.c_void_p(img.data_ptr()), w, h,
                                      c(T_cw.R, 9), c(T_cw.t, 3), c([cam.fx, cam.fy, cam.cx, cam.cy], 4),
                                      c(sensor_origin, 3), float(near), float(kappa), float(delta), float(opacity),
                                      int(sh_coeffs), ctypes.c_void_p(rows.data_ptr()),
                                      ctypes.c_void_p(status.data_ptr()), _lib.stream_ptr()), "init_gaussians")
    made = status.bool()
    if bool(made.any()):
        vmap.set_gaussians_dev(gkeys[made], rows[made])
    return gkeys, rows, made
