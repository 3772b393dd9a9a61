"""Golden fixture for the plane fits and the LiDAR point-to-plane measurement
(SURVEY.md §8(f) rank 2), produced by the REFERENCE (livsplat, read-only at
/root/reference/pkg/src) in this container.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_lidar.py

A map (root 0.4 m, max_level 2) accumulates ~30k noisy points on a floor,
two walls and a box (plus sparse clutter that gives degenerate leaves);
`fit_planes` (voxmap.py:297-335) runs on every touched leaf plus some empty
neighbours; `lidar_measurement` (estimator.py:190-238) runs for a second,
sparser scan seen from a perturbed IMU pose.  Recorded: the points, the
keys, the origin, normals / anchors / validity, and the measurement z, H
and the kept point indices.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from livsplat.estimator import FilterConfig, NavState, lidar_measurement  # noqa: E402
from livsplat.geometry import SE3, so3_exp  # noqa: E402
from livsplat.voxmap import HashOctree, VoxelKey, keys_of_points  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "lidar.npz")


def plane_points(rng, n, origin, u, v, noise):
    a, b = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    nrm = np.cross(u, v)
    nrm = nrm / np.linalg.norm(nrm)
    return origin + a[:, None] * u + b[:, None] * v + rng.normal(0, noise, n)[:, None] * nrm


def scene(rng, scale=1.0):
    pts = [plane_points(rng, int(12000 * scale), np.array([-2.0, -2.0, 0.0]), np.array([4.0, 0, 0]),
                        np.array([0, 4.0, 0]), 0.002),                                  # floor
           plane_points(rng, int(8000 * scale), np.array([-2.0, 2.0, 0.0]), np.array([4.0, 0, 0]),
                        np.array([0, 0, 2.5]), 0.002),                                  # wall y = 2
           plane_points(rng, int(8000 * scale), np.array([2.0, -2.0, 0.0]), np.array([0, 4.0, 0]),
                        np.array([0, 0, 2.5]), 0.002),                                  # wall x = 2
           plane_points(rng, int(2000 * scale), np.array([0.3, 0.3, 0.0]), np.array([0.5, 0.2, 0]),
                        np.array([0, 0, 0.6]), 0.001),                                  # slanted box face
           rng.uniform([-2, -2, 0], [2, 2, 2.5], (int(300 * scale), 3))]                # clutter
    return np.concatenate(pts)


def main():
    rng = np.random.default_rng(11)
    vmap = HashOctree(root_len=0.4, max_level=2, leaf_capacity=1)
    pts = scene(rng)
    vmap.accumulate_points(pts)
    touched = sorted(set(keys_of_points(pts, vmap.leaf_len, vmap.max_level)))
    extra = [VoxelKey(k.ix + 1, k.iy + 2, k.iz + 3, k.level) for k in touched[::50]]
    keys = sorted(set(touched) | set(extra))
    origin = np.array([0.1, -0.2, 1.2])
    fits = vmap.fit_planes(keys, origin)
    normals = np.full((len(keys), 3), np.nan)
    anchors = np.full((len(keys), 3), np.nan)
    valid = np.zeros(len(keys), dtype=bool)
    for i, k in enumerate(keys):
        if fits[k] is not None:
            normals[i], anchors[i] = fits[k]
            valid[i] = True

    # LiDAR measurement: a second scan, in the LiDAR frame, from a perturbed pose
    T_il = SE3(so3_exp([0.01, -0.02, 0.03]), [0.03, 0.0, 0.05])
    T_true = SE3(so3_exp([0.0, 0.0, 0.4]), [0.1, -0.2, 1.1])
    scan_w = scene(np.random.default_rng(12), scale=0.3)
    T_wl_true = T_true @ T_il
    points_l = T_wl_true.inverse().apply(scan_w)
    state = NavState(SE3(T_true.R @ so3_exp([0.003, -0.002, 0.004]), T_true.t + np.array([0.02, -0.01, 0.015])))
    cfg = FilterConfig()
    meas = lidar_measurement(state, points_l, vmap, T_il, cfg)
    assert not np.any(meas.H[:, 6:])           # only the pose block is non-zero
    np.savez_compressed(
        OUT, root_len=0.4, max_level=2, points=pts, keys=np.array([k[:3] for k in keys], dtype=np.int64),
        origin=origin, normals=normals, anchors=anchors, valid=valid,
        T_il_R=T_il.R, T_il_t=T_il.t, T_wi_R=state.T_WI.R, T_wi_t=state.T_WI.t, points_l=points_l,
        lidar_gate=cfg.lidar_gate, lidar_sigma=cfg.lidar_sigma, z=meas.z, H6=meas.H[:, :6], R_diag=meas.R_diag)
    print("wrote", OUT, "keys", len(keys), "valid", int(valid.sum()), "rows", len(meas.z))


if __name__ == "__main__":
    main()
