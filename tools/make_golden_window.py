"""Golden fixture for the sliding-window maintain protocol, produced by the
REFERENCE (livsplat.window.GaussianWindow + livsplat.voxmap.HashOctree,
read-only at /root/reference/pkg/src) in this container.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_window.py

Scenario (window.py:254-276 `maintain`): a 10x10x4 leaf universe (root 0.8 m,
max_level 1), 85% of the leaves seeded with one random Gaussian; 40 frames of
a random walk whose FoV is a box of leaves around the walker; window
capacity 70, so frames that would overflow drop the farthest adds (ranked by
distance to the sensor position, ties by key); from frame 20 on an init_fn
synthesises Gaussians for FoV leaves that have none (window.py:186-199);
between frames a device-side "optimisation" perturbs every live row, as
test_window.py:257-260 does.  Recorded per frame: the FoV keys and sensor
position (inputs), the live keys in slot order, the live rows (f32), and the
report counts.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from livsplat.geometry import Gaussian3D, so3_exp  # noqa: E402
from livsplat.voxmap import HashOctree, VoxelKey, voxel_center  # noqa: E402
from livsplat.window import GaussianWindow  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "window_walk.npz")
ROOT_LEN, MAX_LEVEL, CAP, FRAMES, K = 0.8, 1, 70, 40, 4


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def gaussian_for(rng, center):
    return Gaussian3D(mean_w=f32(center + rng.uniform(-0.1, 0.1, 3)), rot=f32(so3_exp(rng.normal(size=3))),
                      scale=f32(rng.uniform(0.01, 0.2, 3)), opacity=float(np.float32(rng.uniform(0.2, 0.95))),
                      sh=f32(rng.uniform(-0.5, 0.5, (K, 3))), level=MAX_LEVEL)


def init_gaussian(key):
    """Deterministic per-key synthesis (the GPU side replays the same rows)."""
    c = voxel_center(key, ROOT_LEN)
    s = 0.001 * (key.ix + 10 * key.iy + 100 * key.iz + 1)
    return Gaussian3D(mean_w=f32(c), rot=np.eye(3), scale=f32([1e-3, 0.1 + s, 0.1]), opacity=0.5,
                      sh=f32(np.full((K, 3), s)), level=MAX_LEVEL)


def rows_of(win, n):
    a = win.device
    return np.concatenate([a.means[:n], a.rots[:n], a.scales[:n], a.opacities[:n, None],
                           a.shs[:n].reshape(n, -1)], axis=1).astype(np.float32)


def main():
    rng = np.random.default_rng(7)
    vmap = HashOctree(root_len=ROOT_LEN, max_level=MAX_LEVEL, leaf_capacity=1)
    universe = [VoxelKey(x, y, z, MAX_LEVEL) for x in range(10) for y in range(10) for z in range(4)]
    seeded = [k for k in universe if rng.uniform() < 0.85]
    seed_rows = []
    for k in seeded:
        g = gaussian_for(rng, voxel_center(k, ROOT_LEN))
        vmap.ensure_leaf(k).gaussians = [g]
        seed_rows.append(np.concatenate([g.mean_w, g.rot.ravel(), g.scale, [g.opacity], g.sh.ravel()]))
    win = GaussianWindow(capacity=CAP, sh_coeffs=K)
    center = np.array([5.0, 5.0, 2.0])
    rec = {"fov_off": [0], "fov": [], "sensor": [], "n": [], "live_off": [0], "live": [], "rows": [],
           "report": []}
    for f in range(FRAMES):
        center = np.clip(center + rng.integers(-1, 2, size=3), [1, 1, 0], [8, 8, 3])
        r = int(rng.integers(1, 4))
        fov = {k for k in universe if np.abs(np.array(k[:3]) - center).max() <= r}
        sensor = (center + 0.5) * (ROOT_LEN / 2) + rng.uniform(-0.05, 0.05, 3)
        rep = win.maintain(vmap, fov, init_fn=init_gaussian_list if f >= 20 else None, sensor_pos=sensor)
        win.audit()
        n = win.n
        keys = np.array([win.key_of_slot[s][:3] for s in range(n)], dtype=np.int64).reshape(n, 3)
        fk = np.array(sorted(k[:3] for k in fov), dtype=np.int64).reshape(-1, 3)
        rec["fov"].append(fk)
        rec["fov_off"].append(rec["fov_off"][-1] + len(fk))
        rec["sensor"].append(sensor)
        rec["n"].append(n)
        rec["live"].append(keys)
        rec["live_off"].append(rec["live_off"][-1] + n)
        rec["rows"].append(rows_of(win, n))
        rec["report"].append([rep.n_live, rep.added, rep.removed, rep.moved, rep.dropped])
        # device-side optimisation between frames (test_window.py:257-260)
        for key, slot in win.sht.items():
            win.device.shs[slot, 0, 0] += np.float32(0.01 * (key.ix + 1))
            win.device.opacities[slot] = np.float32(win.device.opacities[slot] * np.float32(0.99))
        win.mark_device_dirty_live()
    np.savez_compressed(
        OUT, root_len=ROOT_LEN, max_level=MAX_LEVEL, capacity=CAP, sh_coeffs=K,
        seeded=np.array([k[:3] for k in seeded], dtype=np.int64), seed_rows=np.array(seed_rows, dtype=np.float32),
        fov=np.concatenate(rec["fov"]), fov_off=np.array(rec["fov_off"]), sensor=np.array(rec["sensor"]),
        n=np.array(rec["n"]), live=np.concatenate(rec["live"]), live_off=np.array(rec["live_off"]),
        rows=np.concatenate(rec["rows"]), report=np.array(rec["report"], dtype=np.int64))
    print("wrote", OUT, "frames", FRAMES, "final n", win.n, "reports", rec["report"][-5:])


def init_gaussian_list(key):
    return [init_gaussian(key)]


if __name__ == "__main__":
    main()
