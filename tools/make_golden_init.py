"""Golden fixture for the batched Gaussian initialisation (SURVEY.md §8(f)
rank 3: pipeline.py:99-137 + initialize.py:22-124), produced by the
REFERENCE's functions in this container.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_init.py

A map (root 0.4 m, max_level 2) holds an earlier scan's statistics and a few
Gaussians; a new scan is grouped by leaf, its statistics added, and every
group is offered to `_insert_new_gaussians`' loop (restated here verbatim
around the reference's own init_gaussian / estimate_normal / try_insert):
observability pre-check, plane normal with the view-direction fallback,
bilinear colour from an f32 image, slab frame, scale, opacity, SH.  Recorded:
the scans, the pre-existing Gaussians' keys, the camera, the image and, per
group (sorted key order), the created Gaussian's row or "skipped".
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from livsplat.errors import BehindCamera, OutOfBounds  # noqa: E402
from livsplat.geometry import Gaussian3D, PinholeCamera, SE3, so3_exp  # noqa: E402
from livsplat.initialize import init_gaussian  # noqa: E402
from livsplat.voxmap import HashOctree, voxel_center  # noqa: E402

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(HERE, "tests", "golden", "init.npz")
sys.path.insert(0, os.path.join(HERE, "tools"))
from make_golden_lidar import scene  # noqa: E402


def main():
    rng = np.random.default_rng(21)
    vmap = HashOctree(root_len=0.4, max_level=2, leaf_capacity=1)
    scan0 = scene(np.random.default_rng(22), scale=0.5)
    for key, pts in vmap.group_by_leaf(scan0).items():
        vmap.ensure_leaf(key)
        vmap.add_leaf_stats(key, pts)
    # a few leaves already hold a Gaussian (the loop must skip them)
    keys0 = sorted(vmap.leaf_stats.keys())[::7]
    for k in keys0:
        vmap.ensure_leaf(k).gaussians = [Gaussian3D(mean_w=voxel_center(k, 0.4), rot=np.eye(3), scale=[1e-3, .05, .05],
                                                    opacity=0.9, sh=np.zeros((1, 3)), level=2)]
    scan1 = scene(np.random.default_rng(23), scale=0.3)
    cam = PinholeCamera(fx=60.0, fy=60.0, cx=32.0, cy=24.0, width=64, height=48)
    T_wc = SE3(so3_exp([-1.9, 0.1, 0.2]), [0.2, -0.3, 1.0])
    T_cw = T_wc.inverse()
    origin = np.array([0.25, -0.2, 1.1])
    yy, xx = np.mgrid[0:48, 0:64]
    image = np.stack([0.5 + 0.4 * np.sin(xx / 7.0), 0.5 + 0.4 * np.cos(yy / 5.0), (xx + yy) / 120.0], -1)
    image = image.astype(np.float32).astype(np.float64)
    groups = vmap.group_by_leaf(scan1)
    for key, pts in groups.items():
        vmap.ensure_leaf(key)
        vmap.add_leaf_stats(key, pts)
    gkeys, rows, created = [], [], []
    near, kappa, delta, opacity = 0.01, 0.8, 1e-3, 0.9
    for key in sorted(groups.keys()):               # pipeline.py:106-137
        gkeys.append(key[:3])
        node = vmap.get_leaf(key)
        row = np.full(19, np.nan)
        ok = False
        if node is not None and len(node.gaussians) < 1:
            centroid = groups[key].mean(axis=0)
            p_c = T_cw.apply(centroid)
            if p_c[2] > near:
                u = cam.fx * p_c[0] / p_c[2] + cam.cx
                v = cam.fy * p_c[1] / p_c[2] + cam.cy
                if 1.0 <= u <= cam.width - 2 and 1.0 <= v <= cam.height - 2:
                    try:
                        normal = vmap.estimate_normal(key, origin)
                    except Exception:
                        view = origin - centroid
                        nv = np.linalg.norm(view)
                        normal = view / nv if nv != 0 else None
                    if normal is not None:
                        try:
                            g = init_gaussian(centroid, normal, 2, image, T_wc, cam, 0.4, kappa=kappa, delta=delta,
                                              opacity=opacity, sh_degree=0, near=near)
                            vmap.try_insert(g)
                            row = np.concatenate([g.mean_w, g.rot.ravel(), g.scale, [g.opacity], g.sh.ravel()])
                            ok = True
                        except (BehindCamera, OutOfBounds):
                            pass
        rows.append(row)
        created.append(ok)
    np.savez_compressed(OUT, scan0=scan0, scan1=scan1, keys0=np.array([k[:3] for k in keys0], dtype=np.int64),
                        image=image.astype(np.float32), cam=[cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height],
                        R_wc=T_wc.R, t_wc=T_wc.t, origin=origin, near=near, kappa=kappa, delta=delta,
                        opacity=opacity, gkeys=np.array(gkeys, dtype=np.int64), rows=np.array(rows),
                        created=np.array(created))
    print("wrote", OUT, "groups", len(gkeys), "created", int(np.sum(created)))


if __name__ == "__main__":
    main()
