"""Synthetic benchmark inputs (bench and test support, not part of the product
package): the reference's own scene generator, restated.

The reference bakes its benchmark scenes with sim.bake_scene(default_room())
(sim.py:131-169, 436-445): one Gaussian per surface leaf voxel of a textured
box room, with exact normals and texture-sampled colours.  This module
re-derives the same Gaussians with vectorised numpy (the reference's per-
sample Python loop takes minutes at 2M Gaussians), in the same emission
order, and the orbit keyframe poses of the reference CLI (cli.py:90-95,
126-127).  tests/test_scene.py checks it against the reference's output.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2501_08672_b200.geometry import SE3

SH_C0 = 0.28209479177387814
T_IC = SE3(np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]]), [0.05, 0.0, 0.0])


@dataclass
class Checker:
    color_a: tuple = (0.85, 0.85, 0.85)
    color_b: tuple = (0.15, 0.15, 0.15)
    cells: int = 8

    def sample(self, u, v):
        flag = ((np.floor(u * self.cells) + np.floor(v * self.cells)) % 2).astype(bool)
        return np.where(flag[..., None], np.asarray(self.color_a, float), np.asarray(self.color_b, float))


@dataclass
class GradientTex:
    color_a: tuple = (0.1, 0.2, 0.7)
    color_b: tuple = (0.9, 0.8, 0.2)
    axis: int = 0

    def sample(self, u, v):
        w = np.asarray(u if self.axis == 0 else v, dtype=float)[..., None]
        a = np.asarray(self.color_a, dtype=float)
        b = np.asarray(self.color_b, dtype=float)
        return a + (b - a) * np.clip(w, 0.0, 1.0)


@dataclass
class NoiseTex:
    base: tuple = (0.5, 0.5, 0.5)
    amplitude: float = 0.25
    seed: int = 0
    cells: int = 16

    def sample(self, u, v):
        iu = np.floor(np.asarray(u) * self.cells)
        iv = np.floor(np.asarray(v) * self.cells)
        out = np.empty(np.broadcast(iu, iv).shape + (3,))
        for c in range(3):
            h = np.sin(iu * 12.9898 + iv * 78.233 + self.seed * 0.618 + c * 3.7) * 43758.5453
            out[..., c] = self.base[c] + self.amplitude * (2.0 * (h - np.floor(h)) - 1.0)
        return np.clip(out, 0.05, 0.95)


@dataclass
class Rect:
    origin: np.ndarray
    edge_u: np.ndarray
    edge_v: np.ndarray
    texture: object = field(default_factory=Checker)

    @property
    def normal(self) -> np.ndarray:
        n = np.cross(self.edge_u, self.edge_v)
        return n / np.linalg.norm(n)


def box_rects(center, half, texture, inward=False):
    c = np.asarray(center, dtype=float)
    h = np.asarray(half, dtype=float)
    rects = []
    for axis in range(3):
        for sign in (-1.0, 1.0):
            n = np.zeros(3)
            n[axis] = sign
            ua, va = np.zeros(3), np.zeros(3)
            a1, a2 = (axis + 1) % 3, (axis + 2) % 3
            ua[a1] = 2 * h[a1]
            va[a2] = 2 * h[a2]
            if (sign < 0) != inward:
                ua, va = va, ua
            rects.append(Rect(c + n * h[axis] - 0.5 * (ua + va), ua, va, texture))
    return rects


def default_room(scale: float = 4.0):
    s = scale
    return (box_rects([0, 0, s / 4], [s / 2, s / 2, s / 4], Checker(cells=10), inward=True)
            + box_rects([s / 5, s / 8, 0.3], [0.3, 0.3, 0.3],
                        GradientTex((0.8, 0.3, 0.2), (0.9, 0.8, 0.3), axis=0))
            + box_rects([-s / 5, -s / 6, 0.25], [0.25, 0.25, 0.25], NoiseTex((0.4, 0.5, 0.6), 0.2, seed=3)))


def slab_frame(n) -> np.ndarray:
    """Columns (n, u, n x u) with u from the world x-axis (initialize.py:38-61)."""
    n = np.asarray(n, dtype=float)
    u = np.cross([1.0, 0.0, 0.0], n)
    nu = np.linalg.norm(u)
    if nu < 1e-6:
        u = np.cross([0.0, 1.0, 0.0], n)
        nu = np.linalg.norm(u)
    u = u / nu
    return np.column_stack([n, u, np.cross(n, u)])


def bake_room(v_s: float, max_level: int = 2, kappa: float = 0.8, delta: float = 1e-3,
              opacity: float = 0.9, sh_degree: int = 0, rects=None):
    """One Gaussian per surface leaf voxel, first-come per leaf key
    (sim.py:131-169).  Returns f64 numpy arrays (means, rots, scales,
    opacities, shs)."""
    rects = default_room() if rects is None else rects
    edge = v_s / (1 << max_level)
    s_in = kappa * (v_s / (1 << max_level))
    k = (sh_degree + 1) ** 2
    pts, keys, cols, rots = [], [], [], []
    for rect in rects:
        lu, lv = np.linalg.norm(rect.edge_u), np.linalg.norm(rect.edge_v)
        nu, nv = max(1, int(np.ceil(lu / edge))), max(1, int(np.ceil(lv / edge)))
        uu = (np.arange(nu) + 0.5) / nu
        vv = (np.arange(nv) + 0.5) / nv
        UU, VV = np.meshgrid(uu, vv, indexing="ij")
        p = (rect.origin[None, None, :] + UU[..., None] * rect.edge_u[None, None, :]) \
            + VV[..., None] * rect.edge_v[None, None, :]
        p = p.reshape(-1, 3)
        pts.append(p)
        keys.append(np.floor(p / (v_s / (1 << max_level))).astype(np.int64))
        cols.append(rect.texture.sample(UU.ravel(), VV.ravel()))
        rots.append(np.broadcast_to(slab_frame(rect.normal), (len(p), 3, 3)))
    pts = np.concatenate(pts)
    keys = np.concatenate(keys)
    cols = np.concatenate(cols)
    rots = np.concatenate(rots)
    _, first = np.unique(keys, axis=0, return_index=True)
    keep = np.sort(first)
    n = len(keep)
    shs = np.zeros((n, k, 3))
    shs[:, 0, :] = (cols[keep] - 0.5) / SH_C0
    scales = np.tile([delta, s_in, s_in], (n, 1))
    return pts[keep], rots[keep], scales, np.full(n, float(opacity)), shs


# v_s -> N on the default room: 0.323 -> 9,896;
# 0.0723 -> 203,877; 0.0457 -> 512,808; 0.0229 -> 2,040,705.
CONFIG_VS = {"cfg1": 0.323, "cfg2": 0.0723, "cfg4": 0.0457, "cfg5": 0.0229}


def orbit_imu_pose(a: float) -> SE3:
    c, s = np.cos(a + np.pi / 2), np.sin(a + np.pi / 2)
    return SE3(np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]]), [np.cos(a), np.sin(a), 1.0])


def orbit_views(n_views: int):
    """Keyframe camera poses T_WC on the CLI orbit, yaw in linspace(0, 1.5 pi)."""
    return [orbit_imu_pose(a) @ T_IC for a in np.linspace(0.0, 1.5 * np.pi, n_views)]


def camera_for(width: int, height: int):
    from paper_2501_08672_b200.geometry import PinholeCamera
    return PinholeCamera(0.9375 * width, 0.9375 * width, width / 2, height / 2, width, height)


# -- LiDAR scans of the room (benchmark input for the voxel map, config 3) ----

T_LI = SE3(np.eye(3), [0.03, 0.0, 0.05])      # cli.py:128


def room_triangles(rects=None) -> np.ndarray:
    """(T, 3, 3) triangles, two per rectangle (sim.py:83-86)."""
    rects = default_room() if rects is None else rects
    tris = []
    for r in rects:
        o, u, v = r.origin, r.edge_u, r.edge_v
        tris += [[o, o + u, o + u + v], [o, o + u + v, o + v]]
    return np.asarray(tris, dtype=np.float64)


def scan_directions(n_az=1000, n_el=100, az_span=2 * np.pi, el_span=np.deg2rad(80.0)) -> np.ndarray:
    """ScanPattern.directions (sim.py:300-310): (n_az * n_el, 3) unit rays."""
    az = np.linspace(-az_span / 2, az_span / 2, n_az)
    el = np.linspace(-el_span / 2, el_span / 2, n_el)
    aa, ee = np.meshgrid(az, el, indexing="ij")
    return np.stack([np.cos(ee) * np.cos(aa), np.cos(ee) * np.sin(aa), np.sin(ee)], axis=-1).reshape(-1, 3)


def lidar_scan(T_wl, tris, dirs_l, device="cpu", chunk=1 << 15):
    """Nearest-hit ray casting (Moeller-Trumbore, sim.py:321-346) of the scan
    pattern from T_wl; returns the world-frame hit points (f64 tensor)."""
    import torch
    R = torch.as_tensor(np.asarray(T_wl.R), dtype=torch.float64, device=device)
    o = torch.as_tensor(np.asarray(T_wl.t), dtype=torch.float64, device=device)
    tr = torch.as_tensor(tris, dtype=torch.float64, device=device)
    d_all = torch.as_tensor(dirs_l, dtype=torch.float64, device=device) @ R.T
    v0, e1, e2 = tr[:, 0], tr[:, 1] - tr[:, 0], tr[:, 2] - tr[:, 0]
    tvec = o[None, :] - v0
    qvec = torch.cross(tvec, e1, dim=1)
    out = []
    for s in range(0, d_all.shape[0], chunk):
        d = d_all[s:s + chunk]
        pvec = torch.cross(d[:, None, :].expand(-1, tr.shape[0], -1), e2[None].expand(d.shape[0], -1, -1), dim=2)
        det = (e1[None] * pvec).sum(-1)
        ok = det.abs() > 1e-12
        inv = torch.where(ok, 1.0 / torch.where(ok, det, torch.ones_like(det)), torch.zeros_like(det))
        u = (tvec[None] * pvec).sum(-1) * inv
        v = (d[:, None, :] * qvec[None]).sum(-1) * inv
        t = (e2 * qvec).sum(-1)[None] * inv
        valid = ok & (u >= -1e-12) & (v >= -1e-12) & (u + v <= 1 + 1e-12) & (t > 1e-6)
        t = torch.where(valid, t, torch.full_like(t, float("inf")))
        best = t.min(dim=1).values
        hit = torch.isfinite(best)
        out.append(o[None, :] + d[hit] * best[hit, None])
    return torch.cat(out, dim=0)
