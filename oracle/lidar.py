"""TEST INFRASTRUCTURE ONLY — CPU restatement of the plane fits and the LiDAR
point-to-plane measurement (livsplat voxmap.py:204-335,
estimator.py:190-238), pinned against tests/golden/lidar.npz (produced by the
reference, tools/make_golden_lidar.py)."""
from __future__ import annotations

import numpy as np

NEIGHBORHOOD = ((0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1))


def leaf_stats(points, leaf_len):
    """key -> [count, sum p, sum p p^T] (voxmap.py:204-230)."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    idx = np.floor(pts / leaf_len).astype(np.int64)
    order = np.lexsort((idx[:, 2], idx[:, 1], idx[:, 0]))
    idx, pts = idx[order], pts[order]
    cuts = np.nonzero(np.any(np.diff(idx, axis=0) != 0, axis=1))[0] + 1
    out = {}
    for ci, cp in zip(np.split(idx, cuts), np.split(pts, cuts)):
        out[tuple(int(v) for v in ci[0])] = [len(cp), cp.sum(axis=0), cp.T @ cp]
    return out


def fit_planes(stats, keys, origin):
    """{key: (normal, centroid) or None} (voxmap.py:297-335)."""
    origin = np.asarray(origin, dtype=float)
    out, pend, cnt, sums, outs, anchors = {}, [], [], [], [], []
    for key in keys:
        st = stats.get(key)
        if st is None or st[0] == 0:
            out[key] = None
            continue
        n_tot, s, so = 0, np.zeros(3), np.zeros((3, 3))
        for dx, dy, dz in NEIGHBORHOOD:
            nb = stats.get((key[0] + dx, key[1] + dy, key[2] + dz))
            if nb is not None:
                n_tot += nb[0]
                s = s + nb[1]
                so = so + nb[2]
        if n_tot < 3:
            out[key] = None
            continue
        pend.append(key)
        cnt.append(n_tot)
        sums.append(s)
        outs.append(so)
        anchors.append(st[1] / st[0])
    if not pend:
        return out
    n = np.asarray(cnt, dtype=float)[:, None]
    mean = np.stack(sums) / n
    scatter = np.stack(outs) / n[:, :, None] - mean[:, :, None] * mean[:, None, :]
    w, v = np.linalg.eigh(scatter)
    ok = w[:, 1] > 1e-12 + 1e-6 * np.maximum(w[:, 2], 0.0)
    normals = v[:, :, 0]
    flip = np.einsum("ij,ij->i", normals, origin[None, :] - mean) < 0
    normals = np.where(flip[:, None], -normals, normals)
    for i, key in enumerate(pend):
        out[key] = (normals[i], np.asarray(anchors[i])) if ok[i] else None
    return out


def lidar_measurement(stats, leaf_len, points_l, R_il, t_il, R_wi, t_wi, gate):
    """(z, H6, kept point indices) (estimator.py:190-238)."""
    pts = np.atleast_2d(np.asarray(points_l, dtype=float))
    origin = R_wi @ t_il + t_wi
    p_i = pts @ R_il.T + t_il
    p_w = p_i @ R_wi.T + t_wi
    keys = [tuple(int(v) for v in k) for k in np.floor(p_w / leaf_len).astype(np.int64)]
    planes = fit_planes(stats, sorted(set(keys)), origin)
    valid = np.array([planes[k] is not None for k in keys])
    normals = np.array([planes[k][0] if planes[k] is not None else np.zeros(3) for k in keys])
    anchors = np.array([planes[k][1] if planes[k] is not None else np.zeros(3) for k in keys])
    n_v = normals[valid]
    res = np.einsum("ij,ij->i", n_v, p_w[valid] - anchors[valid])
    gate_ok = np.abs(res) <= gate
    n_v, res = n_v[gate_ok], res[gate_ok]
    p_iv = p_i[valid][gate_ok]
    H = np.zeros((len(res), 6))
    nR = n_v @ R_wi
    H[:, 0] = -(nR[:, 1] * p_iv[:, 2] - nR[:, 2] * p_iv[:, 1])
    H[:, 1] = -(nR[:, 2] * p_iv[:, 0] - nR[:, 0] * p_iv[:, 2])
    H[:, 2] = -(nR[:, 0] * p_iv[:, 1] - nR[:, 1] * p_iv[:, 0])
    H[:, 3:6] = n_v
    kept = np.flatnonzero(valid)[gate_ok]
    return res, H, kept
