"""TEST INFRASTRUCTURE ONLY — CPU oracle for render / backward / pose_rows.

A numpy (+ the C kernels in oracle/blend.c) restatement of the reference's
splatting path, /root/reference/pkg/src/livsplat/raster.py and sh.py.  It is
pinned against golden vectors produced by the reference itself
(tests/golden/, made by tools/make_golden.py) in tests/test_oracle_golden.py.
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use it.

Inputs are plain namespaces / dicts:
  P    : means (N,3), rots (N,3,3), scales (N,3), opacities (N,), shs (N,K,3), f64
  R_cw, t_cw : world->camera rotation / translation (T_cw = T_wc^-1)
  cam  : fx, fy, cx, cy, width, height
  st   : near, dilation, alpha_clamp, transmittance_min, footprint_sigma,
         alpha_cut, max_footprint_px, background (3,), sh_degree
"""

from __future__ import annotations

import numpy as np

from . import _clib
from ._clib import f64, i64, ptr

# Real SH constants (reference sh.py:12-29; standard real spherical harmonics).
C0 = 0.28209479177387814
C1 = 0.4886025119029199
C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
      -1.0925484305920792, 0.5462742152960396)
C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
      0.3731763325901154, -0.4570457994644658, 1.445305721320277,
      -0.5900435899266435)


def sh_basis(degree: int, d: np.ndarray) -> np.ndarray:
    """sh.py:36-63 eval_basis."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    cols = [np.full(len(d), C0)]
    if degree >= 1:
        cols += [-C1 * y, C1 * z, -C1 * x]
    if degree >= 2:
        xx, yy, zz = x * x, y * y, z * z
        cols += [C2[0] * x * y, C2[1] * y * z, C2[2] * (2.0 * zz - xx - yy),
                 C2[3] * x * z, C2[4] * (xx - yy)]
    if degree >= 3:
        xx, yy, zz = x * x, y * y, z * z
        cols += [C3[0] * y * (3.0 * xx - yy), C3[1] * x * y * z,
                 C3[2] * y * (4.0 * zz - xx - yy), C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy),
                 C3[4] * x * (4.0 * zz - xx - yy), C3[5] * z * (xx - yy),
                 C3[6] * x * (xx - 3.0 * yy)]
    return np.stack(cols, axis=1)


def sh_basis_grad(degree: int, d: np.ndarray) -> np.ndarray:
    """sh.py:66-109 eval_basis_grad: (n, K, 3)."""
    n = len(d)
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    g = np.zeros((n, (degree + 1) ** 2, 3))
    if degree >= 1:
        g[:, 1, 1] = -C1
        g[:, 2, 2] = C1
        g[:, 3, 0] = -C1
    if degree >= 2:
        g[:, 4, 0], g[:, 4, 1] = C2[0] * y, C2[0] * x
        g[:, 5, 1], g[:, 5, 2] = C2[1] * z, C2[1] * y
        g[:, 6, 0], g[:, 6, 1], g[:, 6, 2] = C2[2] * (-2.0 * x), C2[2] * (-2.0 * y), C2[2] * (4.0 * z)
        g[:, 7, 0], g[:, 7, 2] = C2[3] * z, C2[3] * x
        g[:, 8, 0], g[:, 8, 1] = C2[4] * (2.0 * x), C2[4] * (-2.0 * y)
    if degree >= 3:
        xx, yy, zz = x * x, y * y, z * z
        g[:, 9, 0], g[:, 9, 1] = C3[0] * 6.0 * x * y, C3[0] * (3.0 * xx - 3.0 * yy)
        g[:, 10, 0], g[:, 10, 1], g[:, 10, 2] = C3[1] * y * z, C3[1] * x * z, C3[1] * x * y
        g[:, 11, 0] = C3[2] * (-2.0 * x * y)
        g[:, 11, 1] = C3[2] * (4.0 * zz - xx - 3.0 * yy)
        g[:, 11, 2] = C3[2] * (8.0 * y * z)
        g[:, 12, 0] = C3[3] * (-6.0 * x * z)
        g[:, 12, 1] = C3[3] * (-6.0 * y * z)
        g[:, 12, 2] = C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy)
        g[:, 13, 0] = C3[4] * (4.0 * zz - 3.0 * xx - yy)
        g[:, 13, 1] = C3[4] * (-2.0 * x * y)
        g[:, 13, 2] = C3[4] * (8.0 * x * z)
        g[:, 14, 0], g[:, 14, 1], g[:, 14, 2] = C3[5] * (2.0 * x * z), C3[5] * (-2.0 * y * z), C3[5] * (xx - yy)
        g[:, 15, 0], g[:, 15, 1] = C3[6] * (3.0 * xx - 3.0 * yy), C3[6] * (-6.0 * x * y)
    return g


def camera_points(means: np.ndarray, R: np.ndarray, t: np.ndarray) -> np.ndarray:
    """raster.py:137 mu_c = means @ R^T + t with the dgemm k=3 FMA order."""
    means, R, t = f64(means), f64(R), f64(t)
    out = np.empty_like(means)
    _clib.lib().oracle_camera_points(ptr(means), ptr(R), ptr(t), len(means), ptr(out))
    return out


def degree_of(shs) -> int:
    return int(np.sqrt(shs.shape[1])) - 1


def splat_geometry(P, R_cw, t_cw, cam, st):
    """raster.py:134-185 — projection, EWA covariance, footprint, bbox, conic."""
    mu_all = camera_points(P["means"], R_cw, t_cw)
    idx = np.flatnonzero(mu_all[:, 2] > st.near)
    mu_c = mu_all[idx]
    x, y, z = mu_c[:, 0], mu_c[:, 1], mu_c[:, 2]
    mu_i = np.column_stack([cam.fx * x / z + cam.cx, cam.fy * y / z + cam.cy])
    n = len(idx)
    J = np.zeros((n, 2, 3))
    J[:, 0, 0] = cam.fx / z
    J[:, 0, 2] = -cam.fx * x / z ** 2
    J[:, 1, 1] = cam.fy / z
    J[:, 1, 2] = -cam.fy * y / z ** 2
    B = P["rots"][idx] * P["scales"][idx][:, None, :]
    cov_w = np.matmul(B, np.swapaxes(B, 1, 2))
    M = np.matmul(J, R_cw)
    cov_i = np.matmul(np.matmul(M, cov_w), np.swapaxes(M, 1, 2))
    cov_i[:, 0, 0] += st.dilation
    cov_i[:, 1, 1] += st.dilation
    a, b, c = cov_i[:, 0, 0], cov_i[:, 0, 1], cov_i[:, 1, 1]
    det = a * c - b * b
    mid = 0.5 * (a + c)
    disc = np.sqrt(np.maximum(0.25 * (a - c) ** 2 + b * b, 0.0))
    nsig = np.full(n, float(st.footprint_sigma))
    if st.alpha_cut > 0.0:
        ratio = np.maximum(P["opacities"][idx] / st.alpha_cut, 1.0)
        nsig = np.minimum(nsig, np.sqrt(2.0 * np.log(ratio)))
    radius = nsig * np.sqrt(np.maximum(mid + disc, 0.0))
    x0 = np.maximum(np.floor(mu_i[:, 0] - radius), 0).astype(np.int64)
    x1 = np.minimum(np.floor(mu_i[:, 0] + radius) + 1, cam.width).astype(np.int64)
    y0 = np.maximum(np.floor(mu_i[:, 1] - radius), 0).astype(np.int64)
    y1 = np.minimum(np.floor(mu_i[:, 1] + radius) + 1, cam.height).astype(np.int64)
    keep = np.flatnonzero((x0 < x1) & (y0 < y1) & (radius <= st.max_footprint_px))
    det_k = det[keep]
    return {
        "ids": idx[keep], "mu_c": mu_c[keep], "mu_i": mu_i[keep], "J": J[keep],
        "cov_w": cov_w[keep], "cov_i": cov_i[keep],
        "conics": np.column_stack([c[keep] / det_k, -b[keep] / det_k, a[keep] / det_k]),
        "bboxes": np.column_stack([x0[keep], x1[keep], y0[keep], y1[keep]]),
        "radius": radius[keep],
    }


def eval_color(degree, shs, dirs):
    """sh.py:112-123 — clip(0.5 + sum b*sh) and the interior mask."""
    k = (degree + 1) ** 2
    raw = 0.5 + np.einsum("nk,nkc->nc", sh_basis(degree, dirs), shs[:, :k, :])
    return np.clip(raw, 0.0, 1.0), (raw > 0.0) & (raw < 1.0)


def render(P, R_cw, t_cw, cam, st):
    """raster.py:212-264 — global stable depth sort, SH colour, CSR composite.

    Returns the reference's cache dict plus image (H,W,3), t_final (H,W) and
    n_proc (H,W).
    """
    L = _clib.lib()
    h, w = cam.height, cam.width
    bg = f64(st.background)
    geo = splat_geometry(P, R_cw, t_cw, cam, st)
    order = np.argsort(geo["mu_c"][:, 2], kind="stable")
    cache = {k: np.ascontiguousarray(v[order]) for k, v in geo.items()}
    ids = cache["ids"]
    cache["opac"] = f64(P["opacities"][ids])
    degree = min(st.sh_degree, degree_of(P["shs"]))
    cam_center = -R_cw.T @ t_cw
    dvec = P["means"][ids] - cam_center
    dnorm = np.linalg.norm(dvec, axis=1)
    dirs = np.where(dnorm[:, None] > 0, dvec / np.maximum(dnorm, 1e-30)[:, None], [0.0, 0.0, 1.0])
    colors, interior = eval_color(degree, P["shs"][ids], dirs)
    colors = f64(colors)
    m = len(ids)
    bb = i64(cache["bboxes"])
    offsets = np.empty(h * w + 1, np.int64)
    splat_offsets = np.empty(m + 1, np.int64)
    total = L.oracle_csr_count(ptr(bb), m, h, w, ptr(offsets), ptr(splat_offsets))
    entry_splat = np.empty(total, np.int64)
    entry_pos = np.empty(total, np.int64)
    entry_pix = np.empty(total, np.int64)
    L.oracle_csr_fill(ptr(bb), m, h, w, ptr(offsets), ptr(entry_splat), ptr(entry_pos),
                      ptr(entry_pix))
    image = np.empty((h * w, 3))
    t_final = np.empty(h * w)
    n_proc = np.empty(h * w, np.int64)
    g_scr = np.empty(total)
    a_scr = np.empty(total)
    t_scr = np.empty(total)
    L.oracle_forward(ptr(offsets), ptr(entry_splat), ptr(cache["mu_i"]), ptr(cache["conics"]),
                     ptr(cache["opac"]), ptr(colors), ptr(bg), h, w, st.alpha_clamp,
                     st.transmittance_min, st.alpha_cut, ptr(image), ptr(t_final),
                     ptr(n_proc), ptr(g_scr), ptr(a_scr), ptr(t_scr))
    cache.update(
        P=P, R_cw=f64(R_cw), t_cw=f64(t_cw), cam=cam, st=st, degree=degree,
        colors=colors, interior=interior, dirs=dirs, dnorm=dnorm, bg=bg,
        offsets=offsets, entry_splat=entry_splat, splat_offsets=splat_offsets,
        entry_pos=entry_pos, entry_pix=entry_pix, t_final=t_final, n_proc=n_proc,
        g_scr=g_scr, a_scr=a_scr, t_scr=t_scr,
        image=image.reshape(h, w, 3),
    )
    return cache


def depth_image(cache) -> np.ndarray:
    """Blend-weighted camera depth sum_k a_k T_k z_k (no background term)."""
    cam = cache["cam"]
    e_s = cache["entry_splat"]
    contrib = cache["a_scr"] * cache["t_scr"] * cache["mu_c"][e_s, 2]
    pix = np.repeat(np.arange(cam.height * cam.width), np.diff(cache["offsets"]))
    return np.bincount(pix, weights=contrib, minlength=cam.height * cam.width).reshape(
        cam.height, cam.width)


def _screen_grads(cache, g_img, sel):
    L = _clib.lib()
    cam = cache["cam"]
    h, w = cam.height, cam.width
    total = len(cache["entry_splat"])
    d_alpha = np.empty(total)
    w_out = np.empty(total)
    L.oracle_backward_entries(ptr(cache["offsets"]), ptr(cache["entry_splat"]),
                              ptr(cache["n_proc"]), ptr(cache["t_final"]), ptr(g_img),
                              ptr(cache["colors"]), ptr(cache["bg"]), ptr(cache["a_scr"]),
                              ptr(cache["t_scr"]), h, w, ptr(sel), ptr(d_alpha), ptr(w_out))
    return d_alpha, w_out


def hat(v):
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def imu_camera_adjoint(R_cw, R_ic, t_ic):
    """geometry.py:202-228: (rho_l, tau_l) = A (rho_r, tau_r)."""
    R_ci = R_ic.T
    t_ci = -R_ci @ t_ic
    A = np.zeros((6, 6))
    A[:3, :3] = -R_ci
    A[3:, :3] = -hat(t_ci) @ R_ci
    A[3:, 3:] = -R_cw
    return A


def _vee_diff(X):
    return np.stack([X[..., 2, 1] - X[..., 1, 2], X[..., 0, 2] - X[..., 2, 0],
                     X[..., 1, 0] - X[..., 0, 1]], axis=-1)


def backward(cache, grad_image, R_ic=None, t_ic=None):
    """raster.py:309-399 — gradients for every group and the pose."""
    L = _clib.lib()
    cam, st, P = cache["cam"], cache["st"], cache["P"]
    h, w = cam.height, cam.width
    R_ic = np.eye(3) if R_ic is None else f64(R_ic)
    t_ic = np.zeros(3) if t_ic is None else f64(t_ic)
    g_img = f64(np.asarray(grad_image, dtype=np.float64).reshape(h * w, 3))
    sel = np.ones(h * w, np.uint8)
    d_alpha, w_out = _screen_grads(cache, g_img, sel)
    m = len(cache["ids"])
    d_color = np.empty((m, 3))
    d_opac = np.empty(m)
    d_mu2 = np.empty((m, 2))
    d_cov2 = np.empty((m, 3))
    L.oracle_accumulate(ptr(cache["splat_offsets"]), m, ptr(cache["entry_pos"]),
                        ptr(cache["entry_pix"]), ptr(d_alpha), ptr(w_out), ptr(cache["g_scr"]),
                        ptr(cache["a_scr"]), ptr(g_img), ptr(cache["mu_i"]),
                        ptr(cache["conics"]), ptr(cache["opac"]), w, st.alpha_clamp,
                        ptr(d_color), ptr(d_opac), ptr(d_mu2), ptr(d_cov2))
    out = chain(cache, d_color, d_opac, d_mu2, d_cov2, R_ic, t_ic)
    out["screen"] = dict(d_color=d_color, d_opac=d_opac, d_mu2=d_mu2, d_cov2=d_cov2)
    return out


def chain(cache, d_color, d_opac, d_mu2, d_cov2, R_ic, t_ic):
    """raster.py:337-399 — screen -> camera -> world chain, pose gradient."""
    P, cam = cache["P"], cache["cam"]
    R = cache["R_cw"]
    ids = cache["ids"]
    J, mu_c, cov_w = cache["J"], cache["mu_c"], cache["cov_w"]
    rots, scales = P["rots"][ids], P["scales"][ids]
    d_col = d_color * cache["interior"]
    # 2D covariance chain (raster.py:286-298)
    M = np.matmul(J, R)
    S = np.empty((len(ids), 2, 2))
    S[:, 0, 0], S[:, 0, 1], S[:, 1, 0], S[:, 1, 1] = d_cov2[:, 0], d_cov2[:, 1], d_cov2[:, 1], d_cov2[:, 2]
    Mt = np.swapaxes(M, 1, 2)
    d_cov_w = np.matmul(np.matmul(Mt, S), M)
    d_M = 2.0 * np.matmul(np.matmul(S, M), cov_w)
    d_J = np.matmul(d_M, R.T)
    d_W = np.matmul(np.swapaxes(J, 1, 2), d_M)
    # mean chain (raster.py:267-283, 347-350)
    d_mu_c = np.einsum("nji,nj->ni", J, d_mu2)
    x, y, z = mu_c[:, 0], mu_c[:, 1], mu_c[:, 2]
    gx, gy = -cam.fx / z ** 2, -cam.fy / z ** 2
    d_mu_c[:, 0] += d_J[:, 0, 2] * gx
    d_mu_c[:, 1] += d_J[:, 1, 2] * gy
    d_mu_c[:, 2] += (d_J[:, 0, 0] * gx + d_J[:, 1, 1] * gy
                     + d_J[:, 0, 2] * (2.0 * cam.fx * x / z ** 3)
                     + d_J[:, 1, 2] * (2.0 * cam.fy * y / z ** 3))
    d_mean = d_mu_c @ R
    # covariance -> rotation tangent and scale (raster.py:352-358)
    B = rots * scales[:, None, :]
    d_B = 2.0 * np.matmul(d_cov_w, B)
    Y = np.matmul(np.swapaxes(rots, 1, 2), d_B * scales[:, None, :])
    d_rot = _vee_diff(Y)
    d_scale = np.einsum("nij,nij->nj", rots, d_B)
    # appearance (raster.py:360-373)
    degree = cache["degree"]
    k = (degree + 1) ** 2
    d_sh = np.einsum("nk,nc->nkc", sh_basis(degree, cache["dirs"]), d_col)
    d_cam_center = np.zeros(3)
    if degree >= 1:
        gb = sh_basis_grad(degree, cache["dirs"])
        d_dir = np.einsum("nc,nkc,nkd->nd", d_col, P["shs"][ids][:, :k, :], gb)
        dirs = cache["dirs"]
        proj = d_dir - dirs * np.sum(dirs * d_dir, axis=1, keepdims=True)
        d_point = proj / np.maximum(cache["dnorm"], 1e-30)[:, None]
        d_mean = d_mean + d_point
        d_cam_center = -d_point.sum(axis=0)
    # pose, camera tangent then IMU tangent (raster.py:375-383)
    rho_cam = np.cross(mu_c, d_mu_c).sum(axis=0) + _vee_diff(np.matmul(d_W, R.T)).sum(axis=0)
    tau_cam = d_mu_c.sum(axis=0) - R @ d_cam_center
    A = imu_camera_adjoint(R, R_ic, t_ic)
    imu = A.T @ np.concatenate([rho_cam, tau_cam])
    n = len(P["means"])
    grads = {
        "mean": np.zeros((n, 3)), "rot": np.zeros((n, 3)), "scale": np.zeros((n, 3)),
        "opacity": np.zeros(n), "sh": np.zeros_like(P["shs"]),
    }
    grads["mean"][ids] = d_mean
    grads["rot"][ids] = d_rot
    grads["scale"][ids] = d_scale
    grads["opacity"][ids] = d_opac
    grads["sh"][ids, :k, :] = d_sh
    pose = {"rho": imu[:3], "tau": imu[3:], "camera_rho": rho_cam, "camera_tau": tau_cam}
    return {"grads": grads, "pose": pose}


def pose_chain_matrices(cache):
    """raster.py:402-447 — per-splat L_mu (6,2) and L_sig (6,3)."""
    mu_c, J, R, cam = cache["mu_c"], cache["J"], cache["R_cw"], cache["cam"]
    m = len(mu_c)
    L_mu = np.zeros((m, 6, 2))
    for i in range(2):
        L_mu[:, :3, i] = np.cross(mu_c, J[:, i, :])
        L_mu[:, 3:, i] = J[:, i, :]
    E = np.zeros((3, 2, 2))
    E[0, 0, 0] = 1.0
    E[1, 0, 1] = E[1, 1, 0] = 1.0
    E[2, 1, 1] = 1.0
    M = np.matmul(J, R)
    MC = np.matmul(M, cache["cov_w"])                       # (m,2,3)
    d_M = 2.0 * np.einsum("bij,njl->nbil", E, MC)           # (m,3,2,3)
    d_J = np.einsum("nbij,kj->nbik", d_M, R)
    d_W = np.einsum("nji,nbjk->nbik", J, d_M)
    x, y, z = mu_c[:, 0], mu_c[:, 1], mu_c[:, 2]
    gx = (-cam.fx / z ** 2)[:, None]
    gy = (-cam.fy / z ** 2)[:, None]
    dmu = np.zeros((m, 3, 3))
    dmu[:, :, 0] = d_J[:, :, 0, 2] * gx
    dmu[:, :, 1] = d_J[:, :, 1, 2] * gy
    dmu[:, :, 2] = (d_J[:, :, 0, 0] * gx + d_J[:, :, 1, 1] * gy
                    + d_J[:, :, 0, 2] * (2.0 * cam.fx * x / z ** 3)[:, None]
                    + d_J[:, :, 1, 2] * (2.0 * cam.fy * y / z ** 3)[:, None])
    Z = np.einsum("nbij,kj->nbik", d_W, R)
    L_sig = np.zeros((m, 6, 3))
    L_sig[:, :3, :] = (np.cross(mu_c[:, None, :], dmu) + _vee_diff(Z)).swapaxes(1, 2)
    L_sig[:, 3:, :] = dmu.swapaxes(1, 2)
    return L_mu, L_sig


def pose_rows(cache, pixel_ids, R_ic=None, t_ic=None):
    """raster.py:450-508 — d gray(I_hat(u)) / d xi_IMU for selected pixels."""
    L = _clib.lib()
    cam, st = cache["cam"], cache["st"]
    h, w = cam.height, cam.width
    npx = h * w
    R_ic = np.eye(3) if R_ic is None else f64(R_ic)
    t_ic = np.zeros(3) if t_ic is None else f64(t_ic)
    pixel_ids = i64(pixel_ids)
    g_img = np.full((npx, 3), 1.0 / 3.0)
    sel = np.zeros(npx, np.uint8)
    sel[pixel_ids] = 1
    d_alpha, w_out = _screen_grads(cache, g_img, sel)
    total = len(cache["entry_splat"])
    keep = np.empty(total, np.uint8)
    e_s = np.empty(total, np.int64)
    e_p = np.empty(total, np.int64)
    e_mu = np.empty((total, 2))
    e_cov = np.empty((total, 3))
    e_w = np.empty(total)
    L.oracle_screen_grads(total, ptr(cache["entry_pos"]), ptr(cache["entry_pix"]),
                          ptr(cache["entry_splat"]), ptr(d_alpha), ptr(w_out),
                          ptr(cache["g_scr"]), ptr(cache["a_scr"]), ptr(cache["mu_i"]),
                          ptr(cache["conics"]), ptr(cache["opac"]), w, st.alpha_clamp,
                          ptr(sel), ptr(keep), ptr(e_s), ptr(e_p), ptr(e_mu), ptr(e_cov),
                          ptr(e_w))
    kk = keep.astype(bool)
    e_s, e_p, e_mu, e_cov, e_w = e_s[kk], e_p[kk], e_mu[kk], e_cov[kk], e_w[kk]
    L_mu, L_sig = pose_chain_matrices(cache)
    contrib = np.einsum("eij,ej->ei", L_mu[e_s], e_mu) + np.einsum("eik,ek->ei", L_sig[e_s], e_cov)
    if cache["degree"] >= 1:
        k = (cache["degree"] + 1) ** 2
        gb = sh_basis_grad(cache["degree"], cache["dirs"])
        Pm = np.einsum("nkc,nkd->ncd", cache["P"]["shs"][cache["ids"]][:, :k, :], gb)
        dirs = cache["dirs"][e_s]
        dc = (e_w / 3.0)[:, None] * cache["interior"][e_s]
        d_dir = np.einsum("ec,ecd->ed", dc, Pm[e_s])
        proj = d_dir - dirs * np.sum(dirs * d_dir, axis=1, keepdims=True)
        d_point = proj / np.maximum(cache["dnorm"], 1e-30)[e_s][:, None]
        contrib[:, 3:] += d_point @ cache["R_cw"].T
    contrib_imu = contrib @ imu_camera_adjoint(cache["R_cw"], R_ic, t_ic)
    row_of = np.full(npx, -1, np.int64)
    row_of[pixel_ids] = np.arange(len(pixel_ids))
    rows = np.zeros((len(pixel_ids), 6))
    np.add.at(rows, row_of[e_p], contrib_imu)
    return rows


def tile_lists(cache, tile: int = 16):
    """CPU restatement of the B200 tile binning (no reference counterpart:
    SURVEY.md §0 fact 1).  For each 16x16 tile, the splats (as indices into the
    depth-sorted cache order) whose bbox intersects the tile, in global depth
    order.  Returns (ranges (ntiles, 2) int64, entries (I,) int64 sorted-splat
    index, gaussian ids (I,))."""
    cam = cache["cam"]
    tx_n = (cam.width + tile - 1) // tile
    ty_n = (cam.height + tile - 1) // tile
    bb = cache["bboxes"]
    tx0, tx1 = bb[:, 0] // tile, (bb[:, 1] - 1) // tile
    ty0, ty1 = bb[:, 2] // tile, (bb[:, 3] - 1) // tile
    cnt = (tx1 - tx0 + 1) * (ty1 - ty0 + 1)
    rank = np.repeat(np.arange(len(bb)), cnt)
    tiles = np.empty(cnt.sum(), np.int64)
    pos = 0
    for s in range(len(bb)):
        ys, xs = np.meshgrid(np.arange(ty0[s], ty1[s] + 1), np.arange(tx0[s], tx1[s] + 1),
                             indexing="ij")
        t = (ys * tx_n + xs).ravel()
        tiles[pos:pos + len(t)] = t
        pos += len(t)
    order = np.argsort(tiles, kind="stable")   # stable: keeps global depth order
    tiles_sorted = tiles[order]
    entries = rank[order]
    starts = np.searchsorted(tiles_sorted, np.arange(tx_n * ty_n), side="left")
    ends = np.searchsorted(tiles_sorted, np.arange(tx_n * ty_n), side="right")
    return np.column_stack([starts, ends]), entries, cache["ids"][entries]


def contributing_tile_rows(cache, tile: int = 16):
    """CPU restatement of the bin_mode-1 tile sets (csrc/preprocess.cu
    cull_row_cols; no reference counterpart).  A pair (pixel, splat) is
    composited by _kernels.py:104 only if q = d^T cov_i^-1 d <= 2 ln(op/cut);
    per tile row the tiles whose rows can reach that ellipse (threshold with
    the kernel's margin x1.001 + 0.01) form one column interval, clipped to the
    bbox.  Returns a list per sorted splat of (ty, tx0, tx1) rows."""
    st = cache["st"]
    assert st.alpha_cut > 0.0
    mu, cov, bb, op = cache["mu_i"], cache["cov_i"], cache["bboxes"], cache["opac"]
    out = []
    for s in range(len(bb)):
        x0, x1, y0, y1 = (int(v) for v in bb[s])
        mux, muy = float(mu[s, 0]), float(mu[s, 1])
        ca, cb, cc = float(cov[s, 0, 0]), float(cov[s, 0, 1]), float(cov[s, 1, 1])
        thr = 2.0 * np.log(max(float(op[s]) / st.alpha_cut, 1.0)) * 1.001 + 0.01
        rows = []
        for ty in range(y0 // tile, (y1 - 1) // tile + 1):
            ya, yb = max(ty * tile, y0), min(ty * tile + tile - 1, y1 - 1)
            hy = np.sqrt(thr * cc)
            da, db = max(ya - muy, -hy), min(yb - muy, hy)
            if not da <= db:
                continue
            det = ca * cc - cb * cb
            k, w2 = cb / cc, det / cc
            dyr = cb * np.sqrt(thr / ca)
            dr, dl = min(max(dyr, da), db), min(max(-dyr, da), db)
            xr = k * dr + np.sqrt(max(w2 * (thr - dr * dr / cc), 0.0))
            xl = k * dl - np.sqrt(max(w2 * (thr - dl * dl / cc), 0.0))
            c0, c1 = max(x0, int(np.ceil(mux + xl))), min(x1 - 1, int(np.floor(mux + xr)))
            if c0 <= c1:
                rows.append((ty, c0 // tile, c1 // tile))
        out.append(rows)
    return out


def contributing_tile_lists(cache, tile: int = 16):
    """tile_lists() for bin_mode 1: the same (ranges, entries, ids) triple
    over the contributing tile sets of contributing_tile_rows()."""
    cam = cache["cam"]
    tx_n = (cam.width + tile - 1) // tile
    ty_n = (cam.height + tile - 1) // tile
    rows = contributing_tile_rows(cache, tile)
    tiles, rank = [], []
    for s, rs in enumerate(rows):
        for ty, a, b in rs:
            t = ty * tx_n + np.arange(a, b + 1)
            tiles.append(t)
            rank.append(np.full(len(t), s, np.int64))
    tiles = np.concatenate(tiles) if tiles else np.zeros(0, np.int64)
    rank = np.concatenate(rank) if rank else np.zeros(0, np.int64)
    order = np.argsort(tiles, kind="stable")
    tiles_sorted = tiles[order]
    entries = rank[order]
    starts = np.searchsorted(tiles_sorted, np.arange(tx_n * ty_n), side="left")
    ends = np.searchsorted(tiles_sorted, np.arange(tx_n * ty_n), side="right")
    return np.column_stack([starts, ends]), entries, cache["ids"][entries]
