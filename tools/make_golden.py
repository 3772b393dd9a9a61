"""Generate golden fixtures by running the REFERENCE (livsplat, read-only at
/root/reference/pkg/src) in this container.  The outputs are committed under
tests/golden/ so the GPU box (which has no /root/reference) can check parity.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py

All Gaussian parameters are rounded to f32 before the reference sees them
(the sliding-window arena stores f32, window.py:51-55, and upcasts for the
render, window.py:111-120), so the CUDA path and the reference consume the
identical values.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from livsplat import sh as shmod  # noqa: E402
from livsplat import sim  # noqa: E402
from livsplat.estimator import FilterConfig, NavState, select_semi_dense_pixels, visual_measurement  # noqa: E402
from livsplat.geometry import PinholeCamera, SE3, so3_exp  # noqa: E402
from livsplat.optimize import AdamState, OptimConfig, optimize_window, photometric_loss  # noqa: E402
from livsplat.raster import GaussianArrays, RasterSettings, backward, pose_rows, render  # noqa: E402
from livsplat.voxmap import HashOctree, hash_key, keys_of_points, leaf_key  # noqa: E402
from livsplat.window import GaussianWindow  # noqa: E402
from livsplat.geometry import Gaussian3D  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
CAM32 = PinholeCamera(fx=40.0, fy=40.0, cx=16.0, cy=16.0, width=32, height=32)
T_IC = SE3(np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]]), [0.05, 0.0, 0.0])


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def random_scene(rng, n, spread=1.0, z_range=(2.0, 6.0), sh_degree=0):
    """Same generator as the reference tests (test_raster.py:22-45), rounded to f32."""
    k = (sh_degree + 1) ** 2
    means = np.column_stack([rng.uniform(-spread, spread, n), rng.uniform(-spread, spread, n),
                             rng.uniform(*z_range, n)])
    rots = np.stack([so3_exp(rng.normal(size=3)) for _ in range(n)])
    scales = np.column_stack([rng.uniform(0.002, 0.01, n), rng.uniform(0.05, 0.4, n),
                              rng.uniform(0.05, 0.4, n)])
    opac = rng.uniform(0.3, 0.9, n)
    shs = np.zeros((n, k, 3))
    shs[:, 0, :] = (rng.uniform(0.1, 0.9, (n, 3)) - 0.5) / shmod.SH_C0
    if k > 1:
        shs[:, 1:, :] = rng.uniform(-0.05, 0.05, (n, k - 1, 3))
    return GaussianArrays(f32(means), f32(rots), f32(scales), f32(opac), f32(shs))


def settings_dict(s: RasterSettings):
    return dict(near=s.near, dilation=s.dilation, alpha_clamp=s.alpha_clamp,
                transmittance_min=s.transmittance_min, footprint_sigma=s.footprint_sigma,
                alpha_cut=s.alpha_cut, max_footprint_px=s.max_footprint_px,
                background=np.asarray(s.background, dtype=float), sh_degree=s.sh_degree)


def dump_render_case(name, arrays, T_wc, cam, settings, T_ic, rng, pix_ids=None):
    out = render(arrays, T_wc, cam, settings)
    c = out.cache
    target = rng.uniform(0, 1, size=(cam.height, cam.width, 3))
    _, grad_img = photometric_loss(out.image, target)
    grads, pose = backward(out, grad_img, T_ic=T_ic)
    if pix_ids is None:
        pix_ids = rng.choice(cam.width * cam.height, size=min(64, cam.width * cam.height),
                             replace=False)
    rows = pose_rows(out, pix_ids, T_ic=T_ic)
    sd = settings_dict(settings)
    np.savez_compressed(
        os.path.join(OUT, name + ".npz"),
        means=arrays.means, rots=arrays.rots, scales=arrays.scales,
        opacities=arrays.opacities, shs=arrays.shs,
        R_wc=T_wc.R, t_wc=T_wc.t, R_ic=T_ic.R, t_ic=T_ic.t,
        cam=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height], dtype=float),
        **{"st_" + k: np.asarray(v) for k, v in sd.items()},
        image=out.image, t_final=out.final_transmittance, n_proc=out.contrib_count,
        ids=c["ids"], bboxes=c["bboxes"], mu_c=c["mu_c"], mu_i=c["mu_i"], conics=c["conics"],
        colors=c["colors"], interior=c["interior"], offsets=c["offsets"],
        entry_splat=c["entry_splat"].astype(np.int32),
        target=target, grad_image=grad_img,
        g_mean=grads.mean, g_rot=grads.rot, g_scale=grads.scale, g_opacity=grads.opacity,
        g_sh=grads.sh, p_rho=pose.rho, p_tau=pose.tau, p_crho=pose.camera_rho,
        p_ctau=pose.camera_tau, pix_ids=np.asarray(pix_ids), pose_rows=rows,
    )
    print(name, "M=", len(c["ids"]), "E=", len(c["entry_splat"]))


def room_scene(v_s, sh_degree=0):
    _, _, gts = sim.bake_scene(sim.default_room(4.0), v_s, max_level=2, kappa=0.8, delta=1e-3,
                               opacity=0.9, sh_degree=sh_degree)
    a = GaussianArrays.from_gaussians(gts)
    return GaussianArrays(f32(a.means), f32(a.rots), f32(a.scales), f32(a.opacities), f32(a.shs))


def orbit_pose(a):
    R = np.array([[np.cos(a + np.pi / 2), -np.sin(a + np.pi / 2), 0.0],
                  [np.sin(a + np.pi / 2), np.cos(a + np.pi / 2), 0.0], [0.0, 0.0, 1.0]])
    return SE3(R, [np.cos(a), np.sin(a), 1.0])


def main():
    os.makedirs(OUT, exist_ok=True)
    # 1. random scenes, reference test scale (CAM32)
    for seed in range(4):
        rng = np.random.default_rng(1000 + seed)
        deg = [0, 0, 1, 3][seed]
        arrays = random_scene(rng, int(rng.integers(8, 50)), sh_degree=deg)
        T_ic = SE3(so3_exp(rng.normal(size=3) * 0.3), rng.normal(size=3) * 0.2) if seed % 2 else SE3.identity()
        T_wi = SE3(so3_exp(rng.normal(size=3) * 0.02), rng.normal(size=3) * 0.02)
        if seed == 0:
            T_wi, T_ic = SE3.identity(), SE3.identity()
        for cut in (0.0, 1.0 / 255.0):
            st = RasterSettings(background=(0.15, 0.25, 0.35), alpha_cut=cut, sh_degree=deg)
            dump_render_case(f"rand{seed}_cut{int(cut > 0)}", arrays, T_wi @ T_ic, CAM32, st, T_ic,
                             np.random.default_rng(seed))
    # 1b. odd image size (partial edge tiles), more Gaussians, non-identity pose
    cam_odd = PinholeCamera(fx=50.0, fy=48.0, cx=22.5, cy=14.0, width=45, height=29)
    for cut in (0.0, 1.0 / 255.0):
        rng = np.random.default_rng(77)
        arrays = random_scene(rng, 120, spread=1.5)
        T_ic = SE3(so3_exp(rng.normal(size=3) * 0.3), rng.normal(size=3) * 0.2)
        T_wi = SE3(so3_exp(rng.normal(size=3) * 0.05), rng.normal(size=3) * 0.05)
        st = RasterSettings(background=(0.05, 0.1, 0.2), alpha_cut=cut)
        dump_render_case(f"odd_cut{int(cut > 0)}", arrays, T_wi @ T_ic, cam_odd, st, T_ic, np.random.default_rng(5))
    # 2. the synthetic room (config-1 scene), reduced resolution, orbit views
    arrays = room_scene(0.323)
    np.savez_compressed(os.path.join(OUT, "scene_room_0323.npz"), means=arrays.means,
                        rots=arrays.rots, scales=arrays.scales, opacities=arrays.opacities,
                        shs=arrays.shs)
    W, H = 160, 128
    cam = PinholeCamera(0.9375 * W, 0.9375 * W, W / 2, H / 2, W, H)
    yaws = np.linspace(0, 1.5 * np.pi, 4)
    for vi, cut in ((0, 1.0 / 255.0), (1, 0.0), (2, 1.0 / 255.0)):
        T_wc = orbit_pose(yaws[vi]) @ T_IC
        st = RasterSettings(alpha_cut=cut)
        dump_render_case(f"room_v{vi}_cut{int(cut > 0)}", arrays, T_wc, cam, st, T_IC,
                         np.random.default_rng(10 + vi))
    # 3. Adam update, and optimize_window on a small plane window (test_optimize.py:71-88)
    cfg = OptimConfig()
    rng = np.random.default_rng(7)
    adam = AdamState({"x": (50, 3)}, cfg)
    g_seq = rng.normal(size=(3, 50, 3)) * np.array([1e-3, 1.0, 1e3])[None, None, :]
    g_seq[:, :5] = 0.0
    steps = []
    for g in g_seq:
        adam.step += 1
        steps.append(adam.update("x", g, 1e-3))
    np.savez_compressed(os.path.join(OUT, "adam.npz"), grads=g_seq, steps=np.stack(steps))

    def plane_window(perturb):
        vmap = HashOctree(root_len=0.4, max_level=1, leaf_capacity=1)
        r = np.random.default_rng(42)
        from livsplat.initialize import init_rotation
        rot = init_rotation([0.0, 0.0, -1.0])
        for i in range(6):
            for j in range(6):
                p = np.array([(i - 2.5) * 0.2, (j - 2.5) * 0.2, 2.0])
                color = np.array([0.3 + 0.4 * (i % 2), 0.35 + 0.3 * (j % 2), 0.55])
                co = np.zeros((1, 3))
                co[0] = shmod.color_from_target(color + perturb * r.uniform(-1, 1, 3))
                vmap.try_insert(Gaussian3D(mean_w=p, rot=rot, scale=[1e-3, 0.12, 0.12],
                                           opacity=0.9, sh=co))
        keys = {k for k, node in vmap.iter_leaves() if node.gaussians}
        win = GaussianWindow(capacity=1000)
        win.maintain(vmap, keys)
        return win

    CAM48 = PinholeCamera(fx=60.0, fy=60.0, cx=24.0, cy=24.0, width=48, height=48)
    st = RasterSettings(background=(0.0, 0.0, 0.0))
    clean = plane_window(0.0)
    observed = render(clean, SE3.identity(), CAM48, st).image
    win = plane_window(0.2)
    n = win.n
    before = {k: getattr(win.device, k)[:n].copy() for k in ("means", "rots", "scales", "opacities", "shs")}
    hist = optimize_window(win, observed, SE3.identity(), CAM48, cfg, st)
    np.savez_compressed(
        os.path.join(OUT, "optimize_plane.npz"), observed=observed,
        **{"in_" + k: v for k, v in before.items()},
        **{"out_" + k: getattr(win.device, k)[:n].copy() for k in before},
        loss=np.array([h.value for h in hist]), mse=np.array([h.mse for h in hist]),
        cam=np.array([60.0, 60.0, 24.0, 24.0, 48, 48], dtype=float))
    # 4. voxel keys, grouping, octree FoV and iteration order
    rng = np.random.default_rng(11)
    pts = np.concatenate([rng.uniform(-3, 3, size=(4000, 3)),
                          rng.normal(scale=0.05, size=(1000, 3)) + 0.3,
                          np.array([[0.0, 0.0, 0.0], [-0.1, 0.2, -0.06], [0.13, 0.0, -0.05]])])
    root_len, max_level = 0.4, 3
    m = HashOctree(root_len, max_level)
    groups = m.group_by_leaf(pts)
    gkeys = np.array([tuple(k) for k in groups.keys()], dtype=np.int64)
    gcount = np.array([len(v) for v in groups.values()])
    gsum = np.stack([v.sum(axis=0) for v in groups.values()])
    m.accumulate_points(pts)
    for p in rng.uniform(-2, 2, size=(600, 3)):
        co = np.zeros((1, 3))
        m.try_insert(Gaussian3D(mean_w=p, rot=np.eye(3), scale=[1e-3, 0.1, 0.1], opacity=0.9, sh=co))
    iter_keys = np.array([tuple(k) for k, _ in m.iter_leaves()], dtype=np.int64)
    iter_has_g = np.array([bool(node.gaussians) for _, node in m.iter_leaves()])
    fov_pts = rng.uniform(-1.5, 1.5, size=(300, 3))
    roots = set(keys_of_points(fov_pts, root_len, 0))
    fov = sorted(m.leaf_keys_under_roots(roots))
    stats = [m.leaf_stats[tuple_k] for tuple_k in sorted(m.leaf_stats.keys())]
    np.savez_compressed(
        os.path.join(OUT, "voxmap.npz"), pts=pts, root_len=root_len, max_level=max_level,
        root_keys=np.array([tuple(hash_key(p, root_len)) for p in pts], dtype=np.int64),
        leaf_keys=np.array([tuple(leaf_key(p, root_len, max_level)) for p in pts], dtype=np.int64),
        group_keys=gkeys, group_count=gcount, group_sum=gsum,
        stat_keys=np.array([tuple(k) for k in sorted(m.leaf_stats.keys())], dtype=np.int64),
        stat_count=np.array([s[0] for s in stats]), stat_sum=np.stack([s[1] for s in stats]),
        stat_outer=np.stack([s[2] for s in stats]),
        insert_pts=np.random.default_rng(11).uniform(size=1),  # marker only
        iter_keys=iter_keys, iter_has_g=iter_has_g, fov_pts=fov_pts,
        fov_roots=np.array(sorted(tuple(r) for r in roots), dtype=np.int64),
        fov_keys=np.array([tuple(k) for k in fov], dtype=np.int64),
        hash_vals=np.array([hash(k) for k in keys_of_points(pts[:50], root_len, 0)], dtype=np.int64),
    )
    # 5. visual measurement on the room (semi-dense selection, gate, rows)
    arrays = room_scene(0.323)
    win = GaussianWindow(capacity=len(arrays.means))

    class _Src:
        def as_gaussian_arrays(self):
            return arrays
    W, H = 160, 128
    cam = PinholeCamera(0.9375 * W, 0.9375 * W, W / 2, H / 2, W, H)
    T_wi = orbit_pose(yaws[1])
    observed = render(arrays, T_wi @ T_IC, cam, RasterSettings(alpha_cut=1 / 255)).image
    prior = NavState(T_WI=SE3(T_wi.R @ so3_exp([0.002, -0.001, 0.003]), T_wi.t + np.array([0.01, -0.005, 0.004])))
    fcfg = FilterConfig()
    meas = visual_measurement(prior, observed, _Src(), cam, T_IC, fcfg, RasterSettings(alpha_cut=1 / 255))
    out = render(arrays, prior.T_WI @ T_IC, cam, RasterSettings(alpha_cut=1 / 255))
    ids = select_semi_dense_pixels(observed, out.final_transmittance, fcfg)
    from livsplat.estimator import ieskf_update, initial_covariance
    cov0 = initial_covariance()
    post, cov_post = ieskf_update(prior, cov0, lambda s: visual_measurement(
        s, observed, _Src(), cam, T_IC, fcfg, RasterSettings(alpha_cut=1 / 255)), max_iter=3)
    np.savez_compressed(os.path.join(OUT, "visual_room.npz"), observed=observed,
                        cov0=cov0, post_R=post.T_WI.R, post_t=post.T_WI.t, post_cov=cov_post,
                        R_wi=prior.T_WI.R, t_wi=prior.T_WI.t, sel_ids=ids, z=meas.z, H=meas.H,
                        R_diag=meas.R_diag, cam=np.array([cam.fx, cam.fy, cam.cx, cam.cy, W, H], dtype=float))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
