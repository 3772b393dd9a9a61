"""The reference entry points of SURVEY.md §8(b) that sit beside the render:
raster.splat (raster.py:188-205), the HashOctree's group_by_leaf /
add_leaf_stats / fov_leaf_keys / iter_leaves / voxel_center
(voxmap.py:54,187,204,213,339), the window's gaussian_at / writeback_deleted /
compact (window.py:106,145,152) and the generic ieskf_update
(estimator.py:292-331) - each against the reference's own arithmetic
restated in numpy, or against this package's batched path."""
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _st(cut=0.0, deg=0):
    return SimpleNamespace(near=0.01, dilation=0.3, alpha_clamp=0.99, transmittance_min=1e-4, footprint_sigma=6.0,
                           alpha_cut=cut, max_footprint_px=512.0, background=np.zeros(3), sh_degree=deg)


@pytest.mark.parametrize("cut", [0.0, 1 / 255])
def test_splat_matches_reference_geometry(cut):
    from oracle import raster as orc
    from paper_2501_08672_b200.geometry import SE3, Gaussian2D, Gaussian3D, so3_exp
    from paper_2501_08672_b200.raster import Culled, RasterSettings, splat
    rng = np.random.default_rng(5)
    cam = SimpleNamespace(fx=110.0, fy=105.0, cx=64.0, cy=48.0, width=128, height=96)
    T_cw = SE3(so3_exp([0.05, -0.02, 0.01]), [0.1, -0.05, 0.2])
    st = _st(cut, 1)
    settings = RasterSettings(alpha_cut=cut, sh_degree=1)
    seen = culled = 0
    for i in range(60):
        g = Gaussian3D(mean_w=[rng.uniform(-3, 3), rng.uniform(-2, 2), rng.uniform(-1, 6)],
                       rot=so3_exp(rng.normal(size=3)), scale=np.exp(rng.uniform(-5, -1, 3)),
                       opacity=float(rng.uniform(0.001, 1.0)), sh=rng.uniform(-1, 1, (4, 3)))
        P = {"means": g.mean_w[None], "rots": g.rot[None], "scales": g.scale[None],
             "opacities": np.array([g.opacity]), "shs": g.sh[None]}
        geo = orc.splat_geometry(P, T_cw.R, T_cw.t, cam, st)
        out = splat(g, T_cw, cam, settings)
        if len(geo["ids"]) == 0:
            assert isinstance(out, Culled)
            culled += 1
            continue
        seen += 1
        assert isinstance(out, Gaussian2D)
        assert np.array_equal(out.mean_i, geo["mu_i"][0])
        assert np.abs(out.cov_i - geo["cov_i"][0]).max() <= 1e-12 * np.abs(geo["cov_i"][0]).max()
        assert out.depth == geo["mu_c"][0, 2]
        c = T_cw.inverse().t
        d = g.mean_w - c
        col, _ = orc.eval_color(1, g.sh[None], (d / np.linalg.norm(d))[None])
        assert np.abs(out.color - col[0]).max() <= 1e-12
        assert out.opacity == g.opacity
    assert seen > 10 and culled > 5


def _map_and_points():
    from paper_2501_08672_b200.voxmap import HashOctree
    rng = np.random.default_rng(11)
    pts = np.concatenate([rng.uniform(-3, 3, size=(4000, 3)), rng.normal(scale=0.05, size=(1000, 3))])
    return HashOctree(0.5, max_level=2), pts


def test_group_by_leaf_is_the_reference_lexsort_grouping():
    m, pts = _map_and_points()
    groups = m.group_by_leaf(pts)
    idx = np.floor(pts / m.leaf_len).astype(np.int64)               # voxmap.py:218-229
    order = np.lexsort((idx[:, 2], idx[:, 1], idx[:, 0]))
    sidx, spts = idx[order], pts[order]
    cuts = np.nonzero(np.any(np.diff(sidx, axis=0) != 0, axis=1))[0] + 1
    ref = [((int(ci[0, 0]), int(ci[0, 1]), int(ci[0, 2])), cp) for ci, cp in zip(np.split(sidx, cuts),
                                                                               np.split(spts, cuts))]
    assert [k[:3] for k in groups] == [k for k, _ in ref]
    for (k, gp), (_, rp) in zip(groups.items(), ref):
        assert k.level == m.max_level and np.array_equal(gp, rp)
    assert m.group_by_leaf(np.zeros((0, 3))) == {}


def test_add_leaf_stats_and_fov_leaf_keys():
    from paper_2501_08672_b200.voxmap import VoxelKey, keys_of_points, voxel_center
    m, pts = _map_and_points()
    groups = m.group_by_leaf(pts)
    for key, gp in groups.items():                                  # pipeline.py:182-185
        m.ensure_leaf(key)
        m.add_leaf_stats(key, gp)
    for key, gp in list(groups.items())[::3]:
        n, s, o = m.leaf_stats(key)
        assert n == len(gp)
        assert np.array_equal(s, gp.sum(axis=0))                    # the reference's own sums, bit for bit
        assert np.array_equal(o, gp.T @ gp)
        c = voxel_center(key, m.root_len)
        assert np.array_equal(c, (np.array(key[:3], float) + 0.5) * (m.root_len / (1 << key.level)))
    assert m.fov_leaf_keys(pts) == set(keys_of_points(pts, m.leaf_len, m.max_level))
    assert isinstance(next(iter(m.fov_leaf_keys(pts))), VoxelKey)


def test_iter_leaves_order_and_payload():
    from paper_2501_08672_b200.geometry import Gaussian3D
    m, pts = _map_and_points()
    m.accumulate_points(pts)
    rng = np.random.default_rng(3)
    gs = [Gaussian3D(p, np.eye(3), [0.01, 0.02, 0.02], 0.5, rng.uniform(-1, 1, (1, 3))) for p in pts[::50]]
    for g in gs:
        m.try_insert(g)
    leaves = list(m.iter_leaves())
    assert [k for k, _ in leaves] == m.iter_leaf_keys()
    with_g = [(k, leaf) for k, leaf in leaves if leaf.gaussians]
    assert len(with_g) == m.gaussian_count()
    for k, leaf in with_g:
        assert leaf.is_leaf and len(leaf.gaussians) == 1
        assert tuple(np.floor(leaf.gaussians[0].mean_w / m.leaf_len).astype(int)) == k[:3]


def test_window_gaussian_at_writeback_deleted_compact():
    """diff -> writeback_deleted -> compact (window.py:136-181), the
    reference's step-by-step protocol, leaves the same window and map as the
    batched writeback_and_compact, on the reference's own window walk."""
    import torch
    from window_case import case
    from paper_2501_08672_b200.voxmap import HashOctree
    from paper_2501_08672_b200.window import GaussianWindow
    d, frames = case()
    K, L, root = int(d["sh_coeffs"]), int(d["max_level"]), float(d["root_len"])
    vmaps, wins = [], []
    for _ in range(2):
        vm = HashOctree(root, max_level=L)
        vm.set_gaussians_dev(d["seeded"], d["seed_rows"])
        w = GaussianWindow(capacity=int(d["capacity"]), sh_coeffs=K)
        w.maintain(vm, torch.as_tensor(frames[0]["fov"], device="cuda"), sensor_pos=frames[0]["sensor"])
        vmaps.append(vm)
        wins.append(w)
    fov1 = torch.as_tensor(frames[1]["fov"], device="cuda")
    diff = wins[0].diff(fov1)
    assert diff.delete                                           # the walk's frame 1 drops leaves
    wins[0].writeback_deleted(vmaps[0], diff)
    moved = wins[0].compact()
    wins[1].diff(fov1)
    _, moved1 = wins[1].writeback_and_compact(vmaps[1])
    assert moved == moved1 and wins[0].n == wins[1].n
    assert bool((wins[0].rows_dev() == wins[1].rows_dev()).all())
    assert bool((vmaps[0].store == vmaps[1].store).all())
    assert wins[0].compact() == 0                                 # nothing pending
    keys = wins[0].live_keys_dev().cpu().numpy()
    rows = wins[0].rows_dev().double().cpu().numpy()
    for slot in (0, len(keys) // 2, len(keys) - 1):
        g = wins[0].gaussian_at((*keys[slot], L))
        assert np.array_equal(g.mean_w, rows[slot, :3]) and np.array_equal(g.rot.ravel(), rows[slot, 3:12])
        assert np.array_equal(g.sh.ravel(), rows[slot, 16:])
    with pytest.raises(KeyError):
        wins[0].gaussian_at((10 ** 5, 0, 0, L))


def test_generic_ieskf_update_equals_the_visual_update():
    """ieskf_update(state, cov, lambda s: visual_measurement(...)) - the
    reference's generic call (pipeline.py:164-172) - gives the one-call
    visual update's posterior."""
    from golden_io import load
    from paper_2501_08672_b200.estimator import (FilterConfig, NavState, ieskf_update, ieskf_visual_update,
                                                 visual_measurement)
    from paper_2501_08672_b200.geometry import PinholeCamera, SE3
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings
    from tools.scene import T_IC
    d = load("visual_room")
    s = load("scene_room_0323")
    arrays = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], s["shs"])
    fx, fy, cx, cy, w, h = d["cam"]
    cam = PinholeCamera(fx, fy, cx, cy, int(w), int(h))
    st = RasterSettings(alpha_cut=1 / 255)
    cfg = FilterConfig()
    prior = NavState(SE3(d["R_wi"], d["t_wi"]))
    p1, c1 = ieskf_update(prior, d["cov0"], lambda x: visual_measurement(x, d["observed"], arrays, cam, T_IC, cfg, st),
                          max_iter=3)
    p2, c2 = ieskf_visual_update(prior, d["cov0"], d["observed"], arrays, cam, T_IC, cfg, st, max_iter=3)
    assert np.array_equal(p1.T_WI.R, p2.T_WI.R) and np.array_equal(p1.T_WI.t, p2.T_WI.t)
    assert np.array_equal(c1, c2)
    assert np.abs(p1.T_WI.t - d["post_t"]).max() <= 1e-4


def test_render_outputs_are_numpy_readable():
    """The reference's consumers of a render (write_ppm raster.py:511-517,
    metrics.psnr metrics.py:12-22) call np.asarray on the image."""
    from golden_io import case_inputs, load
    from paper_2501_08672_b200.geometry import SE3
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
    d = load("room_v0_cut1")
    P, _, _, cam, st = case_inputs(d)
    out = render(GaussianArrays(P["means"], P["rots"], P["scales"], P["opacities"], P["shs"]),
                 SE3(d["R_wc"], d["t_wc"]), cam, RasterSettings(alpha_cut=float(st.alpha_cut)))
    img = np.asarray(out.image, dtype=float)
    assert img.shape == (cam.height, cam.width, 3)
    assert np.array_equal(img, out.image.cpu().numpy().astype(np.float64))
    assert np.array_equal(np.asarray(out.final_transmittance), out.final_transmittance.cpu().numpy())
    img8 = np.clip(np.round(np.asarray(out.image) * 255.0), 0, 255).astype(np.uint8)
    assert img8.shape == img.shape
    assert np.abs(img - np.asarray(d["image"])).max() <= 1e-4
