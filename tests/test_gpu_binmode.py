"""bin_mode 1 (contributing tile lists) on the GPU, through the C ABI.

Mode 1 drops (tile, splat) entries whose alpha >= alpha_cut ellipse misses
the tile.  Bars: the tile lists equal the oracle's restatement bit for bit
(oracle.raster.contributing_tile_lists); image, T, depth, parameter gradients
and pose are BIT-IDENTICAL to mode 0 (the dropped entries only ever added
exact zeros) on the golden cases and on a full-size config-2 view.
"""
import numpy as np
import pytest

from golden_io import case_inputs, load

pytestmark = pytest.mark.gpu

CUT_CASES = [f"rand{s}_cut1" for s in range(4)] + ["odd_cut1", "room_v0_cut1", "room_v2_cut1"]


def _settings(st):
    from paper_2501_08672_b200.raster import RasterSettings
    return RasterSettings(near=st.near, dilation=st.dilation, alpha_clamp=st.alpha_clamp,
                          transmittance_min=st.transmittance_min, footprint_sigma=st.footprint_sigma,
                          alpha_cut=st.alpha_cut, max_footprint_px=st.max_footprint_px,
                          background=tuple(np.asarray(st.background).tolist()), sh_degree=st.sh_degree)


def _both(arrays, T_wc, cam, settings):
    from paper_2501_08672_b200.raster import render
    return [render(arrays, T_wc, cam, settings, with_depth=True, bin_mode=m) for m in (0, 1)]


def _assert_identical(o0, o1, grad_image, T_ic=None):
    import torch
    from paper_2501_08672_b200.raster import backward
    assert torch.equal(o0.image, o1.image)
    assert torch.equal(o0.final_transmittance, o1.final_transmittance)
    assert torch.equal(o0.depth, o1.depth)
    g0, p0 = backward(o0, grad_image, T_ic=T_ic)
    g1, p1 = backward(o1, grad_image, T_ic=T_ic)
    assert torch.equal(g0.flat, g1.flat)
    assert np.array_equal(p0.as_vector(), p1.as_vector())


@pytest.mark.parametrize("name", CUT_CASES)
def test_binmode1_lists_and_outputs(name):
    from oracle import raster as orc
    from paper_2501_08672_b200.geometry import SE3
    from paper_2501_08672_b200.raster import GaussianArrays
    d = load(name)
    P, R_cw, t_cw, cam, st = case_inputs(d)
    arrays = GaussianArrays(P["means"], P["rots"], P["scales"], P["opacities"], P["shs"])
    o0, o1 = _both(arrays, SE3(d["R_wc"], d["t_wc"]), cam, _settings(st))
    ranges, _, gid = orc.contributing_tile_lists(orc.render(P, R_cw, t_cw, cam, st))
    s = o1.cache
    assert s.counts[1] == len(gid) <= o0.cache.counts[1]
    assert np.array_equal(s.export(2), ranges)
    assert np.array_equal(s.export(3), gid)
    _assert_identical(o0, o1, d["grad_image"], T_ic=SE3(d["R_ic"], d["t_ic"]))


def test_binmode1_fullsize_cfg2_view():
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings
    from tools.scene import bake_room, camera_for, orbit_views
    arrays = GaussianArrays(*bake_room(0.0723))
    cam = camera_for(1280, 1024)
    T = orbit_views(10)[3]
    o0, o1 = _both(arrays, T, cam, RasterSettings(alpha_cut=1.0 / 255.0))
    assert o1.cache.counts[1] < 0.9 * o0.cache.counts[1]
    rng = np.random.default_rng(5)
    _assert_identical(o0, o1, rng.normal(size=(1024, 1280, 3)).astype(np.float32))


@pytest.mark.parametrize("bin_mode", [0, 1])
@pytest.mark.parametrize("name", ["rand1_cut1", "room_v0_cut1", "room_v1_cut0"])
def test_countfree_forward_identical(name, bin_mode):
    """The window engine's count-free forward (n_contrib NULL, half-tile skip)
    writes the same image / T bits as the counting forward."""
    import torch
    from paper_2501_08672_b200.raster import GaussianArrays, RenderState, render_bin, render_blend
    d = load(name)
    P, R_cw, t_cw, cam, st = case_inputs(d)
    arrays = GaussianArrays(P["means"], P["rots"], P["scales"], P["opacities"], P["shs"])
    state = RenderState(arrays, cam, R_cw, t_cw, _settings(st), 1 << 20, bin_mode)
    render_bin(state)
    h, w = cam.height, cam.width
    outs = []
    for count in (True, False):
        img = torch.empty((h, w, 3), dtype=torch.float32, device="cuda")
        tf = torch.empty((h, w), dtype=torch.float32, device="cuda")
        nc = torch.empty((h, w), dtype=torch.int32, device="cuda") if count else None
        render_blend(state, img, tf, nc)
        outs.append((img, tf))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
