"""GPU parity of the visual IESKF measurement (semi-dense selection, residual
gate, pose rows, H/b reduction) against the reference (estimator.py:241-323)."""
import numpy as np
import pytest

from golden_io import load

pytestmark = pytest.mark.gpu


def _setup():
    from paper_2501_08672_b200.geometry import PinholeCamera, SE3
    from paper_2501_08672_b200.raster import GaussianArrays
    from tools.scene import T_IC
    d = load("visual_room")
    s = load("scene_room_0323")
    arrays = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], s["shs"])
    fx, fy, cx, cy, w, h = d["cam"]
    return d, arrays, PinholeCamera(fx, fy, cx, cy, int(w), int(h)), SE3(d["R_wi"], d["t_wi"]), T_IC


def test_visual_measurement_matches_reference():
    from paper_2501_08672_b200.estimator import FilterConfig, NavState, visual_measurement
    from paper_2501_08672_b200.raster import RasterSettings
    d, arrays, cam, T_wi, T_ic = _setup()
    meas = visual_measurement(NavState(T_wi), d["observed"], arrays, cam, T_ic, FilterConfig(),
                              RasterSettings(alpha_cut=1 / 255))
    assert len(meas.z) == len(d["z"])
    assert np.abs(meas.z - d["z"]).max() <= 1e-4
    ref = d["H"][:, :6]
    assert np.abs(meas.H[:, :6] - ref).max() / np.abs(ref).max() <= 1e-3
    assert np.all(meas.R_diag == d["R_diag"])
    A, b = meas.hb()
    Ri = 1.0 / d["R_diag"][0]
    A_ref = ref.T @ ref * Ri
    b_ref = ref.T @ d["z"] * Ri
    assert np.abs(A - A_ref).max() / np.abs(A_ref).max() <= 1e-3
    assert np.abs(b - b_ref).max() / np.abs(b_ref).max() <= 1e-3


def test_semidense_selection_matches_reference():
    from paper_2501_08672_b200.estimator import FilterConfig, select_semi_dense_pixels
    from paper_2501_08672_b200.raster import RasterSettings, render
    d, arrays, cam, T_wi, T_ic = _setup()
    out = render(arrays, T_wi @ T_ic, cam, RasterSettings(alpha_cut=1 / 255))
    ids = select_semi_dense_pixels(d["observed"], out.final_transmittance, FilterConfig())
    assert np.array_equal(ids, d["sel_ids"])


def test_too_few_pixels_raises():
    from paper_2501_08672_b200.errors import TooFewPixels
    from paper_2501_08672_b200.estimator import FilterConfig, NavState, visual_measurement
    from paper_2501_08672_b200.raster import RasterSettings
    d, arrays, cam, T_wi, T_ic = _setup()
    with pytest.raises(TooFewPixels):
        visual_measurement(NavState(T_wi), np.zeros_like(d["observed"]), arrays, cam, T_ic,
                           FilterConfig(min_pixels=10 ** 6), RasterSettings(alpha_cut=1 / 255))


def test_ieskf_visual_update_matches_reference():
    """Three IESKF iterations with the photometric measurement: posterior pose
    and covariance vs the reference's ieskf_update (estimator.py:292-331)."""
    from paper_2501_08672_b200.estimator import FilterConfig, NavState, ieskf_visual_update
    from paper_2501_08672_b200.raster import RasterSettings
    d, arrays, cam, T_wi, T_ic = _setup()
    post, cov = ieskf_visual_update(NavState(T_wi), d["cov0"], d["observed"], arrays, cam, T_ic, FilterConfig(),
                                    RasterSettings(alpha_cut=1 / 255), max_iter=3)
    assert np.abs(post.T_WI.t - d["post_t"]).max() <= 1e-4
    assert np.abs(post.T_WI.R - d["post_R"]).max() <= 1e-4
    assert np.abs(cov - d["post_cov"]).max() <= 1e-3 * np.abs(d["post_cov"]).max()


@pytest.mark.parametrize("budget,gate", [(1, 0.15), (2, 0.15), (7, 0.15), (300, 0.02), (1024, 0.15), (10 ** 6, 0.15)])
def test_device_selection_budget_and_gate(budget, gate):
    """The on-device selection (lsb_visual_select) against the reference's
    steps restated in numpy on the same mask and render: linspace subsample
    at every budget regime (1, tiny, below and above the candidate count),
    grey residual, ordered gate (estimator.py:241-277)."""
    import torch

    from paper_2501_08672_b200.estimator import FilterConfig, NavState, select_semi_dense_pixels, visual_measurement
    from paper_2501_08672_b200.raster import RasterSettings, render
    d, arrays, cam, T_wi, T_ic = _setup()
    st = RasterSettings(alpha_cut=1 / 255)
    cfg = FilterConfig(pixel_budget=budget, photo_gate=gate, min_pixels=1)
    out = render(arrays, T_wi @ T_ic, cam, st, bin_mode=1)
    ids = select_semi_dense_pixels(d["observed"], out.final_transmittance, cfg)
    obs = np.asarray(d["observed"], np.float32).astype(np.float64).reshape(-1, 3)
    img = out.image.cpu().numpy().astype(np.float64).reshape(-1, 3)
    res = obs[ids].mean(axis=1) - img[ids].mean(axis=1)
    res = res[np.abs(res) <= gate]
    if len(res) < cfg.min_pixels:
        from paper_2501_08672_b200.errors import TooFewPixels
        with pytest.raises(TooFewPixels):
            visual_measurement(NavState(T_wi), d["observed"], arrays, cam, T_ic, cfg, st)
        return
    meas = visual_measurement(NavState(T_wi), d["observed"], arrays, cam, T_ic, cfg, st)
    torch.cuda.synchronize()
    assert np.array_equal(meas.z, res)


def test_single_sync_pass_bit_identical_to_measurement():
    """The IESKF iteration's one-sync device pass (_VisualPass: the kept count
    stays on the device for the pose rows and H/b) gives the same bits as
    visual_measurement(...).hb(), and raises TooFewPixels the same way."""
    from paper_2501_08672_b200.errors import TooFewPixels
    from paper_2501_08672_b200.estimator import FilterConfig, NavState, _VisualPass, visual_measurement
    from paper_2501_08672_b200.raster import RasterSettings
    d, arrays, cam, T_wi, T_ic = _setup()
    st = RasterSettings(alpha_cut=1 / 255)
    for budget in (1024, 64):
        cfg = FilterConfig(pixel_budget=budget, min_pixels=10)
        A, b = visual_measurement(NavState(T_wi), d["observed"], arrays, cam, T_ic, cfg, st).hb()
        vis = _VisualPass(arrays, d["observed"], cam, cfg, st)
        for _ in range(2):                       # buffers reused across iterations
            A2, b2 = vis.run(NavState(T_wi), T_ic)
            assert np.array_equal(A, A2) and np.array_equal(b, b2)
    with pytest.raises(TooFewPixels):
        _VisualPass(arrays, np.zeros_like(d["observed"]), cam, FilterConfig(min_pixels=10 ** 6), st).run(
            NavState(T_wi), T_ic)


def test_u8_frames_selection_and_residuals():
    """8-bit observed frames through the visual measurement: the selection
    and the residuals equal the reference's steps (estimator.py:241-277,
    scipy's Sobel as the reference calls it) on read_ppm's u / 255.0."""
    import torch
    from scipy import ndimage

    from paper_2501_08672_b200.estimator import FilterConfig, NavState, visual_measurement
    from paper_2501_08672_b200.raster import RasterSettings, render
    d, arrays, cam, T_wi, T_ic = _setup()
    st = RasterSettings(alpha_cut=1 / 255)
    cfg = FilterConfig(min_pixels=10)
    obs8 = np.clip(np.round(np.asarray(d["observed"], np.float64) * 255.0), 0, 255).astype(np.uint8)
    obs = obs8.astype(np.float64) / 255.0
    out = render(arrays, T_wi @ T_ic, cam, st, bin_mode=1)
    gray = obs.mean(axis=2)
    mag = np.hypot(ndimage.sobel(gray, axis=1, mode="nearest") / 8.0, ndimage.sobel(gray, axis=0, mode="nearest") / 8.0)
    T = out.final_transmittance.cpu().numpy()
    ids = np.flatnonzero((mag > cfg.grad_threshold) & (T < cfg.coverage_max_transmittance))
    if len(ids) > cfg.pixel_budget:
        ids = ids[np.unique(np.round(np.linspace(0, len(ids) - 1, cfg.pixel_budget)).astype(int))]
    img = out.image.cpu().numpy().astype(np.float64).reshape(-1, 3)
    res = gray.reshape(-1)[ids] - img[ids].mean(axis=1)
    res = res[np.abs(res) <= cfg.photo_gate]
    meas = visual_measurement(NavState(T_wi), obs8, arrays, cam, T_ic, cfg, st)
    torch.cuda.synchronize()
    assert np.array_equal(meas.z, res)
