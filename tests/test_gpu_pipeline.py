"""The reference's per-frame call sequence driven through this package's names
(`Pipeline.process_frame`, pipeline.py:147-219), against the reference's own
replay of the same frames (tests/golden/pipeline.npz, generator
tools/make_golden_pipeline.py: the `simulate` defaults, 6 frames).

`process_frame` below is the reference's body with every livsplat name bound
to this package: the LiDAR IESKF update (lidar_measurement), the photometric
update (visual_measurement), leaf grouping and statistics
(HashOctree.group_by_leaf / ensure_leaf / add_leaf_stats), Gaussian creation
(the reference's per-leaf `_insert_new_gaussians` loop is
initialize.insert_new_gaussians, one batched call), the FoV
(keys_of_points, leaf_keys_under_roots), window maintenance, optimize_window
and the final render + photometric_loss.  IMU propagation is out of scope
(SURVEY.md §2.1): each frame starts from the prior the reference propagated.

Checked per frame: the applied flags, new-Gaussian count, window report, map
size and live keys in slot order exactly; the visual update's selected
pixel count exactly and its first H/b within 1e-3 relative; the posterior
states within 1e-6 (pose, velocity, biases) and covariances within 1e-3
relative; the window rows after optimisation, the loss history and the
final PSNR within 1e-3 relative."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _unpack(x):
    from paper_2501_08672_b200.estimator import NavState
    from paper_2501_08672_b200.geometry import SE3
    return NavState(SE3(x[:9].reshape(3, 3).copy(), x[9:12].copy()), x[12:15].copy(), x[15:18].copy(),
                    x[18:21].copy())


def _pack(s):
    return np.concatenate([s.T_WI.R.ravel(), s.T_WI.t, s.velocity, s.bias_gyro, s.bias_accel])


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-30)


class _Frame:
    def __init__(self, image, points_l):
        self.image, self.points_l = image, points_l


class _Pipeline:
    """pipeline.Pipeline's mapping state and process_frame body
    (pipeline.py:67-90, 147-219) on this package's names."""

    def __init__(self, cam, T_ic, T_li):
        from paper_2501_08672_b200.estimator import FilterConfig
        from paper_2501_08672_b200.optimize import OptimConfig
        from paper_2501_08672_b200.raster import RasterSettings
        from paper_2501_08672_b200.voxmap import HashOctree
        from paper_2501_08672_b200.window import GaussianWindow
        # config.py defaults: MapConfig(0.06, 2, 1), InitConfig(0.8, 1e-3, 0.9, 0), WindowConfig(100_000)
        self.root_len, self.max_level, self.leaf_capacity = 0.06, 2, 1
        self.kappa, self.delta, self.opacity = 0.8, 1e-3, 0.9
        self.settings = RasterSettings(alpha_cut=0.00392156862745098)
        self.fcfg, self.optim = FilterConfig(), OptimConfig()
        self.vmap = HashOctree(self.root_len, self.max_level, self.leaf_capacity)
        self.window = GaussianWindow(capacity=100_000, sh_coeffs=1)
        self.cam, self.T_ic, self.T_li = cam, T_ic, T_li

    def process_frame(self, frame, state, cov):
        from paper_2501_08672_b200.errors import NoAssociations, SingularGain, TooFewPixels
        from paper_2501_08672_b200.estimator import ieskf_update, lidar_measurement, visual_measurement
        from paper_2501_08672_b200.initialize import insert_new_gaussians
        from paper_2501_08672_b200.optimize import optimize_window, photometric_loss
        from paper_2501_08672_b200.raster import render
        from paper_2501_08672_b200.voxmap import keys_of_points
        fcfg, rec = self.fcfg, {"lidar": 0, "visual": 0}
        plane_cache: dict = {}
        try:
            state, cov = ieskf_update(
                state, cov,
                lambda s: lidar_measurement(s, frame.points_l, self.vmap, self.T_li, fcfg, plane_cache),
                max_iter=fcfg.max_iter, step_tol=fcfg.step_tol, bias_limit=fcfg.bias_limit)
            rec["lidar"] = 1
        except (NoAssociations, SingularGain):
            pass
        rec["lidar_x"], rec["lidar_P"] = _pack(state), cov.copy()
        rec["vis_n"], rec["vis_hb"] = 0, None
        if self.window.n > 0:
            try:        # the update's first linearisation (checked against the reference's)
                m = visual_measurement(state, frame.image, self.window, self.cam, self.T_ic, fcfg, self.settings)
                rec["vis_n"], rec["vis_hb"] = len(m), m.hb()
            except TooFewPixels:
                pass
            try:
                state, cov = ieskf_update(
                    state, cov,
                    lambda s: visual_measurement(s, frame.image, self.window, self.cam, self.T_ic, fcfg,
                                                 self.settings),
                    max_iter=fcfg.visual_max_iter, step_tol=fcfg.step_tol, bias_limit=fcfg.bias_limit)
                rec["visual"] = 1
            except (TooFewPixels, SingularGain):
                pass
        rec["visual_x"], rec["visual_P"] = _pack(state), cov.copy()

        T_wl = state.T_WI @ self.T_li
        p_w = T_wl.apply(frame.points_l)
        groups = self.vmap.group_by_leaf(p_w)
        for key, pts in groups.items():
            self.vmap.ensure_leaf(key)
            self.vmap.add_leaf_stats(key, pts)
        T_wc = state.T_WI @ self.T_ic
        _, _, made = insert_new_gaussians(self.vmap, p_w, frame.image, T_wc, self.cam, T_wl.t, kappa=self.kappa,
                                          delta=self.delta, opacity=self.opacity, sh_coeffs=1,
                                          near=self.settings.near, accumulate=False)
        rec["new"] = int(made.sum().item())
        fov_roots = set(keys_of_points(p_w, self.vmap.root_len, 0))
        fov_keys = self.vmap.leaf_keys_under_roots(fov_roots)
        report = self.window.maintain(self.vmap, fov_keys, sensor_pos=T_wl.t)
        rec["report"] = [rec["new"], report.n_live, report.added, report.removed, report.moved]
        history = optimize_window(self.window, frame.image, T_wc, self.cam, self.optim, self.settings)
        rec["loss"] = np.array([h.value for h in history])
        out = render(self.window, T_wc, self.cam, self.settings, retain_cache=False)
        rep, _ = photometric_loss(out.image, frame.image)
        rec["psnr"] = float(10.0 * np.log10(1.0 / rep.mse)) if rep.mse > 0 else float("inf")
        return state, cov, rec


def test_process_frame_sequence_matches_reference_replay():
    from golden_io import load
    from paper_2501_08672_b200.geometry import PinholeCamera, SE3
    d = load("pipeline")
    fx, fy, cx, cy, w, h = d["cam"]
    cam = PinholeCamera(fx, fy, cx, cy, int(w), int(h))
    pipe = _Pipeline(cam, SE3(d["R_ic"], d["t_ic"]), SE3(d["R_li"], d["t_li"]))
    for i in range(int(d["frames"])):
        # the frame as DatasetReader hands it over: read_ppm's u / 255.0 in f64
        frame = _Frame(d["image"][i].astype(np.float64) / 255.0, d[f"points_{i}"])
        _, _, rec = pipe.process_frame(frame, _unpack(d["prior_x"][i]), d["prior_P"][i].copy())
        assert [rec["lidar"], rec["visual"]] == list(d["flags"][i]), i
        # the visual update's first linearisation: same selected pixels, H/b within 1e-3
        assert rec["vis_n"] == int(d["vis_n"][i]), (i, rec["vis_n"], int(d["vis_n"][i]))
        if rec["vis_hb"] is not None:
            A, b = rec["vis_hb"]
            assert rel(A, d["vis_A"][i]) <= 1e-3 and rel(b, d["vis_b"][i]) <= 1e-3, (i, rel(A, d["vis_A"][i]),
                                                                                       rel(b, d["vis_b"][i]))
        for stage in ("lidar", "visual"):
            x, xr = rec[f"{stage}_x"], d[f"{stage}_x"][i]
            assert np.abs(x[:12] - xr[:12]).max() <= 1e-6, (i, stage, np.abs(x[:12] - xr[:12]).max())
            assert np.abs(x[12:] - xr[12:]).max() <= 1e-6, (i, stage)
            assert rel(rec[f"{stage}_P"], d[f"{stage}_P"][i]) <= 1e-3, (i, stage)
        assert rec["report"] == list(d["report"][i]), (i, rec["report"], list(d["report"][i]))
        live = pipe.window.live_keys_dev().cpu().numpy().reshape(-1, 3)      # slot order
        assert np.array_equal(live, d[f"live_keys_{i}"][:, :3]), i
        assert pipe.vmap.gaussian_count() == int(d["n_gauss"][i]), i
        # the window's rows after optimize_window (10 Adam iterations), in slot order
        rows = pipe.window.rows_dev().cpu().numpy().astype(np.float64)
        assert rel(rows, d[f"rows_{i}"]) <= 1e-3, (i, rel(rows, d[f"rows_{i}"]))
        assert rel(rec["loss"], d[f"loss_{i}"]) <= 1e-3, (i, rec["loss"], d[f"loss_{i}"])
        assert abs(rec["psnr"] - float(d["psnr"][i])) <= 1e-3 * abs(float(d["psnr"][i])), i
