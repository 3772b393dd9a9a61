"""Golden fixture for the reference's per-frame call sequence
(`Pipeline.process_frame`, pipeline.py:147-219), produced by the REFERENCE
(livsplat, read-only at /root/reference/pkg/src) in this container.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_pipeline.py

Scenario: the reference's own `simulate` defaults (cli.py:109-140: the
builtin room, the orbit trajectory, the default Config: 128x108 camera,
72x24 spinning LiDAR, root 0.06 m, max_level 2), exported with
`sim.export_dataset`, read back with `dataset.DatasetReader` and replayed by
`pipeline.Pipeline` for FRAMES frames (initialised at the ground-truth pose,
as pipeline.run does).

IMU propagation (imu_propagate) is outside the hot path, so
the fixture records its output per frame -- the prior (state, covariance)
each frame's updates start from -- and the test feeds it in.  Recorded per
frame: the inputs (8-bit frame bytes as read_ppm decodes them, LiDAR points),
the prior, the posterior after the LiDAR update and after the visual update
(+ applied flags), the mapping results (new Gaussians, window report), the
optimisation loss history, the final render's PSNR and the window's live
keys.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from livsplat import pipeline as pl  # noqa: E402
from livsplat.config import Config  # noqa: E402
from livsplat.dataset import DatasetReader  # noqa: E402
from livsplat.geometry import SE3, PinholeCamera  # noqa: E402
from livsplat.sim import ScanPattern, TrajectorySpec, default_room, export_dataset  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "pipeline.npz")
FRAMES = 6


def pack(s) -> np.ndarray:
    return np.concatenate([s.T_WI.R.ravel(), s.T_WI.t, s.velocity, s.bias_gyro, s.bias_accel]).astype(np.float64)


def main() -> None:
    cfg = Config()
    sim = cfg.sim
    cam = PinholeCamera(sim.fx, sim.fy, sim.cx, sim.cy, sim.width, sim.height)
    T_ic = SE3(np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]]), [0.05, 0.0, 0.0])
    T_li = SE3(np.eye(3), [0.03, 0.0, 0.05])
    # cli.py:90-95 (the builtin orbit)
    times = np.linspace(0.0, 12.0, 13)
    ang = np.linspace(0, 1.5 * np.pi, 13)
    pos = np.column_stack([1.0 * np.cos(ang), 1.0 * np.sin(ang), np.full(13, 1.0)])
    traj = TrajectorySpec(times, pos, ang + np.pi / 2, imu_rate=sim.imu_rate, frame_rate=sim.frame_rate)
    tmp = tempfile.mkdtemp(prefix="lsb_pipe_")
    export_dataset(tmp, default_room(), traj, cam, T_li, T_ic,
                   pattern=ScanPattern(n_azimuth=sim.lidar_azimuth, n_elevation=sim.lidar_elevation,
                                       azimuth_span=sim.lidar_azimuth_span,
                                       elevation_span=sim.lidar_elevation_span),
                   v_s=cfg.map.root_len, max_level=cfg.map.max_level, kappa=cfg.init.kappa,
                   delta=cfg.init.delta, opacity=cfg.init.opacity, seed=0, settings=cfg.raster_settings())
    reader = DatasetReader(tmp)
    pipe = pl.Pipeline(cfg, reader.calib)
    stamps, poses = reader.ground_truth()
    pipe.initialize_pose(poses[0])

    rec: dict = {}
    orig_prop, orig_upd = pl.imu_propagate, pl.ieskf_update

    def prop(state, cov, *a, **k):
        s, c = orig_prop(state, cov, *a, **k)
        rec["prior"] = (pack(s), c.copy())
        return s, c

    def upd(state, cov, meas_fn, **k):
        s, c = orig_upd(state, cov, meas_fn, **k)
        rec.setdefault("updates", []).append((pack(s), c.copy()))
        return s, c

    orig_vis = pl.visual_measurement

    def vis_meas(*a, **k):
        m = orig_vis(*a, **k)
        if "vis_first" not in rec:       # the first linearisation of the frame (at the post-LiDAR state)
            A = m.H.T @ (m.H / m.R_diag[:, None])
            b = m.H.T @ (m.z / m.R_diag)
            rec["vis_first"] = (len(m.z), A[:6, :6].copy(), b[:6].copy())
        return m

    pl.imu_propagate, pl.ieskf_update, pl.visual_measurement = prop, upd, vis_meas
    out = {k: [] for k in ("image", "points", "prior_x", "prior_P", "lidar_x", "lidar_P", "visual_x", "visual_P",
                           "flags", "report", "loss", "psnr", "live_keys", "n_gauss", "vis_n", "vis_A", "vis_b",
                           "rows")}
    try:
        for i, frame in enumerate(reader.frames()):
            if i == FRAMES:
                break
            rec.clear()
            rec["prior"] = (pack(pipe.state), pipe.cov.copy())     # frame 0: no propagation
            r = pipe.process_frame(frame)
            prior = rec["prior"]                                      # imu_propagate's output
            ups = rec.get("updates", [])
            # the updates that ran in order: LiDAR (if it did not raise), visual
            it = iter(ups)
            lid = next(it) if r.lidar_applied else (prior[0], prior[1])
            vis = next(it) if r.visual_applied else lid
            out["image"].append(np.round(frame.image * 255.0).astype(np.uint8))
            assert np.array_equal(out["image"][-1].astype(np.float64) / 255.0, frame.image)
            out["points"].append(np.asarray(frame.points_l, np.float64))
            out["prior_x"].append(prior[0]); out["prior_P"].append(prior[1])
            out["lidar_x"].append(lid[0]); out["lidar_P"].append(lid[1])
            out["visual_x"].append(vis[0]); out["visual_P"].append(vis[1])
            out["flags"].append([r.lidar_applied, r.visual_applied])
            out["report"].append([r.new_gaussians, r.n_live, r.added, r.removed, r.moved])
            hist = [h[2] for h in pipe.loss_history if h[0] == i]
            out["loss"].append(np.asarray(hist, np.float64))
            out["psnr"].append(r.psnr)
            w = pipe.window
            keys = [(k.ix, k.iy, k.iz, k.level) for k in w.key_of_slot[:w.n]]    # slot order
            out["live_keys"].append(np.asarray(keys, np.int64).reshape(-1, 4))
            out["n_gauss"].append(pipe.vmap.gaussian_count())
            vn, vA, vb = rec.get("vis_first", (0, np.zeros((6, 6)), np.zeros(6)))
            out["vis_n"].append(vn); out["vis_A"].append(vA); out["vis_b"].append(vb)
            a = w.device
            n = w.n
            out["rows"].append(np.concatenate([a.means[:n], a.rots[:n].reshape(n, 9), a.scales[:n],
                                               a.opacities[:n, None], a.shs[:n].reshape(n, -1)], axis=1))
            print(f"frame {i}: lidar {r.lidar_applied} visual {r.visual_applied} new {r.new_gaussians} "
                  f"live {r.n_live} loss {r.loss:.5f} psnr {r.psnr:.2f}")
    finally:
        pl.imu_propagate, pl.ieskf_update, pl.visual_measurement = orig_prop, orig_upd, orig_vis
    n = len(out["image"])
    np.savez_compressed(
        OUT, frames=n, cam=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height], np.float64),
        R_ic=reader.calib.T_ic.R, t_ic=reader.calib.T_ic.t, R_li=reader.calib.T_li.R, t_li=reader.calib.T_li.t,
        image=np.stack(out["image"]),
        **{f"points_{i}": out["points"][i] for i in range(n)},
        **{f"loss_{i}": out["loss"][i] for i in range(n)},
        **{f"live_keys_{i}": out["live_keys"][i] for i in range(n)},
        **{f"rows_{i}": out["rows"][i] for i in range(n)},
        **{k: np.asarray(out[k]) for k in ("prior_x", "prior_P", "lidar_x", "lidar_P", "visual_x", "visual_P",
                                             "flags", "report", "psnr", "n_gauss", "vis_n", "vis_A",
                                             "vis_b")})
    print("wrote", OUT)


if __name__ == "__main__":
    main()
