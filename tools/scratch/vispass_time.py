"""Device vs wall time of one visual IESKF iteration (timing aid)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2501_08672_b200.estimator import FilterConfig, NavState, _VisualPass
from paper_2501_08672_b200.geometry import SE3, so3_exp
from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
from paper_2501_08672_b200.scene import T_IC, bake_room, camera_for, orbit_imu_pose
arrays = GaussianArrays(*bake_room(0.0457), device="cuda")
cam = camera_for(1280, 1024); st = RasterSettings(alpha_cut=1 / 255)
T_wi = orbit_imu_pose(0.5 * np.pi)
obs = render(arrays, T_wi @ T_IC, cam, st, retain_cache=False).image.clone()
prior = NavState(SE3(T_wi.R @ so3_exp([0.002, -0.001, 0.003]), T_wi.t + np.array([0.01, -0.005, 0.004])))
vis = _VisualPass(arrays, obs, cam, FilterConfig(), st)
for _ in range(5): vis.run(prior, T_IC)
torch.cuda.synchronize()
N = 50
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
t0 = time.perf_counter()
for a, b in ev:
    a.record(); vis.run(prior, T_IC); b.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / N * 1e3
dev = np.median([a.elapsed_time(b) for a, b in ev])
print(f"wall {wall:.3f} ms/iter, device (event pair, includes host gaps) {dev:.3f}")
# pure device time: enqueue the pass without syncing, several in a row
import ctypes
from paper_2501_08672_b200 import _lib
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a.record()
for _ in range(N):
    vis.run.__func__  # noqa
    st_ = vis.state
    p = st_.arrays.params()
    c = _lib.VisualCfg(); c.budget = 1024; c.observed_u8 = 0; c.grad_thr = 0.05; c.t_max = 0.9; c.gate = 0.15; c.inv_sigma2 = 100.0
    _lib.check(_lib.load().lsb_visual_pass(ctypes.byref(p), ctypes.byref(st_.c_cam), ctypes.byref(st_.c_pose), ctypes.byref(st_.c_set), st_._ws(), st_.ws_bytes, ctypes.byref(st_.dims), ctypes.c_void_p(vis.image.data_ptr()), ctypes.c_void_p(vis.t_final.data_ptr()), ctypes.c_void_p(vis.n_contrib.data_ptr()), ctypes.c_void_p(vis.obs.data_ptr()), ctypes.byref(c), ctypes.byref(vis.bufs), _lib.stream_ptr()), "vp")
b.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"back-to-back passes: device {a.elapsed_time(b)/N:.3f} ms/pass, host enqueue {(t1-t0)/N*1e3:.3f} ms/pass")
