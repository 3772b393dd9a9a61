"""Host-side breakdown of one visual IESKF iteration at config 4 (timing aid)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2501_08672_b200.estimator import FilterConfig, NavState, visual_measurement, select_semi_dense_pixels
from paper_2501_08672_b200.geometry import SE3, so3_exp
from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render, pose_rows
from paper_2501_08672_b200.scene import T_IC, bake_room, camera_for, orbit_imu_pose
arrays = GaussianArrays(*bake_room(0.0457), device="cuda")
cam = camera_for(1280, 1024); st = RasterSettings(alpha_cut=1 / 255)
T_wi = orbit_imu_pose(0.5 * np.pi)
obs = render(arrays, T_wi @ T_IC, cam, st, retain_cache=False).image.clone()
state = NavState(SE3(T_wi.R @ so3_exp([0.002, -0.001, 0.003]), T_wi.t + np.array([0.01, -0.005, 0.004])))
cfg = FilterConfig()
def tic(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = tic(); out = render(arrays, state.T_WI @ T_IC, cam, st, bin_mode=1); t1 = tic()
    ids = select_semi_dense_pixels(obs, out.final_transmittance, cfg); t2 = tic()
    idt = torch.as_tensor(ids, device="cuda")
    rows = pose_rows(out, idt, T_ic=T_IC, as_numpy=False); t3 = tic()
    m = visual_measurement(state, obs, arrays, cam, T_IC, cfg, st); A, b = m.hb(); t4 = tic()
    print(f"render {1e3*(t1-t0):.3f} select {1e3*(t2-t1):.3f} pose_rows {1e3*(t3-t2):.3f} full measurement+hb {1e3*(t4-t3):.3f} ms")
