"""cProfile of the config-4 IESKF update loop (timing aid)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2501_08672_b200.estimator import FilterConfig, NavState, ieskf_visual_update
from paper_2501_08672_b200.geometry import SE3, so3_exp
from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
from paper_2501_08672_b200.scene import T_IC, bake_room, camera_for, orbit_imu_pose
arrays = GaussianArrays(*bake_room(0.0457), device="cuda")
cam = camera_for(1280, 1024); st = RasterSettings(alpha_cut=1 / 255)
T_wi = orbit_imu_pose(0.5 * np.pi)
obs = render(arrays, T_wi @ T_IC, cam, st, retain_cache=False).image.clone()
prior = NavState(SE3(T_wi.R @ so3_exp([0.002, -0.001, 0.003]), T_wi.t + np.array([0.01, -0.005, 0.004])))
cov0 = np.diag(np.concatenate([np.full(3, 1e-8), np.full(3, 1e-8), np.full(3, 1e-6), np.full(3, 1e-8), np.full(3, 1e-6)]))
f = lambda: ieskf_visual_update(prior, cov0, obs, arrays, cam, T_IC, FilterConfig(), st, max_iter=5, step_tol=0.0)
for _ in range(5): f()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): f()
torch.cuda.synchronize()
print("ms/update", (time.perf_counter() - t0) / 20 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): f()
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
