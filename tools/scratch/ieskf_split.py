"""Split of one config-4 IESKF update into the device pass and the host algebra (timing aid)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2501_08672_b200.estimator as E
from paper_2501_08672_b200.geometry import SE3, so3_exp
from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
from paper_2501_08672_b200.scene import T_IC, bake_room, camera_for, orbit_imu_pose
arrays = GaussianArrays(*bake_room(0.0457), device="cuda")
cam = camera_for(1280, 1024); st = RasterSettings(alpha_cut=1 / 255)
T_wi = orbit_imu_pose(0.5 * np.pi)
obs = render(arrays, T_wi @ T_IC, cam, st, retain_cache=False).image.clone()
prior = E.NavState(SE3(T_wi.R @ so3_exp([0.002, -0.001, 0.003]), T_wi.t + np.array([0.01, -0.005, 0.004])))
cov0 = np.diag(np.concatenate([np.full(3, 1e-8), np.full(3, 1e-8), np.full(3, 1e-6), np.full(3, 1e-8), np.full(3, 1e-6)]))
cfg = E.FilterConfig()
tot = {"run": 0.0}
orig = E._VisualPass.run
def timed_run(self, nav, T_ic):
    t0 = time.perf_counter(); r = orig(self, nav, T_ic); tot["run"] += time.perf_counter() - t0; return r
E._VisualPass.run = timed_run
for _ in range(5): E.ieskf_visual_update(prior, cov0, obs, arrays, cam, T_IC, cfg, st, max_iter=5, step_tol=0.0)
torch.cuda.synchronize()
tot["run"] = 0.0
N = 30
t0 = time.perf_counter()
for _ in range(N): E.ieskf_visual_update(prior, cov0, obs, arrays, cam, T_IC, cfg, st, max_iter=5, step_tol=0.0)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / N * 1e3
print(f"update {wall:.3f} ms; passes {tot['run'] / N * 1e3:.3f} ms; rest {wall - tot['run'] / N * 1e3:.3f} ms")
