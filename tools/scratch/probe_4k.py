"""4K-frame probe (debug aid): which stage fails, and where the image differs."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
from types import SimpleNamespace
from oracle import raster as orc
from paper_2501_08672_b200.geometry import SE3
from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
rng = np.random.default_rng(44)
n = 3000
f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
P = {"means": f32(np.column_stack([rng.uniform(-1.6, 1.6, n), rng.uniform(-0.9, 0.9, n), rng.uniform(2, 4, n)])),
     "rots": f32(np.tile(np.eye(3), (n, 1, 1))), "scales": f32(np.column_stack([rng.uniform(0.005, 0.03, n)] * 3)),
     "opacities": f32(rng.uniform(0.2, 0.9, n)), "shs": f32(rng.uniform(-1, 1, (n, 1, 3)))}
W, H = int(sys.argv[1]), int(sys.argv[2])
cam = SimpleNamespace(fx=2000.0 * W / 3840, fy=2000.0 * W / 3840, cx=W / 2, cy=H / 2, width=W, height=H)
st = SimpleNamespace(near=0.01, dilation=0.3, alpha_clamp=0.99, transmittance_min=1e-4, footprint_sigma=6.0,
                     alpha_cut=1 / 255, max_footprint_px=512.0, background=np.array([0.1, 0.2, 0.3]), sh_degree=0)
ref = orc.render(P, np.eye(3), np.zeros(3), cam, st)
arrays = GaussianArrays(P["means"], P["rots"], P["scales"], P["opacities"], P["shs"])
out = render(arrays, SE3.identity(), cam, RasterSettings(alpha_cut=1 / 255, background=(0.1, 0.2, 0.3)))
print("counts", out.cache.counts)
o = out.numpy()
d = np.abs(o["image"] - ref["image"]).max(axis=2)
print("max diff", d.max(), "n>1e-4", int((d > 1e-4).sum()))
ys, xs = np.nonzero(d > 1e-4)
if len(ys):
    print("bad pixels y range", ys.min(), ys.max(), "x range", xs.min(), xs.max())
    print("tiles", sorted(set(((ys // 16) * ((W + 15) // 16) + xs // 16).tolist()))[:20])
    y, x = ys[0], xs[0]
    print("pixel", y, x, "gpu", o["image"][y, x], "ref", ref["image"][y, x], "ncontrib gpu", o["contrib_count"][y, x],
          "ref", ref["n_proc"].reshape(H, W)[y, x], "T gpu", o["final_transmittance"][y, x], "ref", ref["t_final"].reshape(H, W)[y, x])
