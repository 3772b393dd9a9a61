"""Diagnose optimize_window parity: compare the first-iteration gradients of
the engine (fused loss) with the oracle, group by group."""
import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import torch
from types import SimpleNamespace
from golden_io import load
from oracle import raster as orc
from oracle.optim import photometric_loss as ref_loss
from paper_2501_08672_b200.geometry import PinholeCamera, SE3
from paper_2501_08672_b200.optimize import OptimConfig, WindowEngine
from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, backward, render

d = load("optimize_plane")
n = len(d["in_means"])
fx, fy, cx, cy, w, h = d["cam"]
cam = PinholeCamera(fx, fy, cx, cy, int(w), int(h))
P = {"means": d["in_means"].astype(float), "rots": d["in_rots"].astype(float).reshape(n, 3, 3),
     "scales": d["in_scales"].astype(float), "opacities": d["in_opacities"].astype(float), "shs": d["in_shs"].astype(float)}
st = SimpleNamespace(near=0.01, dilation=0.3, alpha_clamp=0.99, transmittance_min=1e-4, footprint_sigma=6.0,
                     alpha_cut=0.0, max_footprint_px=512.0, background=np.zeros(3), sh_degree=0)
c = orc.render(P, np.eye(3), np.zeros(3), cam, st)
val, mse, gimg = ref_loss(c["image"], d["observed"])
ref = orc.backward(c, gimg)["grads"]
arrays = GaussianArrays(P["means"], P["rots"], P["scales"], P["opacities"], P["shs"])
out = render(arrays, SE3.identity(), cam, RasterSettings())
print("image err", np.abs(out.image.cpu().numpy() - c["image"]).max())
g, _ = backward(out, gimg)
gn = g.numpy()
for k in ref:
    print("backward(ref grad img)", k, np.abs(gn[k] - ref[k]).max() / np.abs(ref[k]).max())
eng = WindowEngine(arrays, cam, [SE3.identity()], RasterSettings(), OptimConfig())
obs = torch.as_tensor(d["observed"], dtype=torch.float32, device="cuda").contiguous()
# run the step pieces without Adam
from paper_2501_08672_b200.raster import render_bin, render_blend_loss, render_blend_bwd, render_chain
eng.grads.flat.zero_()
T = eng.views[0]
eng.state.set_pose(T.R, T.t)
render_bin(eng.state)
render_blend_loss(eng.state, eng.image, eng.t_final, eng.n_contrib, obs, 0, 1.0 / (3 * h * w), eng.grad_image,
                  eng.loss.ptr(0))
gi = eng.grad_image.cpu().numpy()
print("grad image sign mismatches", int((np.sign(gi) != np.sign(gimg)).sum()), "max diff", np.abs(gi - gimg).max())
render_blend_bwd(eng.state, eng.image, eng.n_contrib, eng.grad_image, 1.0)
render_chain(eng.state, eng.grads, None)
ge = eng.grads.numpy()
for k in ref:
    print("engine", k, np.abs(ge[k] - ref[k]).max() / np.abs(ref[k]).max())
eng.adam.apply(arrays, eng.grads)
torch.cuda.synchronize()
from oracle.optim import Adam, adam_param_step, DEFAULT_CFG
P2 = {k: v.copy() for k, v in P.items()}
adam = Adam({"mean": (n, 3), "rot": (n, 3), "scale": (n, 3), "opacity": (n,), "sh": P["shs"].shape})
adam_param_step(P2, ref, adam, DEFAULT_CFG, np.zeros(n, bool))
for k, ak in (("means", "means"), ("rots", "rots"), ("scales", "scales"), ("opacities", "opacities"), ("shs", "shs")):
    got = getattr(arrays, ak).cpu().numpy().reshape(P2[k].shape)
    print("after adam", k, np.abs(got - P2[k]).max(), "moved", np.abs(P2[k] - P[k]).max())

# ---- full optimize_window, per iteration, against the oracle ------------------
from paper_2501_08672_b200.optimize import optimize_window
from oracle.optim import optimize_views
arrays2 = GaussianArrays(P["means"], P["rots"], P["scales"], P["opacities"], P["shs"])
hist = optimize_window(arrays2, d["observed"], SE3.identity(), cam, OptimConfig(), RasterSettings(), iters=3)
print("gpu losses", [h.value for h in hist])
print("ref losses", d["loss"][:3])
for it in (1, 2, 3):
    Po, ho = optimize_views(P, [d["observed"]], [(np.eye(3), np.zeros(3))], cam, st, it)
    print("oracle iters", it, "losses", [x[0] for x in ho])
