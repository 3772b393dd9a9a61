"""Per-kernel micro-benchmark of one config-2 view (A/B of library variants).

    LSB_SO=path/to/variant.so python tools/kbench.py [--view 3] [--reps 50] [--bin-mode 1]

Bins one view once, then times each pass back to back `reps` times with CUDA
events on one stream (bin, blend+loss, blend bwd, chain) and prints the mean
microseconds per launch as one JSON line.  The inputs are the bench's own
(room scene v_s 0.0723, 1280x1024, alpha_cut 1/255).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--view", type=int, default=3)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--bin-mode", type=int, default=1)
    ap.add_argument("--vs", type=float, default=0.0723)
    ap.add_argument("--count", action="store_true", help="pass an n_contrib buffer (counting forward)")
    ap.add_argument("--size", default="1280x1024", help="WxH")
    ap.add_argument("--views", type=int, default=10, help="orbit views (the view index is into these)")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2501_08672_b200.optimize import LossBuffers, ParamGradients
    from paper_2501_08672_b200.raster import (GaussianArrays, RasterSettings, RenderState, render, render_bin,
                                              render_blend, render_blend_bwd, render_blend_bwd_loss,
                                              render_blend_fused_loss,
                                              render_blend_loss, render_chain)
    from tools.scene import bake_room, camera_for, orbit_views
    torch.cuda.set_device(0)
    P = bake_room(args.vs)
    W, H = (int(v) for v in args.size.split("x"))
    cam = camera_for(W, H)
    st = RasterSettings(alpha_cut=1.0 / 255.0)
    arrays = GaussianArrays(*P, device="cuda")
    T = orbit_views(args.views)[args.view]
    obs = render(arrays, T, cam, st, retain_cache=False).image.clone()
    Tc = T.inverse()
    state = RenderState(arrays, cam, Tc.R, Tc.t, st, 1 << 23, args.bin_mode)
    h, w = cam.height, cam.width
    img = torch.empty((h, w, 3), device="cuda")
    tf = torch.empty((h, w), device="cuda")
    gimg = torch.empty((h, w, 3), device="cuda")
    nc = torch.empty((h, w), dtype=torch.int32, device="cuda") if args.count else None
    loss = LossBuffers(torch.device("cuda"), 1)
    grads = ParamGradients.zeros(len(arrays), int(arrays.shs.shape[1]), torch.device("cuda"))
    s = torch.cuda.current_stream()
    passes = {
        "bin": lambda: render_bin(state, s),
        "blend_fwd": lambda: render_blend_loss(state, img, tf, nc, obs, 0, 1.0 / (3 * h * w), gimg, loss.ptr(0),
                                               stream=s),
        "blend_bwd": lambda: render_blend_bwd(state, img, nc, gimg, 1.0, s),
        "blend_nc": lambda: render_blend(state, img, tf, nc, stream=s),
        "blend_bwd_loss": lambda: render_blend_bwd_loss(state, img, obs, 0, 1.0 / (3 * h * w), loss.ptr(0), s),
        "blend_fused": lambda: render_blend_fused_loss(state, obs, 0, 1.0 / (3 * h * w), loss.ptr(0), s),
        "chain": lambda: render_chain(state, grads, None, s),
    }
    for f in passes.values():
        f()
    torch.cuda.synchronize()
    M, I, over, _ = state.read_counts()
    out = {"M": M, "I": I, "so": os.path.basename(os.environ.get("LSB_SO", "libsplat_b200.so"))}
    for name, f in passes.items():
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.reps):
            f()
        e1.record(s)
        torch.cuda.synchronize()
        out[name + "_us"] = round(e0.elapsed_time(e1) * 1e3 / args.reps, 2)
    out["loss"] = float(loss.sums().flatten()[0].item())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
