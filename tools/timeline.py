"""Timeline of one eager window step with its view lanes (CUDA events on
each lane's stream, offsets from the step's start in ms): when each view's
binning, fused blend and chain start and end, and when Adam runs — where the
step's time beyond the blends goes (pipeline fill, tail).

    python tools/timeline.py [--config target] [--lanes 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="target")
    ap.add_argument("--lanes", type=int, default=5)
    args = ap.parse_args()
    import torch
    import bench
    from paper_2501_08672_b200.optimize import OptimConfig, WindowEngine
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render

    dev = torch.device("cuda", 0)
    wl = bench.build_workload(args.config, 1.0 / 255.0)
    st = RasterSettings(alpha_cut=wl["alpha_cut"])
    gt = GaussianArrays(*wl["gt"], device=dev)
    obs = [torch.clamp(torch.round(render(gt, T, wl["cam"], st, retain_cache=False).image.double() * 255.0), 0, 255)
           .to(torch.uint8) for T in wl["views"]]
    win = GaussianArrays(*wl["win"], device=dev)
    stream = torch.cuda.Stream(dev)
    eng = WindowEngine(win, wl["cam"], wl["views"], st, OptimConfig(), stream=stream, lanes=args.lanes)
    with torch.cuda.stream(stream):
        for _ in range(3):
            eng.step(obs)
    torch.cuda.synchronize()
    for rep in range(2):
        timers: dict = {}
        t0 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            t0.record(stream)
            eng.step(obs, timers=timers)
        torch.cuda.synchronize()
    off = {k: [t0.elapsed_time(e) for e in v] for k, v in timers.items()}
    print(f"{'view':>4} {'bin':>15} {'blend':>15} {'chain':>15}")
    for v in range(len(wl["views"])):
        row = [f"{off[k][2 * v]:6.3f}-{off[k][2 * v + 1]:6.3f}" for k in ("bin", "blend", "chain")]
        print(f"{v:>4} " + " ".join(f"{r:>15}" for r in row))
    a = off["adam"]
    print(f"adam {a[0]:.3f}-{a[1]:.3f}; step end {a[-1]:.3f} ms; blend sum "
          f"{sum(off['blend'][2 * v + 1] - off['blend'][2 * v] for v in range(len(wl['views']))):.3f} ms")


if __name__ == "__main__":
    main()
