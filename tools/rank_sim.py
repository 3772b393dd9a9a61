"""Per-rank compute of the view-sharded step at G = 1, 2, 4, 8 GPUs, measured
on ONE B200 (this pool has no multi-GPU node): for every rank r of a G-rank
job, the WindowEngine that rank would build (its render units:
dist.shard_units_mixed — whole views first, row bands of the leftover views
when G does not divide them; --units banded bands every view) is captured as a CUDA graph WITHOUT the gradient exchange and timed
alone (L2 flushed before each step, median of --steps).  The job's step is
then max over ranks of that time plus the exchange, which is modelled, not
measured: one NCCL all-reduce of the flat f32 gradient buffer (4 (10 + 3K) N
bytes) at an assumed bus bandwidth (--busbw GB/s; ring all-reduce time =
2 (G-1)/G x bytes / busbw), partly hidden behind the bucketed Adam.

    python tools/rank_sim.py --config target --gpus 1 2 4 8 > gpurun_out/rank_sim_target.json
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="target")
    ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--lanes", type=int, default=5)
    ap.add_argument("--busbw", type=float, default=600.0, help="assumed NCCL all-reduce bus bandwidth, GB/s")
    ap.add_argument("--units", default="mixed", choices=["banded", "mixed"],
                    help="dist.shard_units (band every view) or dist.shard_units_mixed (whole views first)")
    args = ap.parse_args()
    import torch
    import bench
    from paper_2501_08672_b200.dist import shard_units, shard_units_mixed, view_bands
    from paper_2501_08672_b200.optimize import OptimConfig, WindowEngine
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    wl = bench.build_workload(args.config, 1.0 / 255.0)
    settings = RasterSettings(alpha_cut=wl["alpha_cut"])
    V, W, H, N = wl["V"], wl["W"], wl["H"], wl["N"]
    gt = GaussianArrays(*wl["gt"], device=dev)
    frames = {v: torch.clamp(torch.round(render(gt, wl["views"][v], wl["cam"], settings, retain_cache=False)
                                         .image.double() * 255.0), 0, 255).to(torch.uint8) for v in range(V)}
    del gt
    flush = torch.empty(64 * 2 ** 20, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(dev)
    K = int(np.asarray(wl["win"][4]).shape[1])
    grad_bytes = 4 * (10 + 3 * K) * N
    out = {"config": args.config, "gaussians": N, "views": V, "width": W, "height": H,
           "grad_bytes": grad_bytes, "busbw_assumed_GBps": args.busbw, "per_world": {}}
    for G in args.gpus:
        per_rank = []
        for r in range(G):
            units = (shard_units if args.units == "banded" else shard_units_mixed)(V, G, r, H)
            win = GaussianArrays(*wl["win"], device=dev)
            eng = WindowEngine(win, wl["cam"], [wl["views"][u[0]] for u in units], settings, OptimConfig(),
                               n_views_total=V, stream=stream, lanes=args.lanes,
                               bands=[(u[1], u[2]) for u in units])
            obs = [frames[v][y0:y1].contiguous() for v, y0, y1 in units]
            with torch.cuda.stream(stream):
                for _ in range(args.warmup):
                    eng.step(obs)
            eng.capture(obs, None)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            with torch.cuda.stream(stream):
                for a, b in evs:
                    flush.zero_()
                    a.record(stream)
                    eng.replay()
                    b.record(stream)
            torch.cuda.synchronize()
            assert eng.check_capacity()
            per_rank.append(float(np.median([a.elapsed_time(b) for a, b in evs])))
            del eng, win
            torch.cuda.empty_cache()
        comp = max(per_rank)
        ar_ms = 0.0 if G == 1 else 2.0 * (G - 1) / G * grad_bytes / (args.busbw * 1e9) * 1e3
        out["per_world"][str(G)] = {
            "units_per_rank": len((shard_units if args.units == "banded" else shard_units_mixed)(V, G, 0, H)),
            "unit_mode": args.units, "bands_per_view": view_bands(V, G, H),
            "rank_compute_ms": per_rank, "max_rank_compute_ms": comp,
            "allreduce_model_ms": ar_ms, "step_model_ms": comp + ar_ms,
            "mpix_per_s_model": V * W * H / ((comp + ar_ms) * 1e-3) / 1e6}
        print(f"G={G}: per-rank compute {['%.3f' % t for t in per_rank]} ms, all-reduce (model) {ar_ms:.3f} ms",
              file=sys.stderr)
    base = out["per_world"].get("1", {}).get("step_model_ms")
    if base:
        for G, d in out["per_world"].items():
            d["efficiency_model"] = base / (int(G) * d["step_model_ms"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
