"""Per-rank step time of the view-sharded config-2 step, simulated on one GPU
(rank 0's units at world N, no all-reduce): whole views (v mod N) vs row
bands (dist.shard_units).  Timing aid for the scaling design."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2501_08672_b200.dist import shard_units, shard_views
from paper_2501_08672_b200.optimize import OptimConfig, WindowEngine
from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
from paper_2501_08672_b200.scene import bake_room, camera_for, orbit_views
import bench
wl = bench.build_workload("cfg2", 1 / 255)
dev = torch.device("cuda", 0)
st = RasterSettings(alpha_cut=1 / 255)
gt = GaussianArrays(*wl["gt"], device=dev)
V, H = wl["V"], wl["H"]
frames = {v: torch.clamp(torch.round(render(gt, wl["views"][v], wl["cam"], st, retain_cache=False).image.double() * 255), 0, 255).to(torch.uint8) for v in range(V)}
flush = torch.empty(64 * 2 ** 20, dtype=torch.int32, device=dev)
def time_units(units, reps=20):
    win = GaussianArrays(*wl["win"], device=dev)
    s = torch.cuda.Stream()
    eng = WindowEngine(win, wl["cam"], [wl["views"][v] for v, _, _ in units], st, OptimConfig(), n_views_total=V,
                       stream=s, lanes=5, bands=[(a, b) for _, a, b in units])
    obs = [frames[v][a:b].contiguous() for v, a, b in units]
    with torch.cuda.stream(s):
        for _ in range(3): eng.step(obs)
    torch.cuda.synchronize()
    eng.capture(obs)
    ts = []
    for _ in range(reps):
        with torch.cuda.stream(s):
            flush.zero_(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); eng.replay(); b.record(s)
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))
for world in (1, 2, 4, 8):
    whole = [(v, 0, H) for v in shard_views(V, world, 0)]
    banded = shard_units(V, world, 0, H)
    tw = time_units(whole)
    tb = time_units(banded) if banded != whole else tw
    print(f"N={world}: rank-0 whole views {len(whole)} -> {tw:.3f} ms; units {len(banded)} -> {tb:.3f} ms; "
          f"ideal {time_units([(v, 0, H) for v in range(V)]) / world if world == 1 else float('nan'):.3f}")
