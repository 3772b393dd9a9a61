"""The view-sharded window step run as real ranks (2 and 4 processes sharing
cuda:0, gloo) - ViewShardedWindow with whole views and with row bands,
two optimisation steps - against the single-process engine:

* 2 ranks, whole views: every rank's parameters after each Adam step equal,
  bit for bit, the single-process engine stepping on the two ranks' partial
  gradients summed (a two-operand sum is order-free);
* 4 ranks, row bands (6 views -> 12 half views): replicas bit-identical
  across ranks, and within round-off of the single-process whole-view step.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(n_views):
    import torch
    from golden_io import load
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
    from tools.scene import camera_for, orbit_views
    s = load("scene_room_0323")
    cam = camera_for(160, 128)
    views = orbit_views(n_views)
    st = RasterSettings(alpha_cut=1 / 255)
    gt = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], s["shs"])
    frames = [torch.clamp(torch.round(render(gt, T, cam, st, retain_cache=False).image.double() * 255.0), 0, 255)
              .to(torch.uint8) for T in views]
    shs = s["shs"].copy()
    shs[:, 0, :] += np.random.default_rng(0).uniform(-0.1, 0.1, shs[:, 0, :].shape)
    win = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], shs)
    return win, cam, views, st, frames


def _state(arrays):
    return {k: getattr(arrays, k).cpu().numpy().copy() for k in ("means", "rots", "scales", "opacities", "shs")}


def _worker(rank, world, port, n_views, steps, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_08672_b200.dist import ViewShardedWindow, replicas_identical
        from paper_2501_08672_b200.optimize import OptimConfig
        win, cam, views, st, frames = _setup(n_views)
        vw = ViewShardedWindow(win, cam, views, st, OptimConfig(), lanes=2)
        obs = vw.observed_for(frames)
        out = []
        for _ in range(steps):
            vw.step(obs, check=True)
            torch.cuda.synchronize()
            out.append(_state(vw.engine.arrays))
        same = replicas_identical(vw.engine.arrays.means) and replicas_identical(vw.engine.arrays.shs)
        q.put((rank, vw.units, out, same))
    except Exception as exc:                    # noqa: BLE001 - report to the parent
        q.put((rank, None, repr(exc), False))
    finally:
        dist.destroy_process_group()


def _run(world, n_views, steps):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_views, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    out.sort(key=lambda x: x[0])
    for r, units, st, _ in out:
        assert units is not None, f"rank {r}: {st}"
    for p in procs:
        assert p.exitcode == 0
    return out


@pytest.mark.timeout(900)
def test_two_ranks_equal_single_process_bit_for_bit():
    import torch
    from paper_2501_08672_b200.optimize import OptimConfig, WindowEngine
    steps = 2
    out = _run(2, 4, steps)
    assert all(o[3] for o in out), "replicas diverged"
    for k in ("means", "shs", "opacities", "scales", "rots"):
        assert np.array_equal(out[0][2][-1][k], out[1][2][-1][k]), k
    # single process: engine R renders rank 0's views and, in place of the
    # all-reduce, adds the gradient of engine B (rank 1's views, same state)
    win, cam, views, st, frames = _setup(4)
    units = [out[0][1], out[1][1]]
    engR = WindowEngine(win, cam, [views[v] for v, _, _ in units[0]], st, OptimConfig(), n_views_total=4, lanes=2)
    winB = win.clone()
    engB = WindowEngine(winB, cam, [views[v] for v, _, _ in units[1]], st, OptimConfig(), n_views_total=4, lanes=2)
    obsR = [frames[v] for v, _, _ in units[0]]
    obsB = [frames[v] for v, _, _ in units[1]]
    for s in range(steps):
        engB.arrays.copy_from(engR.arrays)
        engB.step(obsB)                        # its own Adam is discarded; its gradient is rank 1's
        engR.step(obsR, allreduce=lambda t: t.add_(engB.grads.flat))
        torch.cuda.synchronize()
        ref = _state(engR.arrays)
        for k in ref:
            assert np.array_equal(out[0][2][s][k], ref[k]), (s, k)


@pytest.mark.timeout(900)
def test_four_ranks_row_bands_match_single_process():
    import torch
    from paper_2501_08672_b200.dist import view_bands
    from paper_2501_08672_b200.optimize import OptimConfig, WindowEngine
    assert view_bands(6, 4, 128) == 2
    out = _run(4, 6, 1)                 # shard_units_mixed: 1 whole view + 1 half of views 4, 5 per rank
    assert all(o[3] for o in out), "replicas diverged"
    assert all(len(o[1]) == 2 for o in out)
    assert any(y0 > 0 for o in out for _, y0, _ in o[1])         # (row bands, not whole views)
    for r in range(1, 4):
        for k in ("means", "shs"):
            assert np.array_equal(out[0][2][0][k], out[r][2][0][k]), (r, k)
    win, cam, views, st, frames = _setup(6)
    eng = WindowEngine(win, cam, views, st, OptimConfig(), lanes=2)
    eng.step(frames)
    torch.cuda.synchronize()
    ref = _state(eng.arrays)
    # Adam's first step is +-lr per entry: compare where the step is firm
    for k in ("means", "shs"):
        d = np.abs(out[0][2][0][k] - ref[k])
        moved = np.abs(ref[k] - getattr(win, k).cpu().numpy().astype(np.float64)).max()
        assert (d <= 1e-9 * max(1.0, np.abs(ref[k]).max())).mean() >= 0.999, k
        assert d.max() <= 2.0001 * moved, k
