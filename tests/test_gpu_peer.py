"""The fused multi-GPU optimiser step (lsb_adam_peer_step: gradient sum over
ranks + Adam + store into every replica), with G ranks simulated on one GPU
(separate replica / gradient / flag buffers).  Every replica must equal,
bit for bit, one Adam step on the rank-order sum of the gradients, and the
shards' moments together must equal that step's moments."""
import numpy as np
import pytest
import torch

from golden_io import load

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [2, 3, 8])
def test_adam_peer_step_simulated_ranks(G):
    from paper_2501_08672_b200.dist import adam_peer_step, shard_range
    from paper_2501_08672_b200.optimize import AdamState, OptimConfig
    from paper_2501_08672_b200.raster import GaussianArrays
    s = load("scene_room_0323")
    base = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], s["shs"]).clone(torch.float64)
    n, k = len(base), int(base.shs.shape[1])
    gen = torch.Generator(device="cuda").manual_seed(G)
    grads = [torch.randn(n * (10 + 3 * k), generator=gen, device="cuda") * 1e-3 for _ in range(G)]
    cfg = OptimConfig()
    # reference: one Adam step on the rank-order sum
    ref = base.clone()
    gsum = grads[0].clone()
    for q in range(1, G):
        gsum = gsum + grads[q]
    from paper_2501_08672_b200.raster import ParamGradients
    st_ref = AdamState(ref, cfg)
    for _ in range(2):
        st_ref.apply_dev(ref, ParamGradients.from_flat(gsum, n, k))
    # simulated ranks
    reps = [base.clone() for _ in range(G)]
    touched = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(G)]
    states = [AdamState(reps[r], cfg) for r in range(G)]
    for _ in range(2):
        for r in range(G):
            lo, hi = shard_range(n, G, r)
            adam_peer_step(reps, grads, touched, r, lo, hi, states[r])
    torch.cuda.synchronize()
    for r in range(G):
        for f in ("means", "rots", "scales", "opacities", "shs"):
            assert torch.equal(getattr(reps[r], f), getattr(ref, f)), (r, f)
        assert torch.equal(touched[r], st_ref.touched)
    m = torch.zeros_like(st_ref.m)
    v = torch.zeros_like(st_ref.v)
    offs = [0, 3 * n, 6 * n, 9 * n, 10 * n]
    widths = [3, 3, 3, 1, 3 * k]
    for r in range(G):
        lo, hi = shard_range(n, G, r)
        for o, wdt in zip(offs, widths):
            sl = slice(o + wdt * lo, o + wdt * hi)
            m[sl] = states[r].m[sl]
            v[sl] = states[r].v[sl]
    for name, a, b in (("m", m, st_ref.m), ("v", v, st_ref.v)):
        bad = (a != b).nonzero().flatten()
        assert bad.numel() == 0, (name, bad[:5].tolist(), a[bad[:5]].tolist(), b[bad[:5]].tolist(), n, k)


def test_peer_exchange_single_rank(tmp_path):
    """dist.PeerExchange end to end on a one-rank NCCL group: symmetric-memory
    arena, peer pointers, device barriers and the fused kernel inside the
    engine step give the same bits as the plain engine step."""
    import torch.distributed as dist
    from paper_2501_08672_b200.dist import PeerExchange
    from paper_2501_08672_b200.optimize import OptimConfig, WindowEngine
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
    from tools.scene import camera_for, orbit_views
    s = load("scene_room_0323")
    cam = camera_for(160, 128)
    views = orbit_views(3)
    st = RasterSettings(alpha_cut=1 / 255)
    gt = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], s["shs"])
    obs = [render(gt, T, cam, st, retain_cache=False).image.clone() for T in views]
    shs = s["shs"].copy()
    shs[:, 0, :] += 0.05
    results = []
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        for peer in (False, True):
            win = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], shs)
            eng = WindowEngine(win, cam, views, st, OptimConfig(), lanes=2)
            if peer:
                eng.exchange = PeerExchange(eng)
            for _ in range(3):
                eng.step(obs)
            eng.finish()
            torch.cuda.synchronize()
            results.append((win, eng.losses()))
    finally:
        dist.destroy_process_group()
    (w0, l0), (w1, l1) = results
    assert np.array_equal(l0, l1)
    for f in ("means", "rots", "scales", "opacities", "shs"):
        assert torch.equal(getattr(w0, f), getattr(w1, f)), f


def test_peer_exchange_in_cuda_graph(tmp_path):
    """The fused peer step (barriers + kernel) replays inside the step's CUDA
    graph with the same bits as eager steps."""
    import torch.distributed as dist
    from paper_2501_08672_b200.dist import PeerExchange
    from paper_2501_08672_b200.optimize import OptimConfig, WindowEngine
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
    from tools.scene import camera_for, orbit_views
    s = load("scene_room_0323")
    cam = camera_for(160, 128)
    views = orbit_views(3)
    st = RasterSettings(alpha_cut=1 / 255)
    gt = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], s["shs"])
    obs = [render(gt, T, cam, st, retain_cache=False).image.clone() for T in views]
    shs = s["shs"].copy()
    shs[:, 0, :] += 0.05
    out = []
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        for graph in (False, True):
            win = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], shs)
            stream = torch.cuda.Stream()
            eng = WindowEngine(win, cam, views, st, OptimConfig(), lanes=2, stream=stream)
            eng.exchange = PeerExchange(eng)
            with torch.cuda.stream(stream):
                eng.step(obs)
                if graph:
                    eng.capture(obs)
                    for _ in range(2):
                        eng.replay()
                else:
                    for _ in range(2):
                        eng.step(obs)
                eng.finish()
            torch.cuda.synchronize()
            out.append(win)
    finally:
        dist.destroy_process_group()
    for f in ("means", "rots", "scales", "opacities", "shs"):
        assert torch.equal(getattr(out[0], f), getattr(out[1], f)), f


@pytest.mark.parametrize("steps", [1, 3])
def test_adam_group_parts_equal_whole_step(steps):
    """lsb_adam_step_dev_groups: the bucketed multi-GPU step applies Adam to
    one all-reduce bucket at a time (exchange_buckets).  The parts of every
    step together give the bits of one whole-step call — parameters, moments,
    touched flags and the device step count — and a bad group set is refused."""
    from paper_2501_08672_b200 import _lib
    from paper_2501_08672_b200.optimize import AdamState, OptimConfig, exchange_buckets
    from paper_2501_08672_b200.raster import GaussianArrays, ParamGradients
    s = load("scene_room_0323")
    base = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], s["shs"]).clone(torch.float64)
    n, k = len(base), int(base.shs.shape[1])
    gen = torch.Generator(device="cuda").manual_seed(7)
    gs = [torch.randn(n * (10 + 3 * k), generator=gen, device="cuda") * 1e-3 for _ in range(steps)]
    for g in gs:
        g[: 5 * n // 7] *= (torch.rand(5 * n // 7, generator=gen, device="cuda") > 0.5)   # idle rows too
    cfg = OptimConfig()
    whole, parts = base.clone(), base.clone()
    sw, sp = AdamState(whole, cfg), AdamState(parts, cfg)
    buckets = exchange_buckets(n, k)
    for g in gs:
        sw.apply_dev(whole, ParamGradients.from_flat(g, n, k))
        for q, (_, _, groups) in enumerate(buckets):
            sp.apply_dev(parts, ParamGradients.from_flat(g, n, k), groups=groups, advance=q == len(buckets) - 1)
    torch.cuda.synchronize()
    for f in ("means", "rots", "scales", "opacities", "shs"):
        assert torch.equal(getattr(whole, f), getattr(parts, f)), f
    assert torch.equal(sw.m, sp.m) and torch.equal(sw.v, sp.v) and torch.equal(sw.touched, sp.touched)
    assert int(sw.step_dev.item()) == int(sp.step_dev.item()) == steps and sw.step == sp.step == steps
    with pytest.raises(Exception):
        sp.apply_dev(parts, ParamGradients.from_flat(gs[0], n, k), groups=1 | 16)   # mean + sh: not contiguous
    assert _lib.load().lsb_last_error() is not None


def test_bucketed_nccl_exchange_in_cuda_graph(tmp_path):
    """The bucketed NCCL exchange (async all-reduce per bucket, Adam per
    bucket as each completes) on a one-rank NCCL group: eager and captured in
    the step's CUDA graph, the same bits as the engine step without an
    exchange (a one-rank all-reduce is the identity)."""
    import torch.distributed as dist
    from paper_2501_08672_b200.dist import AllReduce
    from paper_2501_08672_b200.optimize import OptimConfig, WindowEngine
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
    from tools.scene import camera_for, orbit_views
    s = load("scene_room_0323")
    cam = camera_for(160, 128)
    views = orbit_views(3)
    st = RasterSettings(alpha_cut=1 / 255)
    gt = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], s["shs"])
    obs = [render(gt, T, cam, st, retain_cache=False).image.clone() for T in views]
    shs = s["shs"].copy()
    shs[:, 0, :] += 0.05
    out = []
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        for mode in ("none", "eager", "graph"):
            win = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], shs)
            stream = torch.cuda.Stream()
            eng = WindowEngine(win, cam, views, st, OptimConfig(), lanes=2, stream=stream)
            ar = None if mode == "none" else AllReduce()
            with torch.cuda.stream(stream):
                eng.step(obs, allreduce=ar)
                if mode == "graph":
                    eng.capture(obs, allreduce=ar)
                    for _ in range(2):
                        eng.replay()
                else:
                    for _ in range(2):
                        eng.step(obs, allreduce=ar)
                eng.finish()
            torch.cuda.synchronize()
            out.append(win)
    finally:
        dist.destroy_process_group()
    for w in out[1:]:
        for f in ("means", "rots", "scales", "opacities", "shs"):
            assert torch.equal(getattr(out[0], f), getattr(w, f)), f
