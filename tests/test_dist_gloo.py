"""Multi-process (world size 2, gloo, CPU) tests of the view-sharded window
step's host logic: view partition, the gradient all-reduce over the flat
ParamGradients buffer, and replica identity after the deterministic update.
The per-view gradients come from the CPU oracle (test infrastructure)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_io import load


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_views_partition():
    from paper_2501_08672_b200.dist import shard_views
    for n in (1, 10, 64):
        for world in (1, 2, 4, 8):
            parts = [shard_views(n, world, r) for r in range(world)]
            flat = sorted(v for p in parts for v in p)
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


@pytest.mark.parametrize("n,height", [(10, 1024), (64, 1080), (10, 80), (3, 48), (7, 1024)])
def test_mixed_units_cover_every_row_once_and_balance_pixels(n, height):
    """shard_units_mixed (the default split): every (view, row) rendered by
    exactly one rank, whole views first, every rank the same number of pixel
    rows whenever a band split exists."""
    from paper_2501_08672_b200.dist import shard_units_mixed
    for world in (1, 2, 4, 8):
        parts = [shard_units_mixed(n, world, r, height) for r in range(world)]
        cover = np.zeros((n, height), np.int32)
        for p in parts:
            for v, y0, y1 in p:
                assert y0 % 16 == 0 and y0 < y1
                cover[v, y0:y1] += 1
        assert (cover == 1).all()
        rows = [sum(y1 - y0 for _, y0, y1 in p) for p in parts]
        r, trows = n % world, (height + 15) // 16
        if r == 0 or any(b <= trows and (r * b) % world == 0 for b in (2, 4, 8)):
            assert max(rows) - min(rows) <= 16, rows                 # tile-aligned bands


@pytest.mark.parametrize("n,height", [(10, 1024), (64, 1080), (10, 80), (3, 48), (7, 1024)])
def test_shard_units_cover_every_row_once_and_balance(n, height):
    """Row-band units: every (view, row) rendered by exactly one rank; equal
    unit counts whenever a band split exists; bands start on tile rows."""
    from paper_2501_08672_b200.dist import shard_units, view_bands
    for world in (1, 2, 4, 8):
        parts = [shard_units(n, world, r, height) for r in range(world)]
        cover = np.zeros((n, height), np.int32)
        for p in parts:
            for v, y0, y1 in p:
                assert y0 % 16 == 0 and y0 < y1
                cover[v, y0:y1] += 1
        assert (cover == 1).all()
        b = view_bands(n, world, height)
        if b > 1 or n % world == 0:
            assert len({len(p) for p in parts}) == 1


def _views_and_scene():
    from types import SimpleNamespace
    from tools.scene import camera_for, orbit_views
    s = load("scene_room_0323")
    P = {k: s[k].astype(np.float64) for k in ("means", "rots", "scales", "opacities", "shs")}
    cam = camera_for(96, 80)
    st = SimpleNamespace(near=0.01, dilation=0.3, alpha_clamp=0.99, transmittance_min=1e-4, footprint_sigma=6.0,
                         alpha_cut=1 / 255, max_footprint_px=512.0, background=np.zeros(3), sh_degree=0)
    return P, cam, st, orbit_views(4)


def _view_grad_flat(P, cam, st, T_wc, V):
    """Oracle gradient of one view's L1 loss against a shifted-colour target,
    scaled by 1/V and packed in the ParamGradients flat layout."""
    from oracle import raster as orc
    from oracle.optim import photometric_loss
    from paper_2501_08672_b200.raster import ParamGradients
    T_cw = T_wc.inverse()
    c = orc.render(P, T_cw.R, T_cw.t, cam, st)
    target = np.clip(c["image"] * 0.9 + 0.05, 0, 1)
    _, _, g_img = photometric_loss(c["image"], target)
    g = orc.backward(c, g_img)["grads"]
    n, k = len(P["means"]), P["shs"].shape[1]
    pg = ParamGradients.zeros(n, k, "cpu")
    for name in ("mean", "rot", "scale", "opacity", "sh"):
        getattr(pg, name).copy_(torch.from_numpy(g[name] / V).to(torch.float32))
    return pg.flat


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_08672_b200.dist import make_allreduce, replicas_identical, shard_views
        P, cam, st, views = _views_and_scene()
        V = len(views)
        flat = None
        for v in shard_views(V, world, rank):
            g = _view_grad_flat(P, cam, st, views[v], V)
            flat = g if flat is None else flat + g
        allreduce = make_allreduce()
        assert allreduce is not None
        allreduce(flat)
        # the same deterministic update on every rank keeps replicas identical
        params = torch.from_numpy(P["means"].astype(np.float32).ravel().copy())
        n = len(P["means"])
        params -= 1e-3 * torch.sign(flat[: 3 * n])
        ok = replicas_identical(params)
        q.put((rank, flat.numpy(), ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_view_sharded_allreduce_equals_single_process_mean():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda x: x[0])
    assert np.array_equal(out[0][1], out[1][1]), "ranks disagree after the all-reduce"
    assert out[0][2] and out[1][2], "replicas diverged"
    # single-process reference: the mean of all per-view gradients
    P, cam, st, views = _views_and_scene()
    ref = sum(_view_grad_flat(P, cam, st, T, len(views)) for T in views).numpy()
    assert np.abs(out[0][1] - ref).max() <= 1e-6 * max(np.abs(ref).max(), 1e-12)


def test_exchange_buckets_tile_the_flat_buffer_and_adam_groups():
    """The bucketed exchange's buckets cover the ParamGradients flat layout
    exactly once, in order, and their Adam groups partition every group."""
    from paper_2501_08672_b200.optimize import ADAM_ALL, exchange_buckets
    from paper_2501_08672_b200.raster import ParamGradients
    for n, k in ((1, 1), (37, 1), (1000, 4), (5, 16)):
        b = exchange_buckets(n, k)
        assert b[0][0] == 0 and b[-1][1] == ParamGradients.zeros(n, k, "cpu").flat.numel()
        assert all(b[q][1] == b[q + 1][0] for q in range(len(b) - 1))
        groups = [g for _, _, g in b]
        assert sum(groups) == ADAM_ALL and all(g & h == 0 for i, g in enumerate(groups) for h in groups[i + 1:])
        pg = ParamGradients.zeros(n, k, "cpu")
        # each bucket is exactly the flat range of its groups' tensors
        names = {1: ["mean"], 2: ["rot"], 12: ["scale", "opacity"], 16: ["sh"]}
        for lo, hi, g in b:
            size = sum(getattr(pg, f).numel() for f in names[g])
            assert hi - lo == size


def _bucket_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_08672_b200.dist import make_allreduce
        from paper_2501_08672_b200.optimize import exchange_buckets
        n, k = 301, 1
        g = torch.from_numpy(np.random.default_rng(rank).standard_normal((10 + 3 * k) * n).astype(np.float32))
        one = g.clone()
        ar = make_allreduce()
        ar(one)
        part = g.clone()
        works = [ar.start(part[lo:hi]) for lo, hi, _ in exchange_buckets(n, k)]
        for w in works:
            ar.wait(w)
        q.put((rank, bool(torch.equal(one, part)), one.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_bucketed_allreduce_equals_one_shot_two_ranks():
    """Two ranks: the bucketed (async, in-place on views) all-reduce gives the
    one-shot all-reduce's bits on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_bucket_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    assert np.array_equal(res[0][2], res[1][2])
