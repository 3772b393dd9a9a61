"""View-sharded multi-GPU window optimisation (one process per GPU).

The keyframe views of a sliding-window step are independent until their
gradients meet: view v is rendered and back-propagated on rank v mod world,
every rank keeps a full replica of the window parameters, one all-reduce
(sum) of the flat f32 gradient buffer runs per step through
torch.distributed (NCCL over NVLink on the B200 box), and every rank then
applies the same deterministic Adam step, so the replicas stay bit-identical
(SURVEY.md §8(e)).  The per-view gradient is scaled by 1/n_views_total on
each rank, so the summed buffer is the mean of the per-view gradients — the
same quantity the single-GPU engine computes.
"""

from __future__ import annotations

from typing import Callable, Optional, Sequence

import torch
import torch.distributed as dist


def shard_views(n_views: int, world: int, rank: int) -> list:
    """Views owned by `rank`: v -> rank v mod world."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return [v for v in range(n_views) if v % world == rank]


def view_bands(n_views: int, world: int, height: int, tile: int = 16, max_split: int = 8) -> int:
    """Row bands per view for a view-sharded step: 1 when the ranks divide
    the views, else the smallest b in (2, 4, 8) with (n_views * b) % world
    == 0 and at least one tile row per band — so every rank renders the same
    number of (view, band) units (config 2's 10 views at 4 GPUs: 20 half
    views, 5 per rank; at 8 GPUs: 40 quarter views, 5 per rank)."""
    if world <= 1 or n_views % world == 0:
        return 1
    rows = (height + tile - 1) // tile
    for b in (2, 4, 8):
        if b <= max_split and b <= rows and (n_views * b) % world == 0:
            return b
    return 1


def shard_units(n_views: int, world: int, rank: int, height: int, tile: int = 16) -> list:
    """This rank's (view, y0, y1) render units.  Unbanded: views v -> rank
    v mod world (shard_views).  Banded: the (view, band) units in view-major
    order, cut into `world` equal contiguous runs (each rank gets a mix of
    bands, so systematic cost differences between image regions average
    out)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    b = view_bands(n_views, world, height, tile)
    if b == 1:
        return [(v, 0, height) for v in shard_views(n_views, world, rank)]
    rows = (height + tile - 1) // tile
    edges = [min(height, tile * (k * rows // b)) for k in range(b)] + [height]
    units = [(v, edges[k], edges[k + 1]) for v in range(n_views) for k in range(b)]
    per = len(units) // world
    return units[rank * per:(rank + 1) * per]


def shard_units_mixed(n_views: int, world: int, rank: int, height: int, tile: int = 16) -> list:
    """Whole views first, bands for the remainder: with n_views = q world + r,
    rank r' renders the q whole views r', r' + world, ... and the r leftover
    views are cut into b row bands (b in 2, 4, 8 with r b divisible by
    world) shared out evenly — fewer, larger units than banding every view
    (the target window at 8 ranks: 1 whole + 1 quarter view per rank instead
    of 5 quarter views).  Falls back to shard_units when no split exists."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    q, r = divmod(n_views, world)
    if r == 0:
        return [(v, 0, height) for v in shard_views(n_views, world, rank)]
    rows = (height + tile - 1) // tile
    for b in (2, 4, 8):
        if b <= rows and (r * b) % world == 0:
            edges = [min(height, tile * (k * rows // b)) for k in range(b)] + [height]
            rest = [(v, edges[k], edges[k + 1]) for v in range(q * world, n_views) for k in range(b)]
            per = len(rest) // world
            return [(v, 0, height) for v in range(rank, q * world, world)] + rest[rank * per:(rank + 1) * per]
    return shard_units(n_views, world, rank, height, tile)


class AllReduce:
    """The gradient exchange: in-place sum over the process group.  Called
    on the whole flat buffer it blocks the current stream on one all-reduce;
    `start` / `wait` split it into buckets (WindowEngine steps the Adam
    groups of bucket b while bucket b + 1 is still being reduced).  Each
    element is reduced once and the result broadcast, so every rank receives
    the same bits and the replicas stay identical; with two ranks the sum is
    a + b whichever way the buffer is cut, with more ranks the summation
    order (hence the last bit) may differ from a one-shot all-reduce's."""

    def __init__(self, group=None):
        self.group = group

    def __call__(self, flat: torch.Tensor) -> None:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group)

    def start(self, part: torch.Tensor):
        return dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.group, async_op=True)

    @staticmethod
    def wait(work) -> None:
        work.wait()          # NCCL: the current stream waits on the collective (no host sync)


def make_allreduce(group=None) -> Optional[Callable[[torch.Tensor], None]]:
    """The gradient exchange (None if not distributed or world size 1)."""
    if not dist.is_available() or not dist.is_initialized():
        return None
    if dist.get_world_size(group) == 1:
        return None
    return AllReduce(group)


def replicas_identical(t: torch.Tensor, group=None) -> bool:
    """Check (by max/min all-reduce of a checksum) that every rank holds the
    same tensor bits — the invariant the deterministic Adam keeps."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return True
    x = t.detach().reshape(-1).view(torch.int32) if t.dtype == torch.float32 else \
        t.detach().reshape(-1).view(torch.int64)
    s = (x.to(torch.int64) * (torch.arange(x.numel(), device=x.device, dtype=torch.int64) % 1021 + 1)).sum()
    lo, hi = s.clone().reshape(1), s.clone().reshape(1)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return bool(lo.item() == hi.item())


class ViewShardedWindow:
    """Multi-GPU WindowEngine: this rank's share of the keyframe views —
    whole views, and row bands of the leftover views when the ranks do not
    divide the views (shard_units_mixed)."""

    def __init__(self, arrays, cam, views_all: Sequence, settings, cfg=None, group=None, stream=None,
                 master: str = "f64", lanes: int = 1):
        from .optimize import OptimConfig, WindowEngine

        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.units = shard_units_mixed(len(views_all), world, rank, int(cam.height))
        self.mine = [u[0] for u in self.units]
        self.engine = WindowEngine(arrays, cam, [views_all[v] for v in self.mine], settings, cfg or OptimConfig(),
                                   n_views_total=len(views_all), stream=stream, master=master, lanes=lanes,
                                   bands=[(u[1], u[2]) for u in self.units])
        self.allreduce = make_allreduce(group)

    def observed_for(self, frames: Sequence[torch.Tensor]) -> list:
        """This rank's unit images from the full frames (indexed by view)."""
        return [frames[v][y0:y1].contiguous() for v, y0, y1 in self.units]

    def step(self, observed_mine: Sequence[torch.Tensor], timers: Optional[dict] = None, check: bool = False) -> None:
        """observed_mine: one image per unit (observed_for).  check=True
        syncs after the step and raises CapacityExceeded on every rank if
        any rank's render overflowed (else see check_capacity / finish)."""
        self.engine.step(observed_mine, allreduce=self.allreduce, timers=timers)
        if check:
            self.require_capacity()

    def check_capacity(self) -> bool:
        """True if no render on ANY rank overflowed since the last check
        (syncs; one MAX all-reduce of the ranks' sticky flags)."""
        over = torch.tensor([0 if self.engine.check_capacity(clear=False) else 1],
                            dtype=torch.int32, device=self.engine.grads.flat.device)
        if self.allreduce is not None:
            dist.all_reduce(over, op=dist.ReduceOp.MAX)
        return not bool(over.item())

    def require_capacity(self) -> None:
        from .errors import CapacityExceeded
        if not self.check_capacity():
            raise CapacityExceeded("a rank's render overflowed its intersection capacity: regrow and redo the step")

    def finish(self) -> None:
        self.require_capacity()
        self.engine.finish()


# ---- fused optimiser step over NVLink peer memory ---------------------------------

def shard_range(n: int, world: int, rank: int) -> tuple:
    """Gaussians [lo, hi) whose optimiser step `rank` owns (contiguous shards)."""
    per = (n + world - 1) // world
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def adam_peer_step(replicas: Sequence, grads: Sequence[torch.Tensor], touched: Sequence[torch.Tensor], rank: int,
                   lo: int, hi: int, adam, stream=None) -> None:
    """lsb_adam_peer_step: sum the ranks' gradient buffers (rank order) for
    the Gaussians [lo, hi), step them with `adam`'s moments (device step
    counter, like AdamState.apply_dev) and store the new parameters into
    every replica.  replicas / grads / touched are per-rank views (peer
    memory in a multi-process run; plain device tensors to simulate ranks on
    one GPU)."""
    import ctypes

    from . import _lib
    from .optimize import adam_cfg, bias_correction_table

    G = len(replicas)
    if adam.step_dev is None:
        adam.ibc = torch.from_numpy(bias_correction_table(adam.cfg.beta1, adam.cfg.beta2)).to(adam.m.device)
        adam.step_dev = torch.full((1,), adam.step, dtype=torch.int64, device=adam.m.device)
    adam.step += 1
    c = adam_cfg(adam.cfg, adam.step)
    P = (_lib.Params * G)(*[r.params() for r in replicas])
    gp = (ctypes.c_void_p * G)(*[g.data_ptr() for g in grads])
    tp = (ctypes.c_void_p * G)(*[t.data_ptr() for t in touched])
    _lib.check(_lib.load().lsb_adam_peer_step(
        P, G, int(rank), gp, int(lo), int(hi), ctypes.c_void_p(adam.m.data_ptr()), ctypes.c_void_p(adam.v.data_ptr()),
        tp, ctypes.byref(c), ctypes.c_void_p(adam.ibc.data_ptr()), int(adam.ibc.shape[0]),
        ctypes.c_void_p(adam.step_dev.data_ptr()), _lib.stream_ptr(stream)), "adam_peer")


class PeerExchange:
    """The view-sharded step's gradient exchange + optimiser as ONE kernel
    over NVLink peer memory (instead of an NCCL all-reduce followed by Adam on
    every rank): the window parameters, the flat gradient buffer and the
    touched flags live in torch symmetric memory, so every rank can load its
    peers' gradients and store into their parameter replicas.  Per step:
    device barrier (all ranks' gradients complete) -> lsb_adam_peer_step on
    this rank's shard of Gaussians (reduce-scatter + Adam + all-gather fused)
    -> device barrier (all stores landed).  Replicas stay bit-identical.
    Traffic per rank: (G-1)/G of the gradient rows in, (G-1)/G of the
    parameter rows out; Adam runs on n/G Gaussians instead of n."""

    def __init__(self, engine, group=None):
        import torch.distributed._symmetric_memory as symm

        from .raster import ParamGradients

        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        if self.world > 8:
            raise ValueError("the peer step addresses at most 8 ranks")
        self.engine = engine
        self._handles = []

        def sym(t):
            s = symm.empty(t.shape, dtype=t.dtype, device=t.device)
            s.copy_(t)
            h = symm.rendezvous(s, self.group)
            self._handles.append(h)
            peers = [h.get_buffer(q, tuple(t.shape), t.dtype) for q in range(self.world)]
            return s, h, peers

        arr = engine.arrays
        peer_fields = {}
        for f in ("means", "rots", "scales", "opacities", "shs"):
            s, _, peers = sym(getattr(arr, f))
            setattr(arr, f, s)
            peer_fields[f] = peers
        flat, self._gh, gpeers = sym(engine.grads.flat)
        engine.grads = ParamGradients.from_flat(flat, len(arr), int(arr.shs.shape[1]))
        tflags, _, tpeers = sym(engine.adam.touched)
        engine.adam.touched = tflags
        from types import SimpleNamespace
        self.replicas = [SimpleNamespace(params=(lambda q=q: _peer_params(arr, peer_fields, q))) for q in
                         range(self.world)]
        self.grads = gpeers
        self.touched = tpeers
        self.lo, self.hi = shard_range(len(arr), self.world, self.rank)

    def step(self, stream=None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self._gh.barrier(channel=0)
            adam_peer_step(self.replicas, self.grads, self.touched, self.rank, self.lo, self.hi, self.engine.adam, s)
            self._gh.barrier(channel=1)


def _peer_params(arr, peer_fields, q):
    from . import _lib
    f = peer_fields
    return _lib.Params(f["means"][q].data_ptr(), f["rots"][q].data_ptr(), f["scales"][q].data_ptr(),
                       f["opacities"][q].data_ptr(), f["shs"][q].data_ptr(), len(arr), int(arr.shs.shape[1]),
                       1 if arr.dtype == torch.float64 else 0)
