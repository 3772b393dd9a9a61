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


def make_allreduce(group=None) -> Optional[Callable[[torch.Tensor], None]]:
    """The gradient exchange: in-place sum over the process group (None if
    not distributed or world size 1)."""
    if not dist.is_available() or not dist.is_initialized():
        return None
    if dist.get_world_size(group) == 1:
        return None

    def allreduce(flat: torch.Tensor) -> None:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)

    return allreduce


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
    """Multi-GPU WindowEngine: this rank's share of the keyframe views."""

    def __init__(self, arrays, cam, views_all: Sequence, settings, cfg=None, group=None, stream=None,
                 master: str = "f64"):
        from .optimize import OptimConfig, WindowEngine

        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.mine = shard_views(len(views_all), world, rank)
        self.engine = WindowEngine(arrays, cam, [views_all[v] for v in self.mine], settings, cfg or OptimConfig(),
                                   n_views_total=len(views_all), stream=stream, master=master)
        self.allreduce = make_allreduce(group)

    def step(self, observed_mine: Sequence[torch.Tensor], timers: Optional[dict] = None) -> None:
        self.engine.step(observed_mine, allreduce=self.allreduce, timers=timers)

    def finish(self) -> None:
        self.engine.finish()
