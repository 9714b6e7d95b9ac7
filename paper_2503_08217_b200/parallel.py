"""Multi-GPU plumbing: one process per GPU, views sharded, Gaussians replicated.

The per-view path is independent across views, so a batch is
split into contiguous blocks of views per rank (same-time views stay together
and share K1's compaction).  The only exchange is the point-life merge at the
end of a sweep: Eq.5 is l_s = min(l_s, t), l_e = max(l_e, t), an
order-independent reduction, so replicas merge exactly with one all-reduce MAX
over float[2N] after negating l_s (s3r_life_flip), then every rank commits
(Eq.6) identically.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import torch
import torch.distributed as dist


def shard_bounds(n_items: int, rank: int, world: int):
    """Contiguous block [lo, hi) of n_items for `rank` (sizes differ by <= 1)."""
    base, rem = divmod(n_items, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi


def shard_views(views: Sequence, rank: int, world: int):
    lo, hi = shard_bounds(len(views), rank, world)
    return list(views[lo:hi])


def merge_life(life: torch.Tensor, flip: Callable[[torch.Tensor], None],
               group: Optional[dist.ProcessGroup] = None) -> None:
    """In-place merge of the replicated point life over all ranks of `group`.

    life: (N, 2) float32 (l_s, l_e), contiguous.  flip(life) must negate column
    0 in place (the CUDA path passes Context.life_flip; CPU tests pass their
    own).  After the call every rank holds (min_r l_s, max_r l_e)."""
    flip(life)
    dist.all_reduce(life, op=dist.ReduceOp.MAX, group=group)
    flip(life)


def allreduce_grads(grads: dict, group: Optional[dist.ProcessGroup] = None) -> None:
    """Config 5 with views sharded: sum the per-Gaussian gradients of every
    rank's views (one all-reduce SUM per tensor; fp32 summation order differs
    from one process, so the result agrees to rounding, not bit for bit).
    The pose gradient ("table": per view) belongs to the rank owning the view
    and is not reduced."""
    for k, g in grads.items():
        if k != "table":
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group)
