"""Batch sharding across ranks (one process per GPU).

The DiffMPC solve has no exchange step: problems are independent, so
rank r solves the contiguous slice [r*B/W, (r+1)*B/W) with no data-path collective.
Outputs can be all-gathered for verification (untimed). Works with any
torch.distributed backend (NCCL on the B200 box, gloo in the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced partition; the first B % world ranks get one extra problem."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(B, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard(t, rank: int, world: int):
    lo, hi = shard_range(t.shape[0], rank, world)
    return t[lo:hi]


def all_gather_batch(t: torch.Tensor, B: int, group=None) -> torch.Tensor:
    """Reassemble a batch-sharded tensor on every rank (uneven shards are padded)."""
    world = dist.get_world_size(group)
    sizes = [shard_range(B, r, world) for r in range(world)]
    mx = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sizes)], dim=0)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a scalar over ranks (device timings are reported as the max over ranks)."""
    t = torch.tensor([float(value)], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
