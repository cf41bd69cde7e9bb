"""Token-row sharding across ranks (one process per GPU) -- host logic only.

The BLR forward is row-independent (Y = X W, row t of Y depends only on row t of X),
so the data path needs no collective: each rank multiplies its rows with replicated factors.
This module provides the shard ranges, the max-over-ranks step time used by bench.py, and an
optional all-gather of Y for callers that need the full output (NCCL on GPUs; gloo in tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row range [lo, hi) of rank `rank` (sizes differ by at most one)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (step time) over the default process group."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(y_local: torch.Tensor, n: int) -> torch.Tensor:
    """All-gather row shards (rank order) into the full [n, o] output on every rank."""
    world = dist.get_world_size()
    o = y_local.shape[1]
    sizes = [shard_rows(n, r, world) for r in range(world)]
    maxrows = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((maxrows, o), dtype=y_local.dtype, device=y_local.device)
    pad[: y_local.shape[0]] = y_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sizes)], dim=0)


def sharded_forward(fn, x_full: torch.Tensor, gather: bool = True) -> torch.Tensor:
    """Apply a row-wise layer `fn` to this rank's rows of x_full; optionally gather Y."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    n = x_full.shape[0]
    lo, hi = shard_rows(n, rank, world)
    y = fn(x_full[lo:hi].contiguous())
    return gather_rows(y, n) if (gather and world > 1) else y
