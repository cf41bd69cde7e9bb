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


# ------------------------------------------------- output-block sharding ----
# The weight-memory-saving layout (north_star "output-block sharded BLAST"): rank r owns a
# contiguous range of output blocks k (Y = [Y_1 ... Y_b2], Y_k = X W_{:,k}) and only
# the factors that range needs -- BLAST U[k], S[:, k] (V replicated; S1 recomputed on every rank);
# Monarch U[k] and the V rows m(rho, k); low rank the U columns of the range.  Each rank computes
# its column block of Y with the single-GPU kernels; an all-gather along o (NCCL over NVLink on
# GPUs) assembles Y.  The factor slicing below is pure indexing (no method arithmetic).

def shard_blocks(b2: int, rank: int, world: int) -> tuple[int, int]:
    """Output-block range [k0, k1) of `rank` (contiguous, balanced; may be empty if world > b2)."""
    return shard_rows(b2, rank, world)


def blast_local_factors(V, S, U, k0: int, k1: int):
    """BLAST factors for output blocks [k0, k1): V [b1,p,r] (all), S[:, k0:k1], U[k0:k1]."""
    return V, S[:, k0:k1].contiguous(), U[k0:k1].contiguous()


def monarch_local_factors(V, U, b2: int, r_blk: int, k0: int, k1: int, v_layout: int = 0):
    """Monarch factors for output blocks [k0, k1) as a (b1, k1-k0) Monarch in the same V layout:
    rows m(rho, k) of every V[l] (b2-fastest m = rho*b2 + k, r'-fastest m = k*r' + rho, PAPER.md
    L194) and U[k0:k1]."""
    b1, _, p = V.shape
    Vb = V.reshape(b1, r_blk, b2, p) if v_layout == 0 else V.reshape(b1, b2, r_blk, p)
    if v_layout == 0:
        Vl = Vb[:, :, k0:k1, :].reshape(b1, r_blk * (k1 - k0), p)
    else:
        Vl = Vb[:, k0:k1, :, :].reshape(b1, (k1 - k0) * r_blk, p)
    return Vl.contiguous(), U[k0:k1].contiguous()


def lowrank_local_factors(V, U, c0: int, c1: int):
    """Low-rank factors for output columns [c0, c1): V (all), U[:, c0:c1]."""
    return V, U[:, c0:c1].contiguous()


def gather_columns(y_local: torch.Tensor, widths: list[int]) -> torch.Tensor:
    """All-gather column blocks (rank order; `widths` per rank, possibly 0) into [n, sum(widths)]."""
    world = dist.get_world_size()
    n = y_local.shape[0]
    wmax = max(widths)
    pad = torch.zeros((n, wmax), dtype=y_local.dtype, device=y_local.device)
    pad[:, : y_local.shape[1]] = y_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:, :w] for p, w in zip(parts, widths)], dim=1)


def output_sharded_forward(local_fn, n_blocks: int, block_width: int, gather: bool = True) -> torch.Tensor:
    """Run `local_fn(k0, k1)` (this rank's [n, (k1-k0)*block_width] column block) and optionally
    all-gather the full [n, n_blocks*block_width] output."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    k0, k1 = shard_blocks(n_blocks, rank, world)
    y = local_fn(k0, k1)
    if not gather or world == 1:
        return y
    widths = [(hi - lo) * block_width for lo, hi in (shard_blocks(n_blocks, r, world) for r in range(world))]
    return gather_columns(y, widths)
