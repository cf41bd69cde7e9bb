"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no products, sums, permutations of the BLR
forward); it only draws seeded random tensors with the shapes and scales of the paper's
workloads (Table 3) and rounds them once to bf16 (RNE), which both sides
then consume (DESIGN.md §4 "input recipe").

Scales (fan-in per stage so every stage has unit variance):
  X ~ N(0, 1)
  low-rank  V ~ N(0, 1/i),  U ~ N(0, 1/r)
  Monarch   V ~ N(0, 1/p),  U ~ N(0, 1/(b1 r'))
  BLAST     V ~ N(0, 1/p),  S ~ N(0, 1/b1),  U ~ N(0, 1/r)
Seeds: seed*1000003 + {X:1, V:2, S:3, U:4} + 16*layer_id.
"""
from __future__ import annotations

import math

import torch

_TAG = {"X": 1, "V": 2, "S": 3, "U": 4}


def _seed(seed: int, tag: str, layer_id: int) -> int:
    return int(seed) * 1000003 + _TAG[tag] + 16 * int(layer_id)


def randn_bf16(shape, std: float, seed: int, device="cpu") -> torch.Tensor:
    """N(0, std^2) drawn in fp32 with a seeded generator, rounded RNE to bf16."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    t = torch.randn(*shape, generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        t.mul_(std)
    return t.to(torch.bfloat16)


def make_x(n: int, i: int, seed: int = 0, layer_id: int = 0, device="cpu",
           outliers: int = 0, outlier_scale: float = 20.0) -> torch.Tensor:
    """Activations X [n, i] ~ N(0,1) in bf16.  ``outliers`` > 0 multiplies that many evenly
    spaced input channels by ``outlier_scale`` and then rescales every channel so the expected
    squared row norm stays i (outlier channels stay ``outlier_scale`` x the others; the layer's
    output keeps the recipe's unit variance).  Parity-only stress variant."""
    if not outliers:
        return randn_bf16((n, i), 1.0, _seed(seed, "X", layer_id), device)
    g = torch.Generator(device=device)
    g.manual_seed(_seed(seed, "X", layer_id))
    x = torch.randn(n, i, generator=g, device=device, dtype=torch.float32)
    idx = torch.linspace(0, i - 1, outliers, device=x.device).round().long()
    x[:, idx] *= outlier_scale
    x *= (i / (i - outliers + outliers * outlier_scale ** 2)) ** 0.5
    return x.to(torch.bfloat16)


def lowrank_factors(i: int, o: int, r: int, seed: int = 0, layer_id: int = 0, device="cpu"):
    """V [i, r], U [r, o] (PAPER.md L36 storage)."""
    V = randn_bf16((i, r), 1.0 / math.sqrt(i), _seed(seed, "V", layer_id), device)
    U = randn_bf16((r, o), 1.0 / math.sqrt(r), _seed(seed, "U", layer_id), device)
    return V, U


def monarch_factors(i: int, o: int, b1: int, b2: int, r_blk: int, seed: int = 0,
                    layer_id: int = 0, device="cpu"):
    """V [b1, r'*b2, p], U [b2, q, b1*r'] (PAPER.md L59 storage)."""
    p, q = i // b1, o // b2
    V = randn_bf16((b1, r_blk * b2, p), 1.0 / math.sqrt(p), _seed(seed, "V", layer_id), device)
    U = randn_bf16((b2, q, b1 * r_blk), 1.0 / math.sqrt(b1 * r_blk), _seed(seed, "U", layer_id), device)
    return V, U


def blast_factors(i: int, o: int, b1: int, b2: int, r: int, seed: int = 0, layer_id: int = 0,
                  device="cpu"):
    """V [b1, p, r], S [b1, b2, r], U [b2, r, q] (PAPER.md L81 storage)."""
    p, q = i // b1, o // b2
    V = randn_bf16((b1, p, r), 1.0 / math.sqrt(p), _seed(seed, "V", layer_id), device)
    S = randn_bf16((b1, b2, r), 1.0 / math.sqrt(b1), _seed(seed, "S", layer_id), device)
    U = randn_bf16((b2, r, q), 1.0 / math.sqrt(r), _seed(seed, "U", layer_id), device)
    return V, S, U
