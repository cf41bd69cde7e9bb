"""Closed-form parameter / FLOP / byte counts and the roofline (§2, §2.2, Table 2).

FLOP convention: 2 FLOP per multiply-add (Table 2; reading R6).
Bytes: bf16 = 2 bytes per element.

* ``table2_bytes``  -- the paper's memory model, including the underlined intermediate terms
  2nr (LR), 4bnr (Monarch), 8bnr (BLAST) of the unfused PyTorch baselines.
* ``fused_bytes``   -- the algorithmic bytes of a fused implementation that never writes the
  rank-r intermediate: 2 (n i + params + n o) -- Table 2 minus the underlined terms (with the
  exact parameter count for BLAST, r(i + o + b1 b2)).
"""
from __future__ import annotations

import json
import os

BF16 = 2


def params(method: str, i: int, o: int, r: int = 0, b1: int = 1, b2: int = 1) -> int:
    """Parameter counts of PAPER.md §2.1: dense i*o (L34); LR r(i+o) (L36);
    Monarch b1 b2 r'(p+q) (L50) with r' = r/b2; BLAST r(i + o + b1 b2) (L81, reading R1)."""
    if method == "dense":
        return i * o
    if method == "lowrank":
        return r * (i + o)
    if method == "monarch":
        rp = r // b2
        p, q = i // b1, o // b2
        return b1 * b2 * rp * (p + q)
    if method == "blast":
        return r * (i + o + b1 * b2)
    raise ValueError(method)


def flops(method: str, n: int, i: int, o: int, r: int = 0, b1: int = 1, b2: int = 1) -> int:
    """Table 2 FLOP, 2 FLOP per MAC; BLAST uses b1*b2 for b^2."""
    if method == "dense":
        return 2 * n * i * o
    if method in ("lowrank", "monarch"):
        return 2 * n * r * (i + o)
    if method == "blast":
        return 2 * n * r * (i + o + b1 * b2)
    raise ValueError(method)


def table2_bytes(method: str, n: int, i: int, o: int, r: int = 0, b: int = 1) -> int:
    """Table 2 memory traffic, symmetric b1 = b2 = b."""
    if method == "dense":
        return BF16 * (n * i + i * o + n * o)
    if method == "lowrank":
        return BF16 * (n * i + i * r + r * o + n * o + 2 * n * r)
    if method == "monarch":
        return BF16 * (n * i + i * r + r * o + n * o + 4 * b * n * r)
    if method == "blast":
        return BF16 * (n * i + i * r + r * o + r * b * b + n * o + 8 * b * n * r)
    raise ValueError(method)


def fused_bytes(method: str, n: int, i: int, o: int, r: int = 0, b1: int = 1, b2: int = 1) -> int:
    """Algorithmic bytes with the intermediate kept on chip: read X and the factors once,
    write Y once (Table 2 without the underlined terms)."""
    return BF16 * (n * i + params(method, i, o, r, b1, b2) + n * o)


def intensity(fl: int, by: int) -> float:
    """Arithmetic intensity alpha = FLOP / byte."""
    return fl / by


def layer_counts(layer, n: int) -> dict:
    """FLOP and fused algorithmic bytes of one configs.Layer at n tokens."""
    fl = flops(layer.method, n, layer.i, layer.o, layer.r, layer.b1, layer.b2)
    by = fused_bytes(layer.method, n, layer.i, layer.o, layer.r, layer.b1, layer.b2)
    return {"flops": fl, "bytes": by}


# ------------------------------------------------------------------------------------ peaks -----
# B200_PROFILING.md fallback, used only when MEASURED_PEAKS.json is absent ("of fallback").
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks(repo_root: str | None = None) -> dict:
    root = repo_root or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        d["source"] = "measured"
        return d
    except (OSError, ValueError):
        d = dict(FALLBACK_PEAKS)
        d["source"] = "fallback"
        return d


def roofline_time_s(fl: int, by: int, peaks: dict, sustained: bool = False) -> float:
    """t_roof = max(F / P_tc, B / BW)."""
    tc = peaks["bf16_tflops_sustained" if sustained else "bf16_tflops"] * 1e12
    bw = peaks["hbm_gbs"] * 1e9
    return max(fl / tc, by / bw)
