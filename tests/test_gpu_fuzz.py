"""Seeded shape fuzz of all three formats against the fp64 oracle.

Shapes are drawn so that every planner branch is reached with the round-2 defaults (CTA pairs from
256 tokens, streamed weights, slab-view MN-major weights, 256-wide pair tiles, cooperative stores):
odd and even numbers of 128-token tiles (a pair's second tile past n_tok), ragged token / K / N tails,
b1 != b2, r below and above 128 (compensated and plain intermediates), BLAST fused (b1 r <= 512) and
split paths, both Monarch V layouts, and the small-n weight-streaming path.  Each case checks a
seeded sample of rows (always the first and last) within north_star's tolerance, and the K-major
BLAST entry point is held bitwise to the paper layout wherever it applies."""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import synth
from tests.parity import assert_parity, sample_rows, to64
from tests.test_fp8_budget import FP8_ELEM, FP8_FROB

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda")
SCALE = int(os.environ.get("BLR_FUZZ_SCALE", "1"))   # longer one-off hunts: BLR_FUZZ_SCALE=10
SEED = int(os.environ.get("BLR_FUZZ_SEED", "0"))


BIG = os.environ.get("BLR_FUZZ_BIG") == "1"   # one-off hunts at larger token counts / widths


def _cases(method, count, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.choice([1, 5, 16, 100, 200, 384, 640, 1000, 1300, 2500] + ([4100, 6000, 9000] if BIG else [])))
        if method == "lowrank":
            i, o = (int(8 * rng.integers(8, 512 if BIG else 160)) for _ in range(2))
            r = int(8 * rng.integers(2, 40))
            out.append((n, i, o, r, 1, 1, 0))
        elif method == "monarch":
            b1, b2 = int(rng.integers(1, 9)), int(rng.integers(1, 9))
            p, q = (int(8 * rng.integers(2, 64 if BIG else 24)) for _ in range(2))
            rb = int(8 * rng.integers(1, 13 if BIG else 5))
            out.append((n, b1 * p, b2 * q, rb, b1, b2, int(rng.integers(0, 2))))
        else:
            b1, b2 = int(rng.integers(1, 17)), int(rng.integers(1, 17))
            p, q = (int(8 * rng.integers(2, 64 if BIG else 24)) for _ in range(2))
            r = int(8 * rng.integers(2, 160 if BIG else 48))
            out.append((n, b1 * p, b2 * q, r, b1, b2, 0))
    return out


@pytest.mark.parametrize("case", _cases("lowrank", 12 * SCALE, 101 + SEED))
def test_fuzz_lowrank(cuda_lib, case):
    n, i, o, r, _, _, _ = case
    X = synth.make_x(n, i, seed=n + i)
    V, U = synth.lowrank_factors(i, o, r, seed=o + r)
    Y = cuda_lib.lowrank_matmul(X.to(DEV), V.to(DEV), U.to(DEV))
    torch.cuda.synchronize()
    rows = sample_rows(n, 24)
    ref = orc.lowrank_forward(to64(X[rows]), to64(V), to64(U))
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"lowrank {case}")


@pytest.mark.parametrize("case", _cases("monarch", 12 * SCALE, 202 + SEED))
def test_fuzz_monarch(cuda_lib, case):
    n, i, o, rb, b1, b2, layout = case
    X = synth.make_x(n, i, seed=n + i)
    V, U = synth.monarch_factors(i, o, b1, b2, rb, seed=o + rb)
    # (the same random tensor read in either composite order of V's middle dim, PAPER.md L194-195;
    #  the oracle reads it the same way)
    vl = cuda_lib.RPRIME_FASTEST if layout else cuda_lib.B2_FASTEST
    Y = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, v_layout=vl)
    torch.cuda.synchronize()
    rows = sample_rows(n, 24)
    ref = orc.monarch_forward(to64(X[rows]), to64(V), to64(U), b1, b2, vl)
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"monarch {case}")
    # the transposed output order is the same values permuted, bit for bit
    q = o // b2
    Yt = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, v_layout=vl,
                                 out_order=cuda_lib.OUT_TRANSPOSED)
    torch.cuda.synchronize()
    assert torch.equal(Yt.view(n, q, b2).transpose(1, 2).reshape(n, o), Y), f"monarch transposed {case}"


# regression: odd b1 with b2 <= 2 made the tensor-core S2 zero a pad plane past its smem layout
# (an illegal address for small b2; found by BLR_FUZZ_SCALE=10 BLR_FUZZ_SEED=7)
REGRESSION = [(640, 528, 64, 264, 11, 2, 0), (640, 528, 48, 264, 11, 1, 0), (300, 840, 64, 256, 15, 2, 0)]


@pytest.mark.parametrize("case", _cases("blast", 16 * SCALE, 303 + SEED) + REGRESSION)
def test_fuzz_blast(cuda_lib, case):
    n, i, o, r, b1, b2, _ = case
    X = synth.make_x(n, i, seed=n + i).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(i, o, b1, b2, r, seed=o + r)]
    Y = cuda_lib.blast_matmul(X, V, S, U)
    torch.cuda.synchronize()
    rows = sample_rows(n, 24)
    ref = orc.blast_forward(to64(X[rows].cpu()), to64(V), to64(S), to64(U))
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"blast {case}")
    # FP8 first-stage intermediate: its own derived contract (tests/test_fp8_budget.py)
    Y8 = cuda_lib.blast_matmul(X, V, S, U, fp8_intermediate=True)
    torch.cuda.synchronize()
    g = to64(Y8[torch.as_tensor(rows, device=DEV)])
    nref = np.linalg.norm(ref)
    if nref > 0:
        assert np.linalg.norm(g - ref) / nref <= FP8_FROB, f"fp8z {case}"
    assert np.all(np.abs(g - ref) <= FP8_ELEM * (1.0 + np.abs(ref))), f"fp8z elem {case}"
    # K-major storage: same function, bitwise, wherever the entry point applies
    Vt, Ut = cuda_lib.blast_kmajor_factors(V, U)
    try:
        Yk = cuda_lib.blast_matmul(X, Vt, S, Ut, kmajor=True)
    except cuda_lib.BLRError:
        return  # outside the split tensor-core path: refused before any launch
    torch.cuda.synchronize()
    assert torch.equal(Yk, Y), f"kmajor {case}"
