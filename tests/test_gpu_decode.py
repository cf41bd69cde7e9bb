"""GPU parity of the small-token (decode) path: n_tok <= 16 runs the
weight-streaming tensor-core decode stages (csrc/blr_decode_tc.cuh: TMA weight ring, mma.sync,
K splits reduced in-cluster, BLAST S2 in S1's cluster epilogue) with fp32 intermediates staged as
bf16 hi + lo pairs.  Same tolerance as the prefill path (north_star); the tcgen05 path is also
forced at these sizes (BLR_DECODE=0) so both stay covered."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import synth
from tests.parity import assert_parity, to64

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(autouse=True)
def _force_decode(monkeypatch):
    """Every test here runs the decode kernels at all n <= 16 (the library's default uses them
    only where they measured faster); test_small_n_on_the_tcgen05_path overrides this."""
    monkeypatch.setenv("BLR_DECODE", "1")

NS = [1, 3, 8, 16]


def _lr(lib, n, i, o, r, seed=11):
    X = synth.make_x(n, i, seed=seed)
    V, U = synth.lowrank_factors(i, o, r, seed=seed)
    Y = lib.lowrank_matmul(X.to(DEV), V.to(DEV), U.to(DEV))
    torch.cuda.synchronize()
    return Y, orc.lowrank_forward(to64(X), to64(V), to64(U))


def _mon(lib, n, b1, b2, rp, p, q, layout, seed=12):
    X = synth.make_x(n, b1 * p, seed=seed)
    V, U = synth.monarch_factors(b1 * p, b2 * q, b1, b2, rp, seed=seed)
    Y = lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, v_layout=layout)
    torch.cuda.synchronize()
    return Y, orc.monarch_forward(to64(X), to64(V), to64(U), b1, b2, layout)


def _blast(lib, n, b1, b2, r, p, q, seed=13):
    X = synth.make_x(n, b1 * p, seed=seed)
    V, S, U = synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=seed)
    Y = lib.blast_matmul(X.to(DEV), V.to(DEV), S.to(DEV), U.to(DEV))
    torch.cuda.synchronize()
    return Y, orc.blast_forward(to64(X), to64(V), to64(S), to64(U))


@pytest.mark.parametrize("n", NS)
@pytest.mark.parametrize("i,o,r", [(64, 40, 16), (768, 3072, 192), (3072, 768, 192), (4096, 11008, 1488)])
def test_decode_lowrank(cuda_lib, n, i, o, r):
    Y, ref = _lr(cuda_lib, n, i, o, r)
    assert_parity(Y, ref, f"LR decode {n,i,o,r}")


@pytest.mark.parametrize("n", NS)
@pytest.mark.parametrize("b1,b2,rp,p,q", [(2, 3, 8, 16, 24), (4, 4, 48, 192, 768), (16, 16, 96, 256, 688),
                                          (16, 16, 96, 688, 256)])
@pytest.mark.parametrize("layout", [orc.B2_FASTEST, orc.RPRIME_FASTEST])
def test_decode_monarch(cuda_lib, n, b1, b2, rp, p, q, layout):
    Y, ref = _mon(cuda_lib, n, b1, b2, rp, p, q, layout)
    assert_parity(Y, ref, f"Monarch decode {n,b1,b2,rp,p,q} layout={layout}")


@pytest.mark.parametrize("n", NS)
@pytest.mark.parametrize("b1,b2,r,p,q", [(1, 1, 16, 8, 8), (3, 2, 24, 40, 56), (6, 6, 192, 128, 512),
                                         (16, 16, 1488, 256, 688), (16, 16, 1488, 688, 256),
                                         (11, 3, 40, 16, 24),      # b1 = 11: no cluster split -> S1, S2, S3
                                         (2, 2, 64, 1040, 64),     # p > 1024: S1 with a K split, then S2
                                         (12, 5, 72, 64, 40)])     # 6-CTA cluster x 2 blocks, b2 % 6 != 0
def test_decode_blast(cuda_lib, n, b1, b2, r, p, q):
    Y, ref = _blast(cuda_lib, n, b1, b2, r, p, q)
    assert_parity(Y, ref, f"BLAST decode {n,b1,b2,r,p,q}")


@pytest.mark.parametrize("w,s", [(64, 1), (64, 3), (64, 8), (128, 2), (128, 6), (256, 4), (256, 7)])
def test_decode_forced_plans(cuda_lib, monkeypatch, w, s):
    """Every tile width W and cluster (K split) size S of the decode kernel against the oracle: the
    planner's choice is forced for both launches of a low-rank layer with K = 1000 (every S listed
    is a valid split of 1000 rows into W's row granularity, the last split ragged) and N = 1000 /
    1040 (ragged last tile)."""
    monkeypatch.setenv("BLR_DTC_W", str(w))
    monkeypatch.setenv("BLR_DTC_S", str(s))
    for n in (1, 13):
        Y, ref = _lr(cuda_lib, n, 1000, 1040, 1000)
        assert_parity(Y, ref, f"LR decode W={w} S={s} n={n}")


@pytest.mark.parametrize("n", [17, 100, 333])
def test_decode_token_chunks(cuda_lib, monkeypatch, n):
    """n > 16 on the weight-streaming kernels (BLR_DECODE_MAXN): independent 16-row token chunks,
    the last one ragged, for all three methods (incl. the BLAST cluster S2 and a K split)."""
    monkeypatch.delenv("BLR_DECODE", raising=False)
    monkeypatch.setenv("BLR_DECODE_MAXN", "4096")
    Y, ref = _lr(cuda_lib, n, 3072, 768, 192)
    assert_parity(Y, ref, f"LR chunks n={n}")
    Y, ref = _blast(cuda_lib, n, 6, 6, 192, 128, 512)
    assert_parity(Y, ref, f"BLAST chunks n={n}")
    Y, ref = _blast(cuda_lib, n, 11, 3, 40, 16, 24)
    assert_parity(Y, ref, f"BLAST (S1, S2, S3) chunks n={n}")
    Y, ref = _mon(cuda_lib, n, 4, 4, 48, 192, 768, orc.RPRIME_FASTEST)
    assert_parity(Y, ref, f"Monarch chunks n={n}")


@pytest.mark.parametrize("n", [1, 16])
def test_small_n_on_the_tcgen05_path(cuda_lib, monkeypatch, n):
    """BLR_DECODE=0 keeps small n on the prefill kernels: both paths meet the same bar."""
    monkeypatch.setenv("BLR_DECODE", "0")
    Y, ref = _lr(cuda_lib, n, 768, 3072, 192)
    assert_parity(Y, ref, "LR tcgen05 small n")
    Y, ref = _blast(cuda_lib, n, 6, 6, 192, 128, 512)
    assert_parity(Y, ref, "BLAST tcgen05 small n")
    Y, ref = _mon(cuda_lib, n, 4, 4, 48, 192, 768, orc.B2_FASTEST)
    assert_parity(Y, ref, "Monarch tcgen05 small n")


def test_decode_deterministic_and_row_independent(cuda_lib):
    """Split-K partials are reduced in a fixed order (no atomics): bitwise run-to-run equal, and
    each row's output does not depend on the other rows present."""
    n, i, o, r = 16, 4096, 11008, 1488
    X = synth.make_x(n, i, seed=21).to(DEV)
    V, U = [t.to(DEV) for t in synth.lowrank_factors(i, o, r, seed=21)]
    Y1 = cuda_lib.lowrank_matmul(X, V, U)
    Y2 = cuda_lib.lowrank_matmul(X, V, U)
    Y3 = cuda_lib.lowrank_matmul(X[5:6].contiguous(), V, U)
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    assert torch.equal(Y1[5:6], Y3)


def test_decode_monarch_identity_blocks_bit_exact(cuda_lib):
    """Identity blocks make Monarch a permutation: the decode path is bit-exact too."""
    b1, b2, rp = 3, 2, 16
    p, q = rp * b2, b1 * rp
    V = torch.stack([torch.eye(rp * b2, p) for _ in range(b1)]).to(torch.bfloat16)
    U = torch.stack([torch.eye(q, b1 * rp) for _ in range(b2)]).to(torch.bfloat16)
    X = synth.make_x(7, b1 * p, seed=5)
    for layout in (orc.B2_FASTEST, orc.RPRIME_FASTEST):
        Y = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, v_layout=layout).cpu()
        ref = orc.monarch_forward(to64(X), to64(V), to64(U), b1, b2, layout)
        assert np.array_equal(to64(Y), ref), layout
