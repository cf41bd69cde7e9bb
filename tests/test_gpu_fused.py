"""GPU parity of the one-launch low-rank / Monarch layer (csrc/blr_fused.cuh: S1 and S3 of a token
tile in one CTA, the rank-r intermediate rounded once to bf16 into shared memory, never to HBM)
against the fp64 oracle, with BLR_FUSED=1 forcing the path and BLR_FUSED=0 the two-kernel path.

Tolerance (BASELINE.json north_star): relative Frobenius <= 5e-3 and |err| <= 1e-2 (1 + |ref|);
identity-block Monarch (a pure permutation) bit for bit.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import synth
from tests.parity import assert_parity, sample_rows, to64

pytestmark = pytest.mark.gpu
DEV = "cuda"

LR_FUSED = [  # (n, i, o, r): the fused envelope is 128 <= r <= 256, r % 64 == 0
    (1000, 768, 3072, 192),   # GPT2-S c_fc, ragged tail, S3 split in parts
    (300, 3072, 768, 192),    # contracting layer (default: two kernels; forced fused here)
    (513, 2048, 2048, 256),   # Llama-3.2-1B q/o rank
    (129, 520, 1000, 128),    # K1 % 64 != 0, N2 % 16 != 0
    (256, 64, 200, 128),      # single K block in S1
]


@pytest.mark.parametrize("n,i,o,r", LR_FUSED)
def test_lowrank_fused_parity(cuda_lib, monkeypatch, n, i, o, r):
    monkeypatch.setenv("BLR_FUSED", "1")
    X = synth.make_x(n, i, seed=21)
    V, U = synth.lowrank_factors(i, o, r, seed=21)
    Y = cuda_lib.lowrank_matmul(X.to(DEV), V.to(DEV), U.to(DEV))
    torch.cuda.synchronize()
    rows = sample_rows(n, 160)
    ref = orc.lowrank_forward(to64(X[rows]), to64(V), to64(U))
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"fused LR {n, i, o, r}")


MON_FUSED = [  # (n, b1, b2, r', p, q)
    (1000, 4, 4, 48, 192, 768),   # GPT2-S c_fc Monarch
    (300, 4, 4, 48, 768, 192),    # GPT2-S c_proj Monarch
    (700, 16, 16, 16, 128, 128),  # Llama-3.2-1B q/o Monarch (16 sub-GEMMs of N = 16)
    (257, 2, 4, 64, 256, 256),    # b1 != b2
    (130, 4, 2, 32, 72, 520),     # p % 64 != 0, q = 520 (two S3 chunks)
]


@pytest.mark.parametrize("layout", [orc.B2_FASTEST, orc.RPRIME_FASTEST])
@pytest.mark.parametrize("n,b1,b2,rp,p,q", MON_FUSED)
def test_monarch_fused_parity(cuda_lib, monkeypatch, layout, n, b1, b2, rp, p, q):
    monkeypatch.setenv("BLR_FUSED", "1")
    X = synth.make_x(n, b1 * p, seed=22)
    V, U = synth.monarch_factors(b1 * p, b2 * q, b1, b2, rp, seed=22)
    Y = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, v_layout=layout)
    torch.cuda.synchronize()
    rows = sample_rows(n, 160)
    ref = orc.monarch_forward(to64(X[rows]), to64(V), to64(U), b1, b2, layout)
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"fused Monarch {n, b1, b2, rp, p, q} {layout}")


def test_monarch_fused_identity_blocks_bit_exact(cuda_lib, monkeypatch):
    """Identity blocks: Y is X permuted, exact through the on-chip Z."""
    monkeypatch.setenv("BLR_FUSED", "1")
    b1 = b2 = 4
    rp = 32
    p, q = rp * b2, b1 * rp
    V = torch.stack([torch.eye(rp * b2, p) for _ in range(b1)]).to(torch.bfloat16)
    U = torch.stack([torch.eye(q, b1 * rp) for _ in range(b2)]).to(torch.bfloat16)
    X = synth.make_x(300, b1 * p, seed=23)
    for layout in (orc.B2_FASTEST, orc.RPRIME_FASTEST):
        Y = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, v_layout=layout).cpu()
        ref = orc.monarch_forward(to64(X), to64(V), to64(U), b1, b2, layout)
        assert np.array_equal(to64(Y), ref), layout


def test_fused_matches_two_kernel_path_and_is_deterministic(cuda_lib, monkeypatch):
    """Both paths round Z once to bf16 (RNE) and accumulate in fp32: they may differ only by
    accumulation order, i.e. within a bf16 ulp of Y; the fused path is bitwise repeatable."""
    n, i, o, r = 777, 768, 3072, 192
    X = synth.make_x(n, i, seed=24).to(DEV)
    V, U = [t.to(DEV) for t in synth.lowrank_factors(i, o, r, seed=24)]
    monkeypatch.setenv("BLR_FUSED", "1")
    Yf = cuda_lib.lowrank_matmul(X, V, U)
    Yf2 = cuda_lib.lowrank_matmul(X, V, U)
    monkeypatch.setenv("BLR_FUSED", "0")
    Ys = cuda_lib.lowrank_matmul(X, V, U)
    torch.cuda.synchronize()
    assert torch.equal(Yf, Yf2)
    d = (Yf.float() - Ys.float()).abs()
    assert torch.all(d <= 2.0 ** -6 * Ys.float().abs() + 1e-2)


BLAST_S23 = [  # (n, b1, b2, r, p, q): split path (b1 r > 512) with the S2 + S3 launch (mode 2)
    (1000, 6, 6, 192, 128, 512),   # GPT2-S c_fc BLAST
    (300, 6, 6, 192, 512, 128),    # GPT2-S c_proj BLAST
    (257, 5, 3, 128, 40, 200),     # b1 != b2, q % 16 != 0, ragged tail
    (700, 8, 8, 256, 128, 256),
]


@pytest.mark.parametrize("n,b1,b2,r,p,q", BLAST_S23)
def test_blast_s2_s3_fused_parity(cuda_lib, monkeypatch, n, b1, b2, r, p, q):
    """S2 (fp32 on CUDA cores, ascending l) formed straight into the S3 operand in shared memory."""
    monkeypatch.setenv("BLR_FUSED", "1")
    X = synth.make_x(n, b1 * p, seed=25)
    V, S, U = synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=25)
    Y = cuda_lib.blast_matmul(X.to(DEV), V.to(DEV), S.to(DEV), U.to(DEV))
    torch.cuda.synchronize()
    rows = sample_rows(n, 160)
    ref = orc.blast_forward(to64(X[rows]), to64(V), to64(S), to64(U))
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"BLAST S2+S3 {n, b1, b2, r, p, q}")


def test_blast_s2_s3_fused_asymmetric_S(cuda_lib, monkeypatch):
    """An S with distinct (l, k) blocks: a swapped index in the on-chip block sum cannot pass."""
    monkeypatch.setenv("BLR_FUSED", "1")
    n, b1, b2, r, p, q = 300, 6, 4, 128, 64, 96
    X = synth.make_x(n, b1 * p, seed=26)
    V, S, U = synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=26)
    S = (S.float() * torch.arange(1, b1 * b2 + 1, dtype=torch.float32).view(b1, b2, 1) / (b1 * b2)).to(torch.bfloat16)
    Y = cuda_lib.blast_matmul(X.to(DEV), V.to(DEV), S.to(DEV), U.to(DEV))
    torch.cuda.synchronize()
    ref = orc.blast_forward(to64(X), to64(V), to64(S), to64(U))
    assert_parity(Y, ref, "BLAST S2+S3 asymmetric S")


@pytest.mark.parametrize("n", [17, 127, 128, 129])
def test_single_partial_tile_token_counts(cuda_lib, monkeypatch, n):
    """Token counts inside or at the edge of one 128-row tile through the tile-blocked BLAST split
    path (S1 epilogue tensor store, S2 tensor copies, S3 tensor-box A) and the forced fused layer."""
    monkeypatch.setenv("BLR_DECODE", "0")
    b1, b2, r, p, q = 16, 16, 128, 32, 48
    X = synth.make_x(n, b1 * p, seed=27)
    V, S, U = synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=27)
    Y = cuda_lib.blast_matmul(X.to(DEV), V.to(DEV), S.to(DEV), U.to(DEV))
    torch.cuda.synchronize()
    assert_parity(Y, orc.blast_forward(to64(X), to64(V), to64(S), to64(U)), f"BLAST split n={n}")
    monkeypatch.setenv("BLR_FUSED", "1")
    i, o, rl = 640, 896, 192
    Xl = synth.make_x(n, i, seed=28)
    Vl, Ul = synth.lowrank_factors(i, o, rl, seed=28)
    Yl = cuda_lib.lowrank_matmul(Xl.to(DEV), Vl.to(DEV), Ul.to(DEV))
    torch.cuda.synchronize()
    assert_parity(Yl, orc.lowrank_forward(to64(Xl), to64(Vl), to64(Ul)), f"fused LR n={n}")
