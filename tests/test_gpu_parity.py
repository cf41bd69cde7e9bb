"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element.

Tolerance (BASELINE.json north_star): relative Frobenius <= 5e-3 and per element
|err| <= 1e-2 (1 + |ref|), reference = fp64 oracle on the same bf16-rounded inputs.
Integer-exact cases (identity-block Monarch = permutation) are compared bit for bit.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import configs, synth
from tests.parity import assert_parity, sample_rows, to64

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _rand(shape, std, seed):
    return synth.randn_bf16(shape, std, seed)


# ------------------------------------------------------------------------------ low rank -------
LR_SHAPES = [  # (n, i, o, r)
    (1, 8, 8, 8),
    (5, 64, 64, 16),
    (300, 200, 136, 40),     # ragged tokens, K % 64 != 0, N % 16 != 0
    (129, 768, 3072, 192),   # GPT2 c_fc rank, ragged tail
    (257, 3072, 768, 192),
    (128, 256, 600, 264),    # r > 256 -> two N tiles in phase 1
]


@pytest.mark.parametrize("n,i,o,r", LR_SHAPES)
def test_lowrank_parity(cuda_lib, n, i, o, r):
    X = synth.make_x(n, i, seed=1)
    V, U = synth.lowrank_factors(i, o, r, seed=1)
    Y = cuda_lib.lowrank_matmul(X.to(DEV), V.to(DEV), U.to(DEV))
    torch.cuda.synchronize()
    assert_parity(Y, orc.lowrank_forward(to64(X), to64(V), to64(U)), f"LR {n,i,o,r}")


# ------------------------------------------------------------------------------ Monarch --------
MON_SHAPES = [  # (n, b1, b2, r', p, q)
    (1, 1, 1, 8, 8, 8),
    (130, 2, 2, 8, 16, 24),
    (257, 3, 4, 16, 72, 40),
    (200, 4, 4, 48, 192, 768),    # GPT2-S c_fc Monarch (r=192, b=4)
    (129, 4, 4, 48, 768, 192),    # GPT2-S c_proj
    (131, 16, 16, 16, 128, 128),  # Llama-1B q/o (r=256, b=16)
    (64, 16, 16, 48, 128, 512),   # Llama-1B up (r=768): 5 k-blocks per tile, ragged
    (70, 2, 3, 24, 40, 16),       # r' odd multiple of 8
]


@pytest.mark.parametrize("layout", [orc.B2_FASTEST, orc.RPRIME_FASTEST])
@pytest.mark.parametrize("n,b1,b2,rp,p,q", MON_SHAPES)
def test_monarch_parity(cuda_lib, layout, n, b1, b2, rp, p, q):
    i, o = b1 * p, b2 * q
    X = synth.make_x(n, i, seed=2)
    V, U = synth.monarch_factors(i, o, b1, b2, rp, seed=2)
    Y = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, v_layout=layout)
    torch.cuda.synchronize()
    ref = orc.monarch_forward(to64(X), to64(V), to64(U), b1, b2, layout)
    assert_parity(Y, ref, f"Monarch {n,b1,b2,rp,p,q} layout={layout}")


@pytest.mark.parametrize("b1,b2,rp", [(2, 2, 8), (3, 2, 16), (4, 4, 8)])
def test_monarch_identity_blocks_bit_exact(cuda_lib, b1, b2, rp):
    """north_star: Monarch with identity blocks is a pure permutation -> bit-exact on GPU."""
    p, q = rp * b2, b1 * rp
    V = torch.stack([torch.eye(rp * b2, p) for _ in range(b1)]).to(torch.bfloat16)
    U = torch.stack([torch.eye(q, b1 * rp) for _ in range(b2)]).to(torch.bfloat16)
    n = 150
    X = synth.make_x(n, b1 * p, seed=5)
    for layout in (orc.B2_FASTEST, orc.RPRIME_FASTEST):
        Y = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, v_layout=layout).cpu()
        ref = orc.monarch_forward(to64(X), to64(V), to64(U), b1, b2, layout)
        assert np.array_equal(to64(Y), ref), layout


# ------------------------------------------------------------------------------ BLAST ----------
BLAST_SHAPES = [  # (n, b1, b2, r, p, q)
    (1, 1, 1, 16, 8, 8),
    (129, 2, 3, 24, 40, 56),
    (128, 4, 4, 16, 192, 192),     # C1 shape (768x768, b=4, r=16)
    (200, 16, 16, 48, 16, 16),     # b = 16 (Llama block count), small blocks
    (256, 6, 6, 192, 128, 512),    # GPT2-S c_fc BLAST
    (197, 3, 3, 128, 256, 768),    # ViT-B qkv, one image
    (130, 9, 9, 384, 128, 384),    # DiT-XL/2 qkv
    (100, 5, 2, 40, 24, 64),       # b1 != b2, r % 16 != 0
]


@pytest.mark.parametrize("n,b1,b2,r,p,q", BLAST_SHAPES)
def test_blast_parity(cuda_lib, n, b1, b2, r, p, q):
    i, o = b1 * p, b2 * q
    X = synth.make_x(n, i, seed=3)
    V, S, U = synth.blast_factors(i, o, b1, b2, r, seed=3)
    Y = cuda_lib.blast_matmul(X.to(DEV), V.to(DEV), S.to(DEV), U.to(DEV))
    torch.cuda.synchronize()
    ref = orc.blast_forward(to64(X), to64(V), to64(S), to64(U))
    assert_parity(Y, ref, f"BLAST {n,b1,b2,r,p,q}")


def test_blast_asymmetric_S_index_order(cuda_lib):
    """S[l,k,:] (input block, output block) -- a swapped index order cannot pass (reading R5)."""
    b1, b2, r, p, q, n = 3, 2, 16, 32, 48, 64
    X = synth.make_x(n, b1 * p, seed=9)
    V, S, U = synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=9)
    S = S.clone()
    S[0, 1, :] = 0  # kill W_{0,1}
    Y = cuda_lib.blast_matmul(X.to(DEV), V.to(DEV), S.to(DEV), U.to(DEV)).cpu()
    assert_parity(Y, orc.blast_forward(to64(X), to64(V), to64(S), to64(U)), "asymmetric S")


def test_blast_S_const_matches_lowrank_gpu(cuda_lib):
    """Pin p3 on the GPU: BLAST with S == c (c = 1/b1 = 0.25, exact in bf16, keeps the recipe's
    unit output variance) equals low rank with stacked V and concatenated c*U."""
    b1, b2, r, p, q, n = 4, 3, 32, 64, 64, 200
    X = synth.make_x(n, b1 * p, seed=4)
    V, _, U = synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=4)
    S = torch.full((b1, b2, r), 0.25, dtype=torch.bfloat16)
    Yb = cuda_lib.blast_matmul(X.to(DEV), V.to(DEV), S.to(DEV), U.to(DEV))
    Vlr = V.reshape(b1 * p, r).contiguous()
    Ulr = torch.cat([U[k] for k in range(b2)], dim=1).contiguous()
    ref = orc.lowrank_forward(to64(X), to64(Vlr), 0.25 * to64(Ulr))
    assert_parity(Yb, ref, "BLAST S=1")


# ------------------------------------------------------------------------------ invariants -----
def test_row_permutation_and_determinism(cuda_lib):
    """Rows are independent: permuting X rows permutes Y rows bit-exactly when the
    permutation keeps each row's tile-independent arithmetic; run-to-run output is bitwise equal."""
    b1, b2, r, p, q, n = 6, 6, 192, 128, 512, 512
    X = synth.make_x(n, b1 * p, seed=6).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=6)]
    Y1 = cuda_lib.blast_matmul(X, V, S, U)
    Y2 = cuda_lib.blast_matmul(X, V, S, U)
    assert torch.equal(Y1, Y2)
    perm = torch.randperm(n, generator=torch.Generator().manual_seed(0)).to(DEV)
    Yp = cuda_lib.blast_matmul(X[perm].contiguous(), V, S, U)
    assert torch.equal(Yp, Y1[perm])


def test_token_shards_concat_bitwise(cuda_lib):
    """Pin p12: token-sharded outputs concatenated == unsharded output, bit for bit.

    Every shard must take the same kernel path as the whole batch: shards of <= 256 tokens run
    the weight-streaming small-n Monarch path (another summation order), so the shards here are
    512 tokens (the bench's smallest shard is 8,192 tokens, C4 at N = 8)."""
    L = configs.table3("GPT2-S", "c_fc", "monarch")
    n = 2048
    X = synth.make_x(n, L.i, seed=7).to(DEV)
    V, U = [t.to(DEV) for t in synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r_blk, seed=7)]
    full = cuda_lib.monarch_matmul(X, V, U, L.b1, L.b2)
    parts = [cuda_lib.monarch_matmul(X[s:s + n // 4].contiguous(), V, U, L.b1, L.b2) for s in range(0, n, n // 4)]
    assert torch.equal(torch.cat(parts), full)


def test_zero_tokens_noop(cuda_lib):
    X = torch.empty((0, 64), dtype=torch.bfloat16, device=DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(64, 64, 2, 2, 16)]
    Y = cuda_lib.blast_matmul(X, V, S, U)
    assert Y.shape == (0, 64)


def test_outlier_channels(cuda_lib):
    """Stress variant: 8 input channels scaled x20."""
    L = configs.table3("Llama-3.2-1B", "q_o_proj", "blast")
    n = 256
    X = synth.make_x(n, L.i, seed=8, outliers=8)
    V, S, U = synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r, seed=8)
    Y = cuda_lib.blast_matmul(X.to(DEV), V.to(DEV), S.to(DEV), U.to(DEV))
    assert_parity(Y, orc.blast_forward(to64(X), to64(V), to64(S), to64(U)), "outliers")


# ------------------------------------------------------------------------------ full configs ---
def _layer_run(cuda_lib, L, X, fac):
    if L.method == "lowrank":
        return cuda_lib.lowrank_matmul(X, *fac)
    if L.method == "monarch":
        return cuda_lib.monarch_matmul(X, *fac, L.b1, L.b2)
    return cuda_lib.blast_matmul(X, *fac)


def _layer_ref(L, X, fac):
    f = [to64(t) for t in fac]
    if L.method == "lowrank":
        return orc.lowrank_forward(X, *f)
    if L.method == "monarch":
        return orc.monarch_forward(X, *f, L.b1, L.b2)
    return orc.blast_forward(X, *f)


def _factors(L, seed, layer_id):
    if L.method == "lowrank":
        return synth.lowrank_factors(L.i, L.o, L.r, seed, layer_id)
    if L.method == "monarch":
        return synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r_blk, seed, layer_id)
    return synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r, seed, layer_id)


FULL = [(w.key, j) for w in (configs.C1, configs.C2, configs.C3, configs.C4, configs.C4_MONARCH)
        for j in range(len(w.layers))]


@pytest.mark.parametrize("key,j", FULL)
def test_baseline_config_sampled_rows(cuda_lib, key, j):
    """Every BASELINE.json config at full size, in the launch configuration bench.py times:
    all rows for C1, a seeded sample of 256 rows (incl. first/last) otherwise."""
    w = configs.WORKLOADS[key]
    L = w.layers[j]
    X = synth.make_x(w.n, L.i, seed=0, layer_id=j, device=DEV)
    fac = [t.to(DEV) for t in _factors(L, 0, j)]
    Y = _layer_run(cuda_lib, L, X, fac)
    rows = sample_rows(w.n, 256 if w.n > 256 else w.n)
    ridx = torch.as_tensor(rows, device=DEV)
    ref = _layer_ref(L, to64(X[ridx]), fac)
    assert_parity(Y[ridx], ref, f"{key} layer {j} ({L.model} {L.name} {L.method})")


@pytest.mark.parametrize("images", [1, 64])
def test_c5_vit_dit(cuda_lib, images):
    for w in (configs.c5(images), configs.c5_dit(images)):
        for j, L in enumerate(w.layers):
            X = synth.make_x(w.n, L.i, seed=0, layer_id=j, device=DEV)
            fac = [t.to(DEV) for t in _factors(L, 0, j)]
            Y = _layer_run(cuda_lib, L, X, fac)
            rows = sample_rows(w.n, 128)
            ridx = torch.as_tensor(rows, device=DEV)
            assert_parity(Y[ridx], _layer_ref(L, to64(X[ridx]), fac), f"{w.key} {L.name} {L.method}")


# ------------------------------------------------------------------------------ CTA-pair mode --
@pytest.mark.parametrize("pair", ["1", "2", "0"])
@pytest.mark.parametrize("resident", ["0", "1"])
@pytest.mark.parametrize("method", ["lowrank", "monarch", "blast"])
def test_forced_cta_pair_modes(cuda_lib, monkeypatch, pair, resident, method):
    """Both GEMM variants (one CTA, or a cta_group::2 pair with M=256 and B split across the pair;
    BLR_PAIR=0 = the shape heuristic), streamed or weight-stationary (BLR_RESIDENT=1, opt-in), on
    shapes with ragged token tails and multi-tile N, against the oracle."""
    monkeypatch.setenv("BLR_PAIR", pair)
    monkeypatch.setenv("BLR_RESIDENT", resident)
    n = 1000
    if method == "lowrank":
        L = configs.Layer("t", "t", 1024, 1376, "lowrank", 160, 1)
    elif method == "monarch":
        L = configs.Layer("t", "t", 1024, 1376, "monarch", 256, 16)   # r' = 16, q = 86 -> use 8-mult
        L = configs.Layer("t", "t", 2048, 1408, "monarch", 256, 16)   # q = 88
    else:
        L = configs.Layer("t", "t", 1024, 1408, "blast", 272, 16)     # split path (b1*r > 512)
    X = synth.make_x(n, L.i, seed=11, device=DEV)
    fac = [t.to(DEV) for t in _factors(L, 11, 0)]
    Y = _layer_run(cuda_lib, L, X, fac)
    rows = sample_rows(n, 200)
    ridx = torch.as_tensor(rows, device=DEV)
    assert_parity(Y[ridx], _layer_ref(L, to64(X[ridx]), fac), f"pair={pair} {method}")


# ------------------------------------------------------------------- BLAST split-path S2 variants --
@pytest.mark.parametrize("s2", ["mma", "cuda"])
@pytest.mark.parametrize("n,b1,b2,r,p,q", [(1000, 16, 16, 272, 64, 88),   # ragged rows, r % 64 != 0
                                           (300, 6, 6, 192, 128, 512),    # GPT2-S c_fc shape
                                           (257, 9, 7, 136, 32, 40),      # odd b1 / b2
                                           (130, 16, 16, 1488, 256, 688)])  # Llama-7B gate/up (C4)
def test_blast_split_s2_variants(cuda_lib, monkeypatch, s2, n, b1, b2, r, p, q):
    """The split path's S2 (tensor-core block-diagonal GEMM on chunk-blocked fp16 Z, or the
    CUDA-core streaming kernel on fp16 Z) against the oracle, ragged tails included."""
    monkeypatch.setenv("BLR_S2", s2)
    monkeypatch.setenv("BLR_BLAST_PATH", "split")
    i, o = b1 * p, b2 * q
    X = synth.make_x(n, i, seed=5)
    V, S, U = synth.blast_factors(i, o, b1, b2, r, seed=5)
    Y = cuda_lib.blast_matmul(X.to(DEV), V.to(DEV), S.to(DEV), U.to(DEV))
    torch.cuda.synchronize()
    rows = sample_rows(n, 130)
    ref = orc.blast_forward(to64(X[rows]), to64(V), to64(S), to64(U))
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"S2={s2} {n,b1,b2,r,p,q}")


def test_blast_split_s2_mma_close_to_cuda(cuda_lib, monkeypatch):
    """fp16 Z, fp32 accumulation in both S2 kernels: the tensor core's exact fp16 products summed
    in fp32 and the CUDA cores' ascending-l fp32 FMAs may differ in the last bit of Z'' only, so
    the two Y agree to within one bf16 ulp of Y (|dY| <= 2^-7 |Y| + tiny)."""
    monkeypatch.setenv("BLR_BLAST_PATH", "split")
    n, b1, b2, r, p, q = 512, 16, 16, 272, 64, 88
    X = synth.make_x(n, b1 * p, seed=6).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=6)]
    monkeypatch.setenv("BLR_S2", "mma")
    Ym = cuda_lib.blast_matmul(X, V, S, U).float()
    monkeypatch.setenv("BLR_S2", "cuda")
    Yc = cuda_lib.blast_matmul(X, V, S, U).float()
    torch.cuda.synchronize()
    assert torch.all((Ym - Yc).abs() <= 2.0 ** -6 * Yc.abs() + 1e-2)
