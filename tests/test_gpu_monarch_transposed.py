"""GPU parity of the Monarch "transposed" output order and the chained next layer (SURVEY §8 row
f3; PAPER.md L45 footnote, L219-220 optimization (3)): output block k, column c at Y[t, c*b2 + k];
the next static weight's rows pre-permuted (blr_transposed_row_perm) so that no permutation pass
runs between the layers.  Every kernel path the Monarch entry point dispatches to is covered:
the one-launch fused layer, the two-kernel path (single CTAs and CTA pairs) and the small-token
decode path.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import synth
from tests.parity import assert_parity, to64

pytestmark = pytest.mark.gpu
DEV = "cuda"

SHAPES = [  # (n, b1, b2, r', p, q, env)
    (300, 4, 4, 48, 192, 768, {}),                       # GPT2-S c_fc: one-launch fused layer
    (300, 4, 4, 48, 192, 768, {"BLR_FUSED": "0"}),       # same shape, two-kernel path
    (1000, 16, 16, 96, 64, 88, {"BLR_PAIR": "2"}),       # CTA pairs, long K2 = 1536
    (257, 3, 4, 16, 72, 40, {}),                         # b1 != b2, ragged
    (5, 4, 4, 16, 64, 96, {"BLR_DECODE": "1"}),          # small-token path
    (1, 2, 3, 8, 16, 24, {"BLR_DECODE": "1"}),
]


@pytest.mark.parametrize("layout", [orc.B2_FASTEST, orc.RPRIME_FASTEST])
@pytest.mark.parametrize("n,b1,b2,rp,p,q,env", SHAPES)
def test_monarch_transposed_parity(cuda_lib, monkeypatch, layout, n, b1, b2, rp, p, q, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    i, o = b1 * p, b2 * q
    X = synth.make_x(n, i, seed=12)
    V, U = synth.monarch_factors(i, o, b1, b2, rp, seed=12)
    Y = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, v_layout=layout,
                                out_order=cuda_lib.OUT_TRANSPOSED)
    torch.cuda.synchronize()
    ref = orc.monarch_forward_transposed(to64(X), to64(V), to64(U), b1, b2, layout)
    assert_parity(Y, ref, f"Monarch transposed {n,b1,b2,rp,p,q} {env}")


@pytest.mark.parametrize("fused", ["0", "1"])
def test_monarch_transposed_identity_blocks_bit_exact(cuda_lib, monkeypatch, fused):
    """Identity blocks: the transposed-order output is an integer permutation of X (bit-exact)."""
    monkeypatch.setenv("BLR_FUSED", fused)
    b1, b2, rp = 4, 4, 32          # k2 = b1 r' = 128: the fused layer is eligible
    p, q = rp * b2, b1 * rp
    V = torch.stack([torch.eye(rp * b2, p) for _ in range(b1)]).to(torch.bfloat16)
    U = torch.stack([torch.eye(q, b1 * rp) for _ in range(b2)]).to(torch.bfloat16)
    n = 300
    X = synth.make_x(n, b1 * p, seed=13)
    for layout in (orc.B2_FASTEST, orc.RPRIME_FASTEST):
        Y = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, v_layout=layout,
                                    out_order=cuda_lib.OUT_TRANSPOSED).cpu()
        ref = orc.monarch_forward_transposed(to64(X), to64(V), to64(U), b1, b2, layout)
        assert np.array_equal(to64(Y), ref), layout


def test_transposed_chain_into_prepermuted_lowrank(cuda_lib):
    """GPT2-S-like c_fc (Monarch, transposed order) -> c_proj (low rank with pre-permuted V rows):
    two launches' worth of layers, no permutation pass in between, against the oracle's canonical
    chain."""
    n, b1, b2, rp, p, q, r2, o2 = 512, 4, 4, 48, 192, 768, 192, 768
    X = synth.make_x(n, b1 * p, seed=14)
    V, U = synth.monarch_factors(b1 * p, b2 * q, b1, b2, rp, seed=14)
    V2, U2 = synth.lowrank_factors(b2 * q, o2, r2, seed=15)
    V2p = cuda_lib.permute_rows_for_transposed_input(V2, b2, q)
    H = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2, out_order=cuda_lib.OUT_TRANSPOSED)
    Y = cuda_lib.lowrank_matmul(H, V2p.to(DEV), U2.to(DEV))
    # reference: the canonical chain on the GPU's bf16 intermediate, un-permuted back
    perm = cuda_lib.transposed_row_perm(b2, q).numpy()
    Hc = np.empty_like(to64(H))
    Hc[:, perm] = to64(H)
    ref = orc.lowrank_forward(Hc, to64(V2), to64(U2))
    assert_parity(Y, ref, "Monarch(transposed) -> low rank(pre-permuted)")
    # and the transposed intermediate itself is the canonical one, permuted
    Hcan = cuda_lib.monarch_matmul(X.to(DEV), V.to(DEV), U.to(DEV), b1, b2)
    assert torch.equal(H[:, torch.as_tensor(np.argsort(perm), device=DEV)], Hcan)
