"""Why the BLAST split path stores its S1 output Z in fp16, not bf16 (reading R13): an
emulation of the GPU path's rounding points (fp32 accumulation per stage; RNE to bf16 where the
kernels store bf16, RNE to fp16 for Z) against the fp64 oracle under the north_star per-element
bound |err| <= 1e-2 (1 + |ref|).  Rounding Z to bf16 (three bf16 roundings: Z, Z'', Y) exceeds the
bound on GPT2-S / DiT shapes; an fp32 Z (two roundings) and the implemented fp16 Z (11-bit
significand: ~1/8 of a bf16 rounding) stay inside it, including the Llama-7B (C4) shapes.
CPU only (-m "not gpu")."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import synth


def _bf(x):
    return x.to(torch.bfloat16).to(torch.float32)


def _emulate(X, V, S, U, z_mode):
    n = X.shape[0]
    b1, p, r = V.shape
    b2, _, q = U.shape
    Z = torch.einsum("tla,lar->ltr", X.float().reshape(n, b1, p), V.float())  # S1, fp32 accumulation
    if z_mode == "bf16":
        Z = _bf(Z)
    elif z_mode == "fp16":
        Z = Z.to(torch.float16).to(torch.float32)
    Zf = torch.einsum("lkr,ltr->ktr", S.float(), Z)                              # S2, fp32
    Zpp = _bf(Zf) if r >= 128 else _bf(Zf) + _bf(Zf - _bf(Zf))                   # hi|lo pair when r < 128
    return _bf(torch.einsum("ktr,krc->tkc", Zpp, U.float())).reshape(n, b2 * q).double().numpy()


def _elem_ratio(Y, ref):
    return float(np.max(np.abs(Y - ref) / (1e-2 * (1 + np.abs(ref)))))


CASES = [(256, 6, 6, 192, 128, 512),   # GPT2-S c_fc BLAST
         (130, 9, 9, 384, 128, 384),   # DiT-XL/2 qkv
         (200, 16, 16, 48, 16, 16),
         (64, 16, 16, 1488, 256, 688),  # Llama-7B gate/up (C4)
         (48, 16, 16, 1488, 688, 256)]  # Llama-7B down (C4)


@pytest.mark.parametrize("n,b1,b2,r,p,q", CASES)
def test_fp16_and_fp32_intermediates_meet_the_bound_and_bf16_would_not_always(n, b1, b2, r, p, q):
    worst_bf16 = 0.0
    for outliers in (0, 8):
        X = synth.make_x(n, b1 * p, seed=3, outliers=outliers)
        V, S, U = synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=3)
        ref = orc.blast_forward(X.double().numpy(), V.double().numpy(), S.double().numpy(), U.double().numpy())
        assert _elem_ratio(_emulate(X, V, S, U, "fp32"), ref) < 1.0
        assert _elem_ratio(_emulate(X, V, S, U, "fp16"), ref) < 1.0
        worst_bf16 = max(worst_bf16, _elem_ratio(_emulate(X, V, S, U, "bf16"), ref))
    if r >= 128 and r < 1024:  # large-r shapes: a bf16 Z pushes some element past the north_star bound
        assert worst_bf16 > 1.0
