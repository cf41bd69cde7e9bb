"""GPU parity of the FP8 (e4m3) first-stage intermediate, blr_blast_matmul_fp8z (SURVEY §8 row
f4), against the fp64 oracle under the contract derived in tests/test_fp8_budget.py (relative
Frobenius <= 0.04, per element <= 0.2 (1 + |ref|)), at the shapes where the split path runs
(b1 r > 512) including the Llama-7B MLP at full size; other paths must equal blr_blast_matmul."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import configs, synth
from tests.parity import sample_rows, to64
from tests.test_fp8_budget import FP8_ELEM, FP8_FROB

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _check(Y, ref, what):
    g = to64(Y)
    assert np.all(np.isfinite(g)), what
    rel = np.linalg.norm(g - ref) / np.linalg.norm(ref)
    elem = np.max(np.abs(g - ref) / (1 + np.abs(ref)))
    assert rel <= FP8_FROB and elem <= FP8_ELEM, f"{what}: rel {rel:.3e}, elem {elem:.3e}"
    return rel


@pytest.mark.parametrize("n,b1,b2,r,p,q", [(300, 6, 6, 192, 128, 512),
                                           (257, 9, 7, 136, 32, 40),       # odd panels, b1 != b2
                                           (1000, 16, 16, 272, 64, 88),
                                           (130, 16, 16, 1488, 256, 688)])
def test_fp8z_parity(cuda_lib, n, b1, b2, r, p, q):
    i, o = b1 * p, b2 * q
    X = synth.make_x(n, i, seed=17)
    V, S, U = synth.blast_factors(i, o, b1, b2, r, seed=17)
    Y = cuda_lib.blast_matmul(X.to(DEV), V.to(DEV), S.to(DEV), U.to(DEV), fp8_intermediate=True)
    torch.cuda.synchronize()
    rel = _check(Y, orc.blast_forward(to64(X), to64(V), to64(S), to64(U)), f"fp8z {n,b1,b2,r,p,q}")
    assert rel > 5e-3  # the e4m3 rounding really happened (this path is not the fp16 one)


@pytest.mark.parametrize("j", [0, 1])
def test_fp8z_llama7b_full_size_sampled_rows(cuda_lib, j):
    w = configs.C4
    L = w.layers[j]
    X = synth.make_x(w.n, L.i, seed=0, layer_id=j, device=DEV)
    fac = [t.to(DEV) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r, 0, j)]
    Y = cuda_lib.blast_matmul(X, *fac, fp8_intermediate=True)
    rows = torch.as_tensor(sample_rows(w.n, 256), device=DEV)
    _check(Y[rows], orc.blast_forward(to64(X[rows]), *[to64(t) for t in fac]), f"C4 layer {j} fp8z")


def test_fp8z_other_paths_identical(cuda_lib):
    """b1 r <= 512 (fused S1+S2, no Z in HBM) and r < 128 (compensated CUDA-core S2): the FP8 entry
    point is bit-identical to blr_blast_matmul."""
    for (n, b1, b2, r, p, q) in [(200, 4, 4, 64, 64, 64), (200, 16, 16, 48, 16, 16)]:
        X = synth.make_x(n, b1 * p, seed=18).to(DEV)
        fac = [t.to(DEV) for t in synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=18)]
        assert torch.equal(cuda_lib.blast_matmul(X, *fac, fp8_intermediate=True), cuda_lib.blast_matmul(X, *fac))


def test_fp8z_nonfinite_row_stays_local(cuda_lib):
    n, b1, p, q, r = 384, 16, 16, 24, 136
    X = synth.make_x(n, b1 * p, seed=19).to(DEV)
    fac = [t.to(DEV) for t in synth.blast_factors(b1 * p, b1 * q, b1, b1, r, seed=19)]
    clean = cuda_lib.blast_matmul(X, *fac, fp8_intermediate=True)
    Xp = X.clone()
    Xp[128, 3] = float("nan")
    Y = cuda_lib.blast_matmul(Xp, *fac, fp8_intermediate=True)
    keep = torch.ones(n, dtype=torch.bool, device=DEV)
    keep[128] = False
    assert torch.equal(Y[keep], clean[keep])
