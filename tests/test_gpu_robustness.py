"""GPU robustness: row independence under non-finite inputs, large-magnitude activations, and
the >= 2x-compression / C5 configurations at full size.

Row independence (Y[t, :] depends only on X[t, :]) must hold bit for bit even when
another token carries NaN or Inf: the BLAST split path's tile-blocked intermediate puts the next
token tile's panels right after a tile's last K block, and the S3 kernel must never multiply them
(SURVEY §8(c) c14).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import configs, synth
from tests.parity import assert_parity, sample_rows, to64

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _run(cuda_lib, method, X, fac, b1=1, b2=1):
    if method == "lowrank":
        return cuda_lib.lowrank_matmul(X, *fac)
    if method == "monarch":
        return cuda_lib.monarch_matmul(X, *fac, b1, b2)
    return cuda_lib.blast_matmul(X, *fac)


# (method, n, i, o, r, b): the BLAST rows take the split path (b1 r > 512) with r / 8 odd (17, 93
# panels: the zero-panel half step) and even but not a multiple of 8 (182 panels)
POISON_CASES = [
    ("blast", 384, 16 * 32, 16 * 40, 136, 16),
    ("blast", 300, 16 * 16, 16 * 24, 744, 16),
    ("blast", 260, 16 * 16, 16 * 16, 1456, 16),
    ("blast", 384, 6 * 128, 6 * 512, 192, 6),
    ("monarch", 384, 4 * 192, 4 * 768, 192, 4),
    ("lowrank", 384, 768, 3072, 200, 1),
]


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
@pytest.mark.parametrize("method,n,i,o,r,b", POISON_CASES)
def test_nonfinite_token_does_not_touch_other_rows(cuda_lib, method, n, i, o, r, b, bad):
    X = synth.make_x(n, i, seed=21).to(DEV)
    if method == "lowrank":
        fac = synth.lowrank_factors(i, o, r, seed=21)
    elif method == "monarch":
        fac = synth.monarch_factors(i, o, b, b, r // b, seed=21)
    else:
        fac = synth.blast_factors(i, o, b, b, r, seed=21)
    fac = [t.to(DEV) for t in fac]
    clean = _run(cuda_lib, method, X, fac, b, b)
    for t0 in (0, 127, 128, n - 1):   # tile edges: a tile's K tail would read the next tile's rows
        Xp = X.clone()
        Xp[t0, 5] = bad
        Y = _run(cuda_lib, method, Xp, fac, b, b)
        keep = torch.ones(n, dtype=torch.bool, device=DEV)
        keep[t0] = False
        assert torch.equal(Y[keep], clean[keep]), f"{method} poisoned row {t0} ({bad}) changed other rows"
        if bad != bad:  # NaN propagates into its own row (IEEE)
            assert torch.isnan(Y[t0].float()).any()


@pytest.mark.parametrize("scale", [1e3])
@pytest.mark.parametrize("method,n,i,o,r,b", [("blast", 300, 16 * 256, 16 * 64, 744, 16),
                                              ("blast", 256, 6 * 512, 6 * 128, 192, 6),
                                              ("monarch", 256, 16 * 256, 16 * 64, 1536, 16),
                                              ("lowrank", 256, 4096, 1024, 256, 1)])
def test_large_magnitude_and_raw_outliers(cuda_lib, method, n, i, o, r, b, scale):
    """|X| ~ 1e3 with 8 channels x20 on top and NO renormalisation (|X| up to ~1e5 in those
    channels), at Llama-7B-like block sizes (p = 256): the split path's fp16 Z stays inside its
    range (|X_l V_l| <= 65504, include/blr.h) and the result meets the north_star bound, applied
    at the output's scale, against the fp64 oracle.  (With p = 16 the same X drives |Z| to
    ~7.5e4: outside the documented fp16 range -- test_fp16_range_saturates_and_stays_row_local.
    At GPT2-S c_fc shapes this raw-outlier input exceeds the per-element bound even with exact
    fp32 intermediates before the final two bf16 roundings (emulated: BLAST 1.05x, Monarch 1.08x
    the bound) -- a property of the bound, not of the kernels, reading R17; the cases
    below are Llama-7B-like blocks (emulated worst element 0.7-0.8x the bound).)"""
    g = torch.Generator().manual_seed(33)
    x = torch.randn(n, i, generator=g) * scale
    idx = torch.linspace(0, i - 1, 8).round().long()
    x[:, idx] *= 20.0
    X = x.to(torch.bfloat16)
    if method == "lowrank":
        fac = synth.lowrank_factors(i, o, r, seed=33)
    elif method == "monarch":
        fac = synth.monarch_factors(i, o, b, b, r // b, seed=33)
    else:
        fac = synth.blast_factors(i, o, b, b, r, seed=33)
    Y = _run(cuda_lib, method, X.to(DEV), [t.to(DEV) for t in fac], b, b)
    f64 = [to64(t) for t in fac]
    if method == "lowrank":
        ref = orc.lowrank_forward(to64(X), *f64)
    elif method == "monarch":
        ref = orc.monarch_forward(to64(X), *f64, b, b)
    else:
        ref = orc.blast_forward(to64(X), *f64)
    assert np.abs(ref).max() > 1e3
    # the layer is linear: the north_star bound is stated for the recipe's unit-scale outputs, so
    # it is applied to Y / s and ref / s with s = rms(ref) (the Frobenius criterion is scale-free;
    # the per-element floor 1e-2 would otherwise demand ~1e-5 relative accuracy near zero)
    s = float(np.sqrt(np.mean(ref ** 2)))
    assert_parity(torch.from_numpy(to64(Y) / s), ref / s, f"{method} |X|~{scale:g} raw outliers")


def _factors(L, seed, layer_id):
    if L.method == "lowrank":
        return synth.lowrank_factors(L.i, L.o, L.r, seed, layer_id)
    if L.method == "monarch":
        return synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r_blk, seed, layer_id)
    return synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r, seed, layer_id)


NEW_FULL = [(k, j) for k in ("C4X", "C5V-256", "C5D-256") for j in range(len(configs.WORKLOADS[k].layers))]


@pytest.mark.parametrize("key,j", NEW_FULL)
def test_new_configs_sampled_rows(cuda_lib, key, j):
    """>= 2x-compression ranks (BLAST r = 1456, Monarch r' = 88) at the Llama-7B MLP and the C5
    ViT-B / DiT-XL/2 layers at 256 images, full size, as bench.py launches them; a seeded sample
    of 256 rows (first and last included) against the oracle."""
    w = configs.WORKLOADS[key]
    L = w.layers[j]
    X = synth.make_x(w.n, L.i, seed=0, layer_id=j, device=DEV)
    fac = [t.to(DEV) for t in _factors(L, 0, j)]
    Y = _run(cuda_lib, L.method, X, fac, L.b1, L.b2)
    rows = sample_rows(w.n, 256)
    ridx = torch.as_tensor(rows, device=DEV)
    f64 = [to64(t) for t in fac]
    if L.method == "monarch":
        ref = orc.monarch_forward(to64(X[ridx]), *f64, L.b1, L.b2)
    elif L.method == "lowrank":
        ref = orc.lowrank_forward(to64(X[ridx]), *f64)
    else:
        ref = orc.blast_forward(to64(X[ridx]), *f64)
    assert_parity(Y[ridx], ref, f"{key} layer {j} ({L.name} {L.method} r={L.r})")


def test_fp16_range_saturates_and_stays_row_local(cuda_lib, monkeypatch):
    """Beyond the split path's fp16 range (|X_l V_l| > 65504, include/blr.h) Z saturates at
    +-65504 (cvt.rn.satfinite): the affected rows get finite, clamped values -- never Inf from
    finite inputs -- and the rows below the limit are bit-identical to a run without them."""
    monkeypatch.setenv("BLR_BLAST_PATH", "split")
    n, b, p, q, r = 256, 16, 16, 24, 136
    X = synth.make_x(n, b * p, seed=41).to(DEV)
    fac = [t.to(DEV) for t in synth.blast_factors(b * p, b * q, b, b, r, seed=41)]
    clean = cuda_lib.blast_matmul(X, *fac)
    Xb = X.clone()
    Xb[7] *= 1e6                       # one token far beyond the range
    Y = cuda_lib.blast_matmul(Xb, *fac)
    assert torch.isfinite(Y.float()).all()
    keep = torch.ones(n, dtype=torch.bool, device=DEV)
    keep[7] = False
    assert torch.equal(Y[keep], clean[keep])
