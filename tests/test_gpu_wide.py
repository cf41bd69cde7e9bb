"""Wide CTA-pair tiles (two MMAs of N = BN/2 per K step into one TMEM accumulator, BLR_WIDE=1) with
the per-half accumulator release (KParams::split_rel: the epilogue frees column half 0 first, the
next tile's K blocks start on half 0 and hold their ring slots until half 1 is free, then catch up).

Against the fp64 oracle on ragged token / K / N tails, K shorter than the ring (the catch-up at the
tile end), K much longer than the ring (the hold limit), and the BLAST split path whose S1 writes the
tile-blocked fp16 Z.  The same products in the same K order as the default 256-column tiles, so the
two plans must agree bit for bit (the MMA's K = 16 step sums do not depend on the tile's N)."""
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import synth
from tests.parity import assert_parity, sample_rows, to64

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda")


def _lowrank(cuda_lib, X, V, U):
    Y = cuda_lib.lowrank_matmul(X, V, U)
    torch.cuda.synchronize()
    return Y


@pytest.mark.parametrize("split", ["1", "0"])
@pytest.mark.parametrize("n,i,o,r", [
    (1000, 64, 1104, 264),     # K = 64: one K block per tile (every tile ends with the catch-up)
    (640, 520, 520, 512),      # ragged K tail, N = 520 (two wide tiles, the second mostly empty)
    (2500, 1024, 1376, 320),   # long K for S1 (the hold limit), ragged rows
    (257, 200, 784, 296),      # a CTA pair's second tile past n_tok
])
def test_wide_lowrank(cuda_lib, monkeypatch, split, n, i, o, r):
    X = synth.make_x(n, i, seed=n + 1).to(DEV)
    V, U = [t.to(DEV) for t in synth.lowrank_factors(i, o, r, seed=o + 1)]
    Y0 = _lowrank(cuda_lib, X, V, U)
    monkeypatch.setenv("BLR_WIDE", "1")
    monkeypatch.setenv("BLR_SPLITREL", split)
    Y = _lowrank(cuda_lib, X, V, U)
    rows = sample_rows(n, 64)
    ref = orc.lowrank_forward(to64(X[rows].cpu()), to64(V.cpu()), to64(U.cpu()))
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"wide lowrank {n, i, o, r} split={split}")
    assert torch.equal(Y, Y0), f"wide vs default tiles {n, i, o, r} split={split}"
    # deterministic: the hand-over order depends on timing, the arithmetic must not
    Y2 = _lowrank(cuda_lib, X, V, U)
    assert torch.equal(Y2, Y)


@pytest.mark.parametrize("n,b1,b2,r,p,q", [(1000, 16, 16, 272, 64, 88),
                                           (4100, 4, 4, 1488, 176, 688)])   # C4 down-proj-like S1 (N = r)
def test_wide_blast_split(cuda_lib, monkeypatch, n, b1, b2, r, p, q):
    i, o = b1 * p, b2 * q
    X = synth.make_x(n, i, seed=7).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(i, o, b1, b2, r, seed=7)]
    monkeypatch.setenv("BLR_BLAST_PATH", "split")
    Y0 = cuda_lib.blast_matmul(X, V, S, U)
    monkeypatch.setenv("BLR_WIDE", "1")
    Y = cuda_lib.blast_matmul(X, V, S, U)
    torch.cuda.synchronize()
    rows = sample_rows(n, 64)
    ref = orc.blast_forward(to64(X[rows].cpu()), to64(V.cpu()), to64(S.cpu()), to64(U.cpu()))
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"wide blast {n, b1, b2, r}")
    assert torch.equal(Y, Y0)


@pytest.mark.parametrize("method,n,i,o,r,b", [
    ("blast", 1000, 1024, 16 * 88, 272, 16),   # S3 N = q = 88 < 256: one narrow tile per group
    ("blast", 2100, 512, 4 * 688, 320, 4),     # S3 N = 688 = 256 + 256 + 176 (C4 gate S3's split)
    ("lowrank", 700, 520, 600, 264, 1),        # S3 N = 600 = 2 x 256 + 88 -> a 96-column last MMA
    ("lowrank", 1300, 1000, 1032, 328, 1),     # N = 1032: a 16-column last tile (8 valid)
])
def test_last_tile_narrow_mma(cuda_lib, monkeypatch, method, n, i, o, r, b):
    """The last N tile's MMA covers only its valid columns (KParams::last_nb, each CTA of a pair
    loading half of them): the same dot products as the full-width MMA, bit for bit, and the oracle."""
    X = synth.make_x(n, i, seed=3).to(DEV)
    if method == "blast":
        fac = [t.to(DEV) for t in synth.blast_factors(i, o, b, b, r, seed=3)]
        run = lambda: cuda_lib.blast_matmul(X, *fac)  # noqa: E731
    else:
        fac = [t.to(DEV) for t in synth.lowrank_factors(i, o, r, seed=3)]
        run = lambda: cuda_lib.lowrank_matmul(X, *fac)  # noqa: E731
    monkeypatch.setenv("BLR_BLAST_PATH", "split")
    Y = run()
    monkeypatch.setenv("BLR_LASTN", "0")
    Y0 = run()
    torch.cuda.synchronize()
    assert torch.equal(Y, Y0), f"last-tile MMA width {method} {n, i, o, r, b}"
    rows = sample_rows(n, 48)
    Xr = to64(X[rows].cpu())
    fr = [to64(t.cpu()) for t in fac]
    ref = orc.blast_forward(Xr, *fr) if method == "blast" else orc.lowrank_forward(Xr, *fr)
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"last tile {method} {n, i, o, r, b}")


@pytest.mark.parametrize("n,b1,b2,r,p,q", [(1000, 16, 16, 272, 64, 88),    # r/8 = 34 panels: half-valid K tail
                                           (2100, 4, 4, 1488, 176, 688),  # C4-like gate S3 (2 x 352 columns)
                                           (300, 6, 6, 200, 128, 512)])   # r/8 = 25: odd panel count
def test_wide_kmajor_blocked_a(cuda_lib, monkeypatch, n, b1, b2, r, p, q):
    """K-major factor storage, wide tiles forced on every phase: S3's tile-blocked A goes through
    the per-half-release MMA path with its partial-panel K tail (zero panel), bit for bit equal to
    the paper-layout call and within the oracle's tolerance."""
    i, o = b1 * p, b2 * q
    X = synth.make_x(n, i, seed=9).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(i, o, b1, b2, r, seed=9)]
    monkeypatch.setenv("BLR_BLAST_PATH", "split")
    Y0 = cuda_lib.blast_matmul(X, V, S, U)
    Vt, Ut = cuda_lib.blast_kmajor_factors(V, U)
    monkeypatch.setenv("BLR_WIDE", "1")
    Yk = cuda_lib.blast_matmul(X, Vt, S, Ut, kmajor=True)
    Yw = cuda_lib.blast_matmul(X, V, S, U)
    torch.cuda.synchronize()
    assert torch.equal(Yk, Y0), f"kmajor wide {n, b1, b2, r}"
    assert torch.equal(Yw, Y0), f"paper layout wide {n, b1, b2, r}"
    rows = sample_rows(n, 48)
    ref = orc.blast_forward(to64(X[rows].cpu()), to64(V.cpu()), to64(S.cpu()), to64(U.cpu()))
    assert_parity(Yk[torch.as_tensor(rows, device=DEV)], ref, f"kmajor wide {n, b1, b2, r}")


from tests.test_gpu_fuzz import _cases  # noqa: E402  (the fuzz's seeded shape generator)


@pytest.mark.parametrize("case", _cases("lowrank", 10, 4242) + _cases("blast", 10, 4343))
def test_wide_forced_fuzz(cuda_lib, monkeypatch, case):
    """Every GEMM phase forced onto the wide tiles (BLR_WIDE=1: any width, tile-blocked A too, the
    per-half release, single-half last tiles) over the fuzz's random shapes: bit for bit the default
    plans' result (same products, same K order)."""
    n, i, o, r, b1, b2, _ = case
    X = synth.make_x(n, i, seed=n + i).to(DEV)
    if b1 == 1 and b2 == 1:
        fac = [t.to(DEV) for t in synth.lowrank_factors(i, o, r, seed=o + r)]
        run = lambda: cuda_lib.lowrank_matmul(X, *fac)  # noqa: E731
    else:
        fac = [t.to(DEV) for t in synth.blast_factors(i, o, b1, b2, r, seed=o + r)]
        run = lambda: cuda_lib.blast_matmul(X, *fac)  # noqa: E731
    Y0 = run()
    monkeypatch.setenv("BLR_WIDE", "1")
    Y = run()
    torch.cuda.synchronize()
    assert torch.equal(Y, Y0), f"forced wide {case}"
