"""The pipelined BLAST layer (one launch; S1 / S2 / S3 roles hand token tiles over through ready
counters) against the fp64 oracle, and bit for bit against the three-launch
split path (same kernels, same rounding points, same K order per output element)."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import synth
from tests.parity import assert_parity, sample_rows, to64

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda")


@pytest.mark.parametrize("n,b1,b2,r,p,q,split", [
    (1024, 16, 16, 272, 64, 88, None),      # 8 token tiles, ragged K tail (r/8 = 34 panels)
    (1000, 16, 16, 128, 32, 48, None),      # ragged token tail inside a CTA pair's 256 rows
    (2304, 16, 16, 376, 64, 64, "2,1"),     # one cluster per producer role: long waits
    (4096, 8, 12, 512, 64, 96, "3,2"),      # b1 != b2 (asymmetric S)
    (640, 16, 16, 208, 48, 40, "1,1"),      # every role at its minimum
])
def test_pipe_parity_and_bitwise(cuda_lib, monkeypatch, n, b1, b2, r, p, q, split):
    monkeypatch.setenv("BLR_BLAST_PATH", "split")
    i, o = b1 * p, b2 * q
    X = synth.make_x(n, i, seed=11).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(i, o, b1, b2, r, seed=11)]
    monkeypatch.setenv("BLR_PIPE", "0")
    Y3 = cuda_lib.blast_matmul(X, V, S, U)
    monkeypatch.setenv("BLR_PIPE", "1")
    if split:
        monkeypatch.setenv("BLR_PIPE_SPLIT", split)
    Yp = cuda_lib.blast_matmul(X, V, S, U)
    assert cuda_lib.last_launch_count() == 1, "the pipelined layer is one launch"
    torch.cuda.synchronize()
    rows = sample_rows(n, 96)
    ref = orc.blast_forward(to64(X[rows].cpu()), to64(V), to64(S), to64(U))
    assert_parity(Yp[torch.as_tensor(rows, device=DEV)], ref, f"pipe {n, b1, b2, r, p, q}")
    assert torch.equal(Yp, Y3), "pipelined layer differs from the three-launch split path"


def test_pipe_repeatable_and_row_independent(cuda_lib, monkeypatch):
    """Bitwise run-to-run determinism (no atomics in the data path; the counters only order it),
    and row independence through the pipelined layer."""
    monkeypatch.setenv("BLR_PIPE", "1")
    n, b1, b2, r, p, q = 1536, 16, 16, 160, 32, 32
    X = synth.make_x(n, b1 * p, seed=12).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=12)]
    Y1 = cuda_lib.blast_matmul(X, V, S, U)
    Y2 = cuda_lib.blast_matmul(X, V, S, U)
    assert torch.equal(Y1, Y2)
    perm = torch.randperm(n, generator=torch.Generator().manual_seed(3)).to(DEV)
    Yp = cuda_lib.blast_matmul(X[perm].contiguous(), V, S, U)
    assert torch.equal(Yp, Y1[perm])


def test_pipe_nonfinite_row_stays_local(cuda_lib, monkeypatch):
    """A NaN token row poisons only its own output row (row independence, IEEE propagation)."""
    monkeypatch.setenv("BLR_PIPE", "1")
    n, b1, b2, r, p, q = 768, 16, 16, 200, 32, 32
    X = synth.make_x(n, b1 * p, seed=13)
    X[300, 5] = float("nan")
    X = X.to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=13)]
    Y = cuda_lib.blast_matmul(X, V, S, U).float()
    bad = ~torch.isfinite(Y).all(dim=1)
    assert bad[300].item()
    bad[300] = False
    assert not bad.any()


@pytest.mark.parametrize("n", [640, 1152, 1300])
def test_pair_s1_odd_token_tiles(cuda_lib, monkeypatch, n):
    """Split path with S1 as CTA pairs (256-row tiles) over an odd number of 128-token tiles: the
    pair's second tile past n_tok must not store (its tile-blocked box would alias the next
    group's first tile; found through the pipelined layer, where S1 always runs as pairs)."""
    monkeypatch.setenv("BLR_BLAST_PATH", "split")
    monkeypatch.setenv("BLR_PAIR", "2")
    b1, b2, r, p, q = 16, 16, 208, 48, 40
    X = synth.make_x(n, b1 * p, seed=14).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=14)]
    Y = cuda_lib.blast_matmul(X, V, S, U)
    torch.cuda.synchronize()
    rows = np.concatenate([np.arange(0, 128, 7), sample_rows(n, 40)])
    ref = orc.blast_forward(to64(X[rows].cpu()), to64(V), to64(S), to64(U))
    assert_parity(Y[torch.as_tensor(rows, device=DEV)], ref, f"pair S1 n={n}")


@pytest.mark.parametrize("n,b1,b2,r,p,q", [
    (1000, 16, 16, 272, 64, 88),     # ragged tails, r % 64 != 0
    (4096, 8, 12, 512, 64, 96),      # b1 != b2
    (130, 16, 16, 1488, 256, 688),   # Llama-7B gate/up shapes (C4)
    (130, 16, 16, 1488, 688, 256),   # Llama-7B down shapes (C4)
])
def test_kmajor_factor_layout(cuda_lib, n, b1, b2, r, p, q):
    """blr_blast_matmul_kmajor (statically re-laid-out K-major V, U) is the same
    function of the same factors: bitwise equal to the paper layout and within tolerance of the
    fp64 oracle (which takes the paper layout)."""
    i, o = b1 * p, b2 * q
    X = synth.make_x(n, i, seed=15).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(i, o, b1, b2, r, seed=15)]
    Vt, Ut = cuda_lib.blast_kmajor_factors(V, U)
    Y = cuda_lib.blast_matmul(X, V, S, U)
    Yk = cuda_lib.blast_matmul(X, Vt, S, Ut, kmajor=True)
    torch.cuda.synchronize()
    rows = sample_rows(n, 64)
    ref = orc.blast_forward(to64(X[rows].cpu()), to64(V), to64(S), to64(U))
    assert_parity(Yk[torch.as_tensor(rows, device=DEV)], ref, f"kmajor {n, b1, b2, r, p, q}")
    assert torch.equal(Yk, Y)


def test_kmajor_unsupported_paths_enqueue_nothing(cuda_lib):
    """Outside the split tensor-core path the K-major entry point refuses before any launch."""
    from paper_2512_20861_b200 import BLRError
    X = synth.make_x(64, 768, seed=16).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(768, 768, 4, 4, 16, seed=16)]  # b1 r <= 512: fused path
    Vt, Ut = cuda_lib.blast_kmajor_factors(V, U)
    with pytest.raises(BLRError):
        cuda_lib.blast_matmul(X, Vt, S, Ut, kmajor=True)
