"""Output-block sharding on one GPU: each emulated rank runs the single-GPU
kernels on its output blocks' factors (paper_2512_20861_b200.dist.*_local_factors); the
column blocks, concatenated in rank order, must equal the unsharded GPU output bit for bit (the
per-element arithmetic does not depend on which other blocks are computed) and meet the oracle
tolerance.  The NCCL all-gather itself is host plumbing, tested over gloo in test_dist.py."""
import pytest
import torch

from oracle import oracle as orc
from paper_2512_20861_b200 import dist as bdist
from paper_2512_20861_b200 import synth
from tests.parity import assert_parity, to64

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("world", [2, 4, 16])
def test_blast_output_block_sharded(cuda_lib, world):
    n, b1, b2, r, p, q = 300, 16, 16, 64, 32, 48
    X = synth.make_x(n, b1 * p, seed=31).to(DEV)
    V, S, U = [t.to(DEV) for t in synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=31)]
    full = cuda_lib.blast_matmul(X, V, S, U)
    parts = []
    for rank in range(world):
        k0, k1 = bdist.shard_blocks(b2, rank, world)
        Vl, Sl, Ul = bdist.blast_local_factors(V, S, U, k0, k1)
        parts.append(cuda_lib.blast_matmul(X, Vl, Sl, Ul))
    Y = torch.cat(parts, dim=1)
    torch.cuda.synchronize()
    assert torch.equal(Y, full)
    assert_parity(Y, orc.blast_forward(to64(X.cpu()), to64(V.cpu()), to64(S.cpu()), to64(U.cpu())), "BLAST sharded")


@pytest.mark.parametrize("layout", [orc.B2_FASTEST, orc.RPRIME_FASTEST])
@pytest.mark.parametrize("world", [2, 4])
def test_monarch_output_block_sharded(cuda_lib, layout, world):
    n, b1, b2, rp, p, q = 260, 4, 4, 48, 192, 768  # GPT2-S c_fc Monarch
    X = synth.make_x(n, b1 * p, seed=32).to(DEV)
    V, U = [t.to(DEV) for t in synth.monarch_factors(b1 * p, b2 * q, b1, b2, rp, seed=32)]
    full = cuda_lib.monarch_matmul(X, V, U, b1, b2, v_layout=layout)
    parts = []
    for rank in range(world):
        k0, k1 = bdist.shard_blocks(b2, rank, world)
        Vl, Ul = bdist.monarch_local_factors(V, U, b2, rp, k0, k1, layout)
        parts.append(cuda_lib.monarch_matmul(X, Vl, Ul, b1, k1 - k0, v_layout=layout))
    Y = torch.cat(parts, dim=1)
    torch.cuda.synchronize()
    assert torch.equal(Y, full)
    ref = orc.monarch_forward(to64(X.cpu()), to64(V.cpu()), to64(U.cpu()), b1, b2, layout)
    assert_parity(Y, ref, "Monarch sharded")


def test_lowrank_output_column_sharded(cuda_lib):
    n, i, o, r = 257, 768, 3072, 192
    X = synth.make_x(n, i, seed=33).to(DEV)
    V, U = [t.to(DEV) for t in synth.lowrank_factors(i, o, r, seed=33)]
    full = cuda_lib.lowrank_matmul(X, V, U)
    cols = [(0, 1024), (1024, 2048), (2048, 3072)]
    Y = torch.cat([cuda_lib.lowrank_matmul(X, *bdist.lowrank_local_factors(V, U, c0, c1)) for c0, c1 in cols], dim=1)
    torch.cuda.synchronize()
    assert torch.equal(Y, full)
