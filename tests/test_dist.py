"""Multi-process host logic of token sharding, world_size 2 over gloo on CPU (-m "not gpu")."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_20861_b200 import dist as bdist


def test_shard_rows_partition():
    for n in (0, 1, 7, 128, 8192, 65537):
        for world in (1, 2, 3, 8):
            spans = [bdist.shard_rows(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(0)
        n, i, o = 37, 16, 24
        x = torch.randn(n, i, generator=g, dtype=torch.float64)
        w = torch.randn(i, o, generator=g, dtype=torch.float64)
        # a row-wise layer: sharded + gathered must equal the unsharded product exactly
        y = bdist.sharded_forward(lambda xs: xs @ w, x, gather=True)
        ok_gather = torch.equal(y, x @ w)
        t = bdist.max_over_ranks(1.0 + rank)
        q.put((rank, ok_gather, t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_gather_and_max():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(ok for _, ok, _ in res)
    assert all(t == 2.0 for _, _, t in res)  # max over ranks of (1 + rank)


# ------------------------------------------- output-block sharding, host logic --
def _blast_dense_ref(X, V, S, U):
    """fp64 reference through the oracle (the GPU kernels replace this on a device)."""
    from oracle import oracle as orc
    return torch.from_numpy(orc.blast_forward(X.numpy(), V.numpy(), S.numpy(), U.numpy()))


def _worker_cols(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(3)
        n, b1, b2, r, p, qd = 5, 3, 5, 8, 4, 6   # b2 = 5 blocks over 2 ranks: uneven split
        X = torch.randn(n, b1 * p, generator=g, dtype=torch.float64)
        V = torch.randn(b1, p, r, generator=g, dtype=torch.float64)
        S = torch.randn(b1, b2, r, generator=g, dtype=torch.float64)
        U = torch.randn(b2, r, qd, generator=g, dtype=torch.float64)

        def local(k0, k1):
            Vl, Sl, Ul = bdist.blast_local_factors(V, S, U, k0, k1)
            if k1 == k0:
                return torch.zeros((n, 0), dtype=torch.float64)
            return _blast_dense_ref(X, Vl, Sl, Ul)

        y = bdist.output_sharded_forward(local, b2, qd)
        ok = torch.allclose(y, _blast_dense_ref(X, V, S, U), rtol=1e-12, atol=1e-12)
        q.put((rank, ok, tuple(y.shape)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_output_block_sharded_blast():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_cols, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(ok for _, ok, _ in res), res
    assert all(shape == (5, 30) for _, _, shape in res)


def test_monarch_local_factors_select_the_block_rows():
    """The V rows of output blocks [k0, k1) in both layouts (pure index bookkeeping)."""
    from oracle import oracle as orc
    b1, b2, rp, p, qd, n = 2, 4, 3, 5, 6, 3
    g = torch.Generator().manual_seed(4)
    X = torch.randn(n, b1 * p, generator=g, dtype=torch.float64)
    V = torch.randn(b1, rp * b2, p, generator=g, dtype=torch.float64)
    U = torch.randn(b2, qd, b1 * rp, generator=g, dtype=torch.float64)
    for layout in (orc.B2_FASTEST, orc.RPRIME_FASTEST):
        full = orc.monarch_forward(X.numpy(), V.numpy(), U.numpy(), b1, b2, layout)
        for k0, k1 in ((0, 1), (1, 3), (2, 4)):
            Vl, Ul = bdist.monarch_local_factors(V, U, b2, rp, k0, k1, layout)
            part = orc.monarch_forward(X.numpy(), Vl.numpy(), Ul.numpy(), b1, k1 - k0, layout)
            assert abs(part - full[:, k0 * qd:k1 * qd]).max() < 1e-12, (layout, k0, k1)



def test_bench_gpus2_self_launch_dry_run():
    """`python bench.py --gpus 2` starts two ranks itself (torch.distributed.run, 127.0.0.1) and
    strong-shards C4's 65,536 tokens contiguously (8,192 per GPU at N = 8); the --dry-run
    plumbing pass runs the rank/shard logic over gloo without touching a GPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["shards"] == [[0, 32768], [32768, 65536]]
    assert [bdist.shard_rows(65536, r, 8) for r in range(8)] == [(8192 * r, 8192 * (r + 1)) for r in range(8)]
