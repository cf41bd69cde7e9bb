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
