"""Graph-replayed time of single BLR layer calls (PDL active between the call's kernels, no events
inside): t(layer) = t(graph of R x [flush, call]) - t(graph of R x [flush]) over R.
Usage: python scripts/layer_time.py [n_tokens] [method/model/layer ...]   (default: the C2 layers)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from paper_2512_20861_b200 import configs, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
specs = sys.argv[2:] or [f"{m}/GPT2-S/{l}" for m in ("lowrank", "monarch", "blast") for l in ("c_fc", "c_proj")]
dev = torch.device("cuda")
blr.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
R = 10


def gtime(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best * 1e3  # us


def flush_only():
    for _ in range(R):
        flush.zero_()


t_flush = gtime(flush_only)
for spec in specs:
    method, model, layer = spec.split("/")
    L = configs.table3(model, layer, method)
    X = synth.make_x(n, L.i, device=dev)
    Y = torch.empty(n, L.o, dtype=torch.bfloat16, device=dev)
    if L.method == "lowrank":
        fac = [t.to(dev) for t in synth.lowrank_factors(L.i, L.o, L.r)]
        call = lambda: blr.lowrank_matmul(X, *fac, out=Y)
    elif L.method == "monarch":
        fac = [t.to(dev) for t in synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r_blk)]
        call = lambda: blr.monarch_matmul(X, *fac, L.b1, L.b2, out=Y)
    else:
        fac = [t.to(dev) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r)]
        call = lambda: blr.blast_matmul(X, *fac, out=Y)
    ws = {}

    def body():
        for _ in range(R):
            flush.zero_()
            call()

    t_all = gtime(body)
    print(f"{L.model}.{L.name}.{L.method:8s} n={n}: {(t_all - t_flush) / R:7.1f} us/call (graph, L2 flushed)",
          flush=True)
