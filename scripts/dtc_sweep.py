"""Sweep the tensor-core decode plan (tile width W, K split S) of each launch of a decode call:
graph-replayed call time (L2 flushed by a write, as decode_bench.py) for every forced (W, S) of
launch 0 with launch 1 on its default plan, and vice versa.
    python scripts/dtc_sweep.py [methods] [ns]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BLR_DECODE"] = "1"
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from paper_2512_20861_b200 import configs, synth  # noqa: E402

methods = sys.argv[1].split(",") if len(sys.argv) > 1 else ["lowrank", "blast", "monarch"]
ns = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 16]
dev = torch.device("cuda")
blr.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def gtime(f, reps=20):
    f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        flush.zero_()
        a.record()
        g.replay()
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return ts[len(ts) // 2]


def clear():
    for k in ("BLR_DTC_W0", "BLR_DTC_S0", "BLR_DTC_W1", "BLR_DTC_S1"):
        os.environ.pop(k, None)


for method in methods:
    L = configs.table3("Llama-7B", "gate_up_proj", method)
    if method == "lowrank":
        fac = [t.to(dev) for t in synth.lowrank_factors(L.i, L.o, L.r)]
        call = lambda X: blr.lowrank_matmul(X, *fac)  # noqa: E731
    elif method == "monarch":
        fac = [t.to(dev) for t in synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r // L.b1)]
        call = lambda X: blr.monarch_matmul(X, *fac, L.b1, L.b2)  # noqa: E731
    else:
        fac = [t.to(dev) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r)]
        call = lambda X: blr.blast_matmul(X, *fac)  # noqa: E731
    for n in ns:
        X = synth.make_x(n, L.i, device=dev)
        clear()
        base = gtime(lambda: call(X))
        print(f"{method} n={n}: default {base:.1f} us", flush=True)
        for li in (0, 1):
            res = []
            for w in (64, 128, 256):
                for s in range(1, 9):
                    clear()
                    os.environ[f"BLR_DTC_W{li}"] = str(w)
                    if not (method == "blast" and li == 0):
                        os.environ[f"BLR_DTC_S{li}"] = str(s)
                    elif s > 1:
                        continue
                    try:
                        t = gtime(lambda: call(X))
                    except Exception:
                        continue
                    res.append((t, w, s))
            res.sort()
            print(f"  launch {li}: " + "  ".join(f"W{w}/S{s} {t:.1f}" for t, w, s in res[:8]), flush=True)
        clear()
