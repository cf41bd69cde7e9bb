"""Per-launch breakdown of the small-token (decode) path: each launch of one call bracketed by the
C-ABI profiling hook's events (serialised: upper bounds), graph-replayed with L2 flushed."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BLR_DECODE", "1")
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from paper_2512_20861_b200 import configs, synth  # noqa: E402

LAYERS = [("lowrank", "Llama-7B", "gate_up_proj"), ("monarch", "Llama-7B", "gate_up_proj"),
          ("blast", "Llama-7B", "gate_up_proj")]
dev = torch.device("cuda")
lib = blr.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
for method, model, name in LAYERS:
    L = configs.table3(model, name, method)
    if method == "lowrank":
        fac = [t.to(dev) for t in synth.lowrank_factors(L.i, L.o, L.r)]
        f = lambda X: blr.lowrank_matmul(X, *fac)  # noqa: E731
    elif method == "monarch":
        fac = [t.to(dev) for t in synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r // L.b1)]
        f = lambda X: blr.monarch_matmul(X, *fac, L.b1, L.b2)  # noqa: E731
    else:
        fac = [t.to(dev) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r)]
        f = lambda X: blr.blast_matmul(X, *fac)  # noqa: E731
    for n in (1, 8, 16):
        X = synth.make_x(n, L.i, device=dev)
        f(X)
        torch.cuda.synchronize()
        nl = lib.blr_last_launch_count() if hasattr(lib, "blr_last_launch_count") else 8
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * 16)]
        for e in ev:
            e.record(st)
        arr = (ctypes.c_void_p * 32)(*[e.cuda_event for e in ev])
        got = [0]

        def step():
            lib.blr_profile_begin(arr, 32)
            f(X)
            got[0] = lib.blr_profile_end()
        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        acc = [0.0] * got[0]
        R = 20
        for _ in range(R):
            flush.zero_()
            g.replay()
            torch.cuda.synchronize()
            for j in range(got[0]):
                acc[j] += ev[2 * j].elapsed_time(ev[2 * j + 1]) * 1e3 / R
        print(f"{model}.{name}.{method} n={n}: " + " ".join(f"{a:6.1f}" for a in acc) + f"  sum={sum(acc):.1f} us")
