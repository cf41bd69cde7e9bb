"""Time single BLR layer calls (per kernel launch, CUDA events) across token counts to separate
fixed per-launch cost from per-token cost.  Usage: python scripts/scan.py [method] [model] [layer]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from paper_2512_20861_b200 import configs, synth  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "lowrank"
model = sys.argv[2] if len(sys.argv) > 2 else "GPT2-S"
layer = sys.argv[3] if len(sys.argv) > 3 else "c_fc"
L = configs.table3(model, layer, method)
lib = blr.load()
dev = torch.device("cuda")
if L.method == "lowrank":
    fac = [t.to(dev) for t in synth.lowrank_factors(L.i, L.o, L.r)]
    run = lambda X: blr.lowrank_matmul(X, *fac)
elif L.method == "monarch":
    fac = [t.to(dev) for t in synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r_blk)]
    run = lambda X: blr.monarch_matmul(X, *fac, L.b1, L.b2)
else:
    fac = [t.to(dev) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r)]
    run = lambda X: blr.blast_matmul(X, *fac)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
print(f"{L.model}.{L.name}.{L.method} i={L.i} o={L.o} r={L.r} b={L.b}")
for n in [int(x) for x in os.environ.get("SCAN_N", "128,512,2048,8192,32768").split(",")]:
    X = synth.make_x(n, L.i, device=dev)
    run(X)
    nl = lib.blr_last_launch_count()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * nl)]
    for e in evs:
        e.record()
    tot = [0.0] * nl
    reps = 20
    for _ in range(reps):
        flush.zero_()
        arr = (ctypes.c_void_p * (2 * nl))(*[e.cuda_event for e in evs])
        lib.blr_profile_begin(arr, 2 * nl)
        run(X)
        lib.blr_profile_end()
        torch.cuda.synchronize()
        for j in range(nl):
            tot[j] += evs[2 * j].elapsed_time(evs[2 * j + 1]) / reps
    print(f"  n={n:6d}: " + "  ".join(f"k{j}={t*1e3:8.1f}us" for j, t in enumerate(tot)))
