"""One small-token call (for ncu): python scripts/dtc_one.py METHOD N [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BLR_DECODE", "1")
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from paper_2512_20861_b200 import configs, synth  # noqa: E402

method, n = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
L = configs.table3("Llama-7B", "gate_up_proj", method)
dev = torch.device("cuda")
X = synth.make_x(n, L.i, device=dev)
if method == "lowrank":
    fac = [t.to(dev) for t in synth.lowrank_factors(L.i, L.o, L.r)]
    f = lambda: blr.lowrank_matmul(X, *fac)  # noqa: E731
elif method == "monarch":
    fac = [t.to(dev) for t in synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r // L.b1)]
    f = lambda: blr.monarch_matmul(X, *fac, L.b1, L.b2)  # noqa: E731
else:
    fac = [t.to(dev) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r)]
    f = lambda: blr.blast_matmul(X, *fac)  # noqa: E731
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(reps):
    flush.zero_()
    f()
torch.cuda.synchronize()
