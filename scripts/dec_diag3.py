"""Does the small-n path read workspace / output memory it did not write?  Fill both with NaN."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from paper_2512_20861_b200 import synth  # noqa: E402

dev = torch.device("cuda")
n, i, o, r = 16, 4096, 11008, 1488
X = synth.make_x(n, i, seed=21).to(dev)
V, U = [t.to(dev) for t in synth.lowrank_factors(i, o, r, seed=21)]
ref = blr.lowrank_matmul(X, V, U)
torch.cuda.synchronize()
lib = blr.load()
wsb = lib.blr_lowrank_workspace_size(n, i, o, r)
bad = 0
for rep in range(20):
    ws = torch.full((wsb // 4 + 64,), float("nan"), dtype=torch.float32, device=dev)
    Y = torch.full((n, o), float("nan"), dtype=torch.bfloat16, device=dev)
    blr.lowrank_matmul(X, V, U, out=Y, workspace=ws)
    torch.cuda.synchronize()
    d = ~(Y == ref)
    if d.any():
        bad += 1
        nz = d.nonzero()
        print(rep, "differ", int(d.sum()), "nan", int(torch.isnan(Y.float()).sum()), "first", nz[:3].tolist())
print("bad runs", bad, "of 20")
