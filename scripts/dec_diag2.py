"""Fresh-process decode determinism check mimicking tests/test_gpu_decode.py."""
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
Y1 = blr.lowrank_matmul(X, V, U)
Y2 = blr.lowrank_matmul(X, V, U)
Y3 = blr.lowrank_matmul(X[5:6].contiguous(), V, U)
torch.cuda.synchronize()
Y4 = blr.lowrank_matmul(X, V, U)
torch.cuda.synchronize()
for name, A, B in (("Y1-Y2", Y1, Y2), ("Y1-Y4", Y1, Y4), ("Y2-Y4", Y2, Y4), ("Y3-Y1[5]", Y3[0], Y1[5])):
    d = A != B
    if d.any():
        nz = d.nonzero()
        print(name, "differ:", int(d.sum()), "first", nz[:4].tolist(), "max", float((A.float() - B.float()).abs().max()))
    else:
        print(name, "equal")
