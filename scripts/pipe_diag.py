"""Diagnose the pipelined BLAST layer against the three-launch path: which token tiles / output
blocks differ, over a few role splits and repetitions."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from paper_2512_20861_b200 import synth  # noqa: E402

dev = torch.device("cuda")
n, b1, b2, r, p, q = [int(x) for x in (sys.argv[1:7] if len(sys.argv) > 6 else (640, 16, 16, 208, 48, 40))]
X = synth.make_x(n, b1 * p, seed=11).to(dev)
V, S, U = [t.to(dev) for t in synth.blast_factors(b1 * p, b2 * q, b1, b2, r, seed=11)]
os.environ["BLR_PIPE"] = "0"
Y3 = blr.blast_matmul(X, V, S, U)
os.environ["BLR_PIPE"] = "1"
for split in ["1,1", "4,4"]:
  os.environ["BLR_PIPE_SPLIT"] = split
  for win in ["1", "2", "3", "5", "8"]:
    os.environ["BLR_PIPE_WIN"] = win
    for rep in range(1):
        Yp = blr.blast_matmul(X, V, S, U)
        torch.cuda.synchronize()
        d = (Yp.float() - Y3.float()).abs() > 0
        bad_t = sorted(set((d.any(dim=1).nonzero().flatten() // 128).tolist()))
        bad_k = sorted(set((d.any(dim=0).nonzero().flatten() // q).tolist()))
        print(f"split {split} win {win} rep {rep}: {int(d.sum())} differ; token tiles {bad_t}; out blocks {bad_k[:20]}")
