"""Decode-path determinism diagnostic: repeat one small-n call and report which outputs change."""
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
for env in ["", "BLR_DTC_S0=1", "BLR_DTC_S1=1", "BLR_NO_PDL=1", "BLR_DTC_S0=1 BLR_DTC_S1=1"]:
    for k in ["BLR_DTC_S0", "BLR_DTC_S1", "BLR_NO_PDL"]:
        os.environ.pop(k, None)
    for kv in env.split():
        a, b = kv.split("=")
        os.environ[a] = b
    Y0 = blr.lowrank_matmul(X, V, U)
    bad = 0
    cols = set()
    for rep in range(60):
        Y = blr.lowrank_matmul(X, V, U)
        d = Y != Y0
        if d.any():
            bad += 1
            cols.update((d.any(dim=0).nonzero().flatten() // 64).tolist()[:8])
    torch.cuda.synchronize()
    print(f"[{env or 'default'}] {bad}/60 runs differ; 64-col tiles {sorted(cols)[:12]}")
