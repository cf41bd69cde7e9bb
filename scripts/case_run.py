"""Run one BLAST case (n i o r b1 b2 from argv) and compare with the oracle on sampled rows;
prints OK / BAD / the CUDA error.  For bisecting a fuzz failure across env knobs, one process each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2512_20861_b200 import synth  # noqa: E402

n, i, o, r, b1, b2 = [int(x) for x in sys.argv[1:7]]
dev = torch.device("cuda")
X = synth.make_x(n, i, seed=n + i).to(dev)
V, S, U = [t.to(dev) for t in synth.blast_factors(i, o, b1, b2, r, seed=o + r)]
try:
    Y = blr.blast_matmul(X, V, S, U)
    torch.cuda.synchronize()
    rows = np.arange(0, n, max(1, n // 37))
    ref = orc.blast_forward(X[rows].float().cpu().numpy().astype(np.float64), V.float().cpu().numpy(),
                            S.float().cpu().numpy(), U.float().cpu().numpy())
    g = Y[torch.as_tensor(rows, device=dev)].float().cpu().numpy()
    rel = np.linalg.norm(g - ref) / np.linalg.norm(ref)
    print("OK" if rel < 5e-3 else f"BAD rel={rel:.3e}", "launches", blr.last_launch_count())
except Exception as e:  # noqa: BLE001
    print("ERR", str(e).splitlines()[0][:120])
