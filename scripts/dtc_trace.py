"""Timeline of the tensor-core decode launches (debug globaltimer stamps per CTA, ns):
(Needs a debug build: BLR_NVCC_EXTRA=-DBLR_DEBUG_KNOBS before __graft_entry__.build(); release builds
compile the stamps out.)
    python scripts/dtc_trace.py METHOD N
stamps: 0 start, 1 producer go, 2 consumer past wait, 3 A staged, 8.. first ring stages landed,
4 mainloop done, 5 after cluster sync 1, 6 reduce done, 7 end."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BLR_DECODE", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from paper_2512_20861_b200 import configs, synth  # noqa: E402

method, n = sys.argv[1], int(sys.argv[2])
L = configs.table3("Llama-7B", "gate_up_proj", method)
dev = torch.device("cuda")
lib = blr.load()
lib.blr_debug_trace.argtypes = [ctypes.c_void_p]
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
f(); f()
buf = torch.zeros(2 * 128 * 256, dtype=torch.int64, device=dev)
flush.zero_()
torch.cuda.synchronize()
lib.blr_debug_trace(buf.data_ptr())
f()
lib.blr_debug_trace(None)
torch.cuda.synchronize()
t = buf.view(2, 2048, 16).cpu().numpy().astype(np.float64)
t0 = t[t[:, :, 0] > 0][:, 0].min()
for li in range(2):
    a = t[li]
    a = a[a[:, 0] > 0]
    if not len(a):
        continue
    print(f"launch {li}: {len(a)} CTAs; kernel span {(a[:, 7].max() - a[:, 0].min()) / 1e3:.2f} us "
          f"(from first CTA start of the call: start {(a[:, 0].min() - t0) / 1e3:.2f}, end {(a[:, 7].max() - t0) / 1e3:.2f})")
    def q(x):
        x = x / 1e3
        return f"p0 {np.min(x):6.2f} p50 {np.median(x):6.2f} p90 {np.percentile(x, 90):6.2f} max {np.max(x):6.2f}"
    base = a[:, 0]
    print("  start - first start  ", q(base - base.min()))
    for k, nm in [(1, "producer go"), (2, "consumer past wait"), (3, "A staged"), (8, "stage0 landed"),
                  (9, "stage1 landed"), (15, "stage7 landed"), (4, "mainloop done"), (5, "cluster sync 1"),
                  (6, "reduce done"), (7, "end")]:
        m = a[:, k] > 0
        if m.any():
            print(f"  {nm:22s}", q(a[m, k] - base[m]))
