"""Per-stage timeline of one CTA of a GEMM launch (debug trace stamps, clock64): producer issue
(Needs a debug build of the GEMM kernels' trace stamps: BLR_NVCC_EXTRA=-DBLR_DEBUG_KNOBS before
__graft_entry__.build(); release builds compile the stamps out.)
time and MMA start time of the first 32 ring steps, to tell a load-latency-bound mainloop (MMA
start = issue + latency, gaps > the MMA time) from an MMA-bound one.
    python scripts/trace_steps.py blast Llama-7B gate_up_proj 65536 <launch index> [cta]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_20861_b200 as blr
from paper_2512_20861_b200 import configs, synth
method, model, layer, n, li = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
ctas = [int(c) for c in sys.argv[6].split(",")] if len(sys.argv) > 6 else [0, 1, 70, 71]
L = configs.table3(model, layer, method)
lib = blr.load()
lib.blr_debug_trace.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda")
fac = [t.to(dev) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r)] if method == "blast" else \
      [t.to(dev) for t in synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r_blk)]
run = (lambda X: blr.blast_matmul(X, *fac)) if method == "blast" else (lambda X: blr.monarch_matmul(X, *fac, L.b1, L.b2))
X = synth.make_x(n, L.i, device=dev)
run(X); run(X); torch.cuda.synchronize()
buf = torch.zeros(4 * 256 * 128, dtype=torch.int64, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev); flush.zero_()
lib.blr_debug_trace(buf.data_ptr()); run(X); lib.blr_debug_trace(None); torch.cuda.synchronize()
t = buf.view(4, 256, 128).cpu()
for c in ctas:
    row = t[li, c]
    prod = [int(row[64 + i]) for i in range(32) if row[64 + i] != 0]
    mma = [int(row[96 + i]) for i in range(32) if row[96 + i] != 0]
    base = min(prod[0], mma[0]) if prod and mma else 0
    print(f"launch {li} CTA {c}: step: producer issue / MMA start (clk since first), MMA gap")
    for i in range(min(len(prod), len(mma))):
        gap = mma[i] - mma[i - 1] if i else 0
        print(f"  {i:2d} {prod[i] - base:8d} {mma[i] - base:8d}   gap {gap:6d}   wait-after-issue {mma[i] - prod[i]:7d}")
