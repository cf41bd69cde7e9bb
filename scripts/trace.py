"""Intra-kernel timeline: per-CTA %globaltimer stamps for each GEMM-kernel launch of one layer call.
(Needs a debug build of the GEMM kernels' trace stamps: BLR_NVCC_EXTRA=-DBLR_DEBUG_KNOBS before
__graft_entry__.build(); release builds compile the stamps out.)
stamps: 0 entry, 1 setup done, 2 after griddepcontrol.wait, 3 MMA got first stage, 4 last MMA commit,
5 epilogue done (warp 2), 6 bulk stores drained, 7 exit."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_20861_b200 as blr
from paper_2512_20861_b200 import configs, synth
method, model, layer = (sys.argv[1:4] + ["lowrank", "GPT2-S", "c_fc"][len(sys.argv[1:4]):])[:3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 8192
L = configs.table3(model, layer, method)
lib = blr.load()
lib.blr_debug_trace.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda")
if L.method == "lowrank":
    fac = [t.to(dev) for t in synth.lowrank_factors(L.i, L.o, L.r)]; run = lambda X: blr.lowrank_matmul(X, *fac)
elif L.method == "monarch":
    fac = [t.to(dev) for t in synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r_blk)]; run = lambda X: blr.monarch_matmul(X, *fac, L.b1, L.b2)
else:
    fac = [t.to(dev) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r)]; run = lambda X: blr.blast_matmul(X, *fac)
X = synth.make_x(n, L.i, device=dev)
run(X); run(X); torch.cuda.synchronize()
buf = torch.zeros(4 * 256 * 128, dtype=torch.int64, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev); flush.zero_()
fmode = os.environ.get("TRACE_FLUSH", "zero")  # zero: dirty L2 (bench default) | read: clean L2 | none
if fmode == "read":
    torch.cuda.synchronize(); flush.view(torch.float32).sum()
elif fmode == "none":
    run(X)
lib.blr_debug_trace(buf.data_ptr()); run(X); lib.blr_debug_trace(None); torch.cuda.synchronize()
t = buf.view(4, 256, 128).cpu().clone()
# stamps other than [0] (globaltimer ns) and [8] (clock64 at entry) are clock64 values
ghz = float(os.environ.get("TRACE_GHZ", "1.92"))
for k in range(4):
    for c in range(256):
        row = t[k, c]
        if row[0] == 0: continue
        for f in range(1, 128):
            if f != 8 and row[f] != 0:
                row[f] = row[0] + int((int(row[f]) - int(row[8])) / ghz)
print(f"{L.model}.{L.name}.{L.method} n={n}")
for k in range(4):
    tk = t[k]; ctas = tk[:, 0] > 0
    if not ctas.any(): break
    tk = tk[ctas].double()
    t0 = tk[:, 0].min() if not os.environ.get("TRACE_COMMON_T0") else t[:, :, 0][t[:, :, 0] > 0].double().min()
    rel = (tk - t0) / 1000.0  # us
    names = ["entry", "setup", "gdwait", "1stfull", "lastmma", "epidone", "drained", "exit"]
    if os.environ.get("TRACE_BRIEF"): names = ["gdwait", "lastmma", "drained"]
    print(f" launch {k}: {int(ctas.sum())} CTAs; us since first CTA entry (min/med/max):")
    for c, nm in enumerate(names):
        col = rel[:, c][tk[:, c] > 0]
        if len(col): print(f"   {nm:8s} {col.min():7.2f} {col.median():7.2f} {col.max():7.2f}")
    c0 = tk[0]
    mm = [(c0[16 + i] - t0).item() / 1000 for i in range(24) if c0[16 + i] > 0]
    ep = [(c0[40 + i] - t0).item() / 1000 for i in range(24) if c0[40 + i] > 0]
    setup = [(tk[:, f][tk[:, f] > 0] - tk[:, 0][tk[:, f] > 0]).median().item() / 1000 for f in (13, 14, 15) if (tk[:, f] > 0).any()]
    if setup and L.method != "blast": print("   median since own entry: barriers init / TMEM alloc / tile table us:", " ".join(f"{v:.2f}" for v in setup))
    extra = [(c0[f] - t0).item() / 1000 for f in (9, 10, 12, 13, 14, 11) if c0[f] > 0]
    if extra: print("   CTA0 epilogue tile0 (S staged / tfull / 1st ld / sc0 / sc1 / computed) us:", " ".join(f"{v:.2f}" for v in extra))
    print("   CTA0 per-tile MMA-commit us:", " ".join(f"{v:.2f}" for v in mm))
    print("   CTA0 per-tile epilogue-done us:", " ".join(f"{v:.2f}" for v in ep))
    pi = [(c0[64 + i] - t0).item() / 1000 for i in range(32) if c0[64 + i] > 0]
    mf = [(c0[96 + i] - t0).item() / 1000 for i in range(32) if c0[96 + i] > 0]
    print("   CTA0 producer issue  us:", " ".join(f"{v:.2f}" for v in pi))
    print("   CTA0 MMA full-ready  us:", " ".join(f"{v:.2f}" for v in mf))
