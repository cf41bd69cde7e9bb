"""Run one BLR layer call a few times (for ncu captures): python scripts/one_call.py method model layer n reps"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_20861_b200 as blr
from paper_2512_20861_b200 import configs, synth
method, model, layer = sys.argv[1:4]
n = int(sys.argv[4]); reps = int(sys.argv[5])
L = configs.table3(model, layer, method)
dev = torch.device("cuda")
X = synth.make_x(n, L.i, device=dev)
if L.method == "lowrank":
    fac = [t.to(dev) for t in synth.lowrank_factors(L.i, L.o, L.r)]; run = lambda: blr.lowrank_matmul(X, *fac)
elif L.method == "monarch":
    fac = [t.to(dev) for t in synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r_blk)]; run = lambda: blr.monarch_matmul(X, *fac, L.b1, L.b2)
else:
    fac = [t.to(dev) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r)]; run = lambda: blr.blast_matmul(X, *fac)
for _ in range(reps):
    run()
torch.cuda.synchronize()
