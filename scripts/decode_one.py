import sys, os
sys.path.insert(0, '/root/repo')
os.environ.setdefault("BLR_DECODE", "1")
import torch, paper_2512_20861_b200 as blr
from paper_2512_20861_b200 import configs, synth
L = configs.table3("Llama-7B", "gate_up_proj", "lowrank")
dev = torch.device("cuda")
fac = [t.to(dev) for t in synth.lowrank_factors(L.i, L.o, L.r)]
for n in (1, 16):
    X = synth.make_x(n, L.i, device=dev)
    for _ in range(3): blr.lowrank_matmul(X, *fac)
torch.cuda.synchronize()
