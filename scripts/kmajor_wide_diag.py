import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2512_20861_b200 as blr
from paper_2512_20861_b200 import synth
import os
DEV=torch.device("cuda")
n,b1,b2,r,p,q=300,6,6,200,128,512
X=synth.make_x(n,b1*p,seed=9).to(DEV)
V,S,U=[t.to(DEV) for t in synth.blast_factors(b1*p,b2*q,b1,b2,r,seed=9)]
os.environ["BLR_BLAST_PATH"]="split"
Vt,Ut=blr.blast_kmajor_factors(V,U)
os.environ["BLR_WIDE"]="1"
for nm,f in [("paper",lambda: blr.blast_matmul(X,V,S,U)),("kmajor",lambda: blr.blast_matmul(X,Vt,S,Ut,kmajor=True))]:
    try:
        f(); torch.cuda.synchronize(); print(nm,"ok")
    except Exception as e:
        print(nm,"ERR",e)
