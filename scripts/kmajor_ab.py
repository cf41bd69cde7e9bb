"""In-process A/B of the BLAST factor layouts (paper MN-major vs statically re-laid-out K-major,
blr_blast_matmul_kmajor) on the C4 layers: each call captured as a CUDA graph, replays interleaved
with an L2 flush before each."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from paper_2512_20861_b200 import configs, synth  # noqa: E402

dev = torch.device("cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
n = int(os.environ.get("N", 65536))
for name in ("gate_up_proj", "down_proj"):
    L = configs.table3("Llama-7B", name, "blast")
    X = synth.make_x(n, L.i, device=dev)
    V, S, U = [t.to(dev) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r)]
    Vt, Ut = blr.blast_kmajor_factors(V, U)
    Y = torch.empty((n, L.o), dtype=torch.bfloat16, device=dev)
    ws = torch.empty(blr.load().blr_blast_workspace_size(n, L.i, L.o, L.b1, L.b2, L.r), dtype=torch.uint8, device=dev)
    runs = {"paper": lambda: blr.blast_matmul(X, V, S, U, out=Y, workspace=ws),
            "kmajor": lambda: blr.blast_matmul(X, Vt, S, Ut, out=Y, workspace=ws, kmajor=True)}
    graphs = {}
    for k, f in runs.items():
        f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graphs[k] = g
    t = {k: [] for k in graphs}
    for _ in range(9):
        for k, g in graphs.items():
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            t[k].append(a.elapsed_time(b))
    print(name, {k: round(statistics.median(v), 4) for k, v in t.items()})
