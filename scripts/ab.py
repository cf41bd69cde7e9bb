"""In-process A/B of plan knobs on one workload: every setting's step is captured as its own CUDA
graph (the library reads its env knobs at call time), then the graphs are replayed interleaved
with an L2 flush before each replay, so box-to-box clock/power variance cancels out.

    python scripts/ab.py C4 "" "BLR_WIDE=1" "BLR_WIDE=1 BLR_BUFS=1" [--reps 15] [--layer j]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_20861_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("settings", nargs="+")
ap.add_argument("--reps", type=int, default=15)
ap.add_argument("--layer", type=int, default=-1, help="time only layer j of the workload")
args = ap.parse_args()
w = configs.WORKLOADS[args.config]
if args.layer >= 0:
    w = configs.Workload(w.key, w.desc, w.n, (w.layers[args.layer],), w.fp8z)
dev = torch.device("cuda")
arm = bench.Arm(w, w.n, dev, seed=0)
flush = bench.L2Flush(512 << 20, dev, "write+read")
graphs = []
base_env = dict(os.environ)
for st in args.settings:
    os.environ.clear()
    os.environ.update(base_env)
    for kv in st.split():
        k, v = kv.split("=", 1)
        os.environ[k] = v
    graphs.append(bench.graph_of(arm.step))
os.environ.clear()
os.environ.update(base_env)
times = [[] for _ in graphs]
for _ in range(3):
    for g in graphs:
        g.replay()
torch.cuda.synchronize()
for _ in range(args.reps):
    for i, g in enumerate(graphs):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        times[i].append(a.elapsed_time(b))
for st, t in zip(args.settings, times):
    print(f"{args.config} layer={args.layer} [{st or 'default'}] median {statistics.median(t):.4f} ms  min {min(t):.4f}")
