"""Our GEMM kernel on plain dense shapes against cuBLAS (is the main loop itself at cuBLAS's rate?):
low rank Y = (X V) U with r = 2048 at 65,536 tokens is two long-K dense GEMMs
(65536x4096x2048 and 65536x2048x11008).  Graph replay, L2 flushed before each replay."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402

dev = torch.device("cuda")
n, i, o, r = 65536, 4096, 11008, int(os.environ.get("PROBE_R", "2048"))
X = torch.randn(n, i, device=dev, dtype=torch.bfloat16)
V = (torch.randn(i, r, device=dev) / i ** 0.5).to(torch.bfloat16)
U = (torch.randn(r, o, device=dev) / r ** 0.5).to(torch.bfloat16)
Z = torch.empty(n, r, device=dev, dtype=torch.bfloat16)
Yc = torch.empty(n, o, device=dev, dtype=torch.bfloat16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)



def ours():
    return blr.lowrank_matmul(X, V, U)


def cub():
    torch.mm(X, V, out=Z)
    torch.mm(Z, U, out=Yc)


def graph(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


if os.environ.get("PROBE_ONCE") == "1":  # one eager call per setting + one cuBLAS pair (for ncu)
    base_env = dict(os.environ)
    for st in sys.argv[1:] or [""]:
        for kv in st.split():
            k, v = kv.split("=", 1)
            os.environ[k] = v
        ours()
        os.environ.clear()
        os.environ.update(base_env)
    cub()
    torch.cuda.synchronize()
    sys.exit(0)
# settings: env knob strings, each captured as its own graph (the library reads knobs per call)
settings = sys.argv[1:] or [""]
gs = {}
base_env = dict(os.environ)
for st in settings:
    os.environ.clear()
    os.environ.update(base_env)
    for kv in st.split():
        k, v = kv.split("=", 1)
        os.environ[k] = v
    gs["ours[" + (st or "default") + "]"] = graph(ours)
os.environ.clear()
os.environ.update(base_env)
gs["cublas"] = graph(cub)
ts = {k: [] for k in gs}
for _ in range(12):
    for k, g in gs.items():
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts[k].append(a.elapsed_time(b))
fl = 2 * n * r * (i + o)
for k, t in ts.items():
    ms = statistics.median(t)
    print(f"dense r={r} {k:30s} {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s")
