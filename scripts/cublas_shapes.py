"""cuBLAS (torch.matmul, bf16) times for the C2 GEMM shapes, graph-replayed with an L2 flush, for
comparison with the library's per-launch times."""
import torch
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
R = 10
def gtime(fn):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best * 1e3
def fl():
    for _ in range(R): flush.zero_()
t_fl = gtime(fl)
for (m, k, n, what) in [(8192, 192, 3072, "LR c_fc expand"), (8192, 768, 192, "LR c_fc proj"),
                        (8192, 3072, 192, "LR c_proj proj"), (8192, 192, 768, "LR c_proj expand"),
                        (8192, 768, 3072, "dense c_fc"), (8192, 3072, 768, "dense c_proj")]:
    A = torch.randn(m, k, device=dev, dtype=torch.bfloat16); B = torch.randn(k, n, device=dev, dtype=torch.bfloat16)
    C = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    def body():
        for _ in range(R):
            flush.zero_(); torch.matmul(A, B, out=C)
    t = (gtime(body) - t_fl) / R
    print(f"{what:18s} {m}x{k}x{n}: {t:6.1f} us  ({2*m*k*n/t/1e6:6.0f} TFLOP/s, {(m*k+k*n+m*n)*2/t/1e3:6.0f} GB/s)")
