"""cuBLAS reference points for the grouped GEMMs of the C4 BLAST / Monarch layers (torch.bmm,
bf16, L2 flushed between reps): what a vendor GEMM achieves on exactly these shapes."""
import torch
dev = torch.device("cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
n = 65536
shapes = {  # name: (groups, M, K, N)
    "gate S3 (Z''_k U_k)": (16, n, 1488, 688),
    "down S1 (X_l V_l)": (16, n, 688, 1488),
    "gate S1 (X_l V_l)": (16, n, 256, 1488),
    "down S3 (Z''_k U_k)": (16, n, 1488, 256),
    "Monarch gate S3": (16, n, 1536, 688),
    "dense gate": (1, n, 4096, 11008),
}
for name, (g, M, K, N) in shapes.items():
    A = torch.randn(g, M, K, device=dev, dtype=torch.bfloat16)
    B = torch.randn(g, K, N, device=dev, dtype=torch.bfloat16)
    C = torch.empty(g, M, N, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        torch.bmm(A, B, out=C)
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); torch.bmm(A, B, out=C); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    fl = 2 * g * M * K * N
    print(f"{name:24s} {ms:7.3f} ms  {fl / ms / 1e9:7.1f} TFLOP/s")
    del A, B, C
