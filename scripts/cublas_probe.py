"""One torch.bmm of a C4 grouped shape (for an ncu capture of the cuBLAS kernel cuBLAS picks):
python scripts/cublas_probe.py gateS3|downS1|downS3|dense"""
import sys
import torch
shapes = {"gateS3": (16, 65536, 1488, 688), "downS1": (16, 65536, 688, 1488),
          "downS3": (16, 65536, 1488, 256), "dense": (1, 65536, 4096, 11008)}
g, M, K, N = shapes[sys.argv[1]]
dev = torch.device("cuda")
A = torch.randn(g, M, K, device=dev, dtype=torch.bfloat16)
B = torch.randn(g, K, N, device=dev, dtype=torch.bfloat16)
C = torch.empty(g, M, N, device=dev, dtype=torch.bfloat16)
torch.bmm(A, B, out=C)
torch.cuda.synchronize()
