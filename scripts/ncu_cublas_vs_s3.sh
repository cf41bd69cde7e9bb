#!/bin/bash
# ncu --set full of cuBLAS bmm on the C4 gate S3 shape next to our S3 kernel (same box)
cd $GRAFT_REPO_ROOT
cat > /tmp/bmm_one.py <<'PY'
import torch
A = torch.randn(16, 65536, 1488, device="cuda", dtype=torch.bfloat16)
B = torch.randn(16, 1488, 688, device="cuda", dtype=torch.bfloat16)
C = torch.empty(16, 65536, 688, device="cuda", dtype=torch.bfloat16)
for _ in range(2): torch.bmm(A, B, out=C)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:nvjet -s 1 -c 1 -o gpurun_out/prof_cublas_s3 -f python /tmp/bmm_one.py > gpurun_out/ncu_cublas.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:blr_gemm -s 1 -c 1 -o gpurun_out/prof_ours_s3 -f python scripts/one_call.py blast Llama-7B gate_up_proj 65536 1 > gpurun_out/ncu_ours.log 2>&1
