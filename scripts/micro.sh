#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_ingress benchmarks/micro/tma_ingress.cu && timeout 120 /tmp/tma_ingress | tee gpurun_out/micro_tma_ingress.txt
