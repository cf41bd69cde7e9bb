#!/bin/bash
# cuBLAS kernels on the C4 grouped shapes (ncu full) + our GEMM on plain dense shapes vs cuBLAS
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python scripts/dense_probe.py > gpurun_out/dense_probe.txt 2>&1
PROBE_R=1024 python scripts/dense_probe.py >> gpurun_out/dense_probe.txt 2>&1
BLR_PLAN=1 python scripts/dense_probe.py > gpurun_out/dense_probe_plan.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/dense_probe_launches.csv \
   python scripts/dense_probe.py > /dev/null 2>&1
bash scripts/r02_cublas_ncu.sh
