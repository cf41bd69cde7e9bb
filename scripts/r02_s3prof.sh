#!/bin/bash
# plans of the C4 step + full ncu capture (source-level) of gate S3 and down S1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BLR_PLAN=1 timeout 300 python bench.py --config C4 --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-variants --eager > gpurun_out/plan_C4.json 2> gpurun_out/plan_C4.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"blr_gemm" -s 1 -c 2 \
   -o gpurun_out/prof_s3 -f python bench.py --config C4 --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-variants --eager > gpurun_out/ncu_s3.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_s3.log
