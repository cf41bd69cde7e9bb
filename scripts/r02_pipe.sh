#!/bin/bash
# pipelined BLAST layer: parity + bitwise tests, then C4 A/B against the three-launch path
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BLR_PLAN=1 timeout 600 python -m pytest tests/test_gpu_pipe.py -m gpu -q -x > gpurun_out/pipe_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pipe_pytest.txt
grep -q "rc=0" gpurun_out/pipe_pytest.txt || exit 0
BLR_PLAN=1 BLR_PIPE=1 timeout 300 python bench.py --config C4 --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-variants --eager > /dev/null 2> gpurun_out/pipe_plan.txt
timeout 900 python scripts/ab.py C4 "BLR_PIPE=0" "BLR_PIPE=1" "BLR_PIPE=1 BLR_PIPE_SPLIT=14,12" "BLR_PIPE=1 BLR_PIPE_SPLIT=18,10" --reps 7 > gpurun_out/pipe_ab.txt 2>&1
