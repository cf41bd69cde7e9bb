#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pipe.py -m gpu -q -x > gpurun_out/pipe_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pipe_pytest.txt
grep -q "rc=0" gpurun_out/pipe_pytest.txt || exit 0
: > gpurun_out/pipe_ab.txt
timeout 900 python scripts/ab.py C4 "BLR_PIPE=0" "BLR_PIPE=1 BLR_PIPE_SPLIT=18,8" "BLR_PIPE=1 BLR_PIPE_SPLIT=16,12" "BLR_PIPE=1 BLR_PIPE_SPLIT=14,16" --reps 5 --layer 0 >> gpurun_out/pipe_ab.txt 2>&1
timeout 900 python scripts/ab.py C4 "BLR_PIPE=0" "BLR_PIPE=1 BLR_PIPE_SPLIT=48,8" "BLR_PIPE=1 BLR_PIPE_SPLIT=44,12" "BLR_PIPE=1 BLR_PIPE_SPLIT=40,16" --reps 5 --layer 1 >> gpurun_out/pipe_ab.txt 2>&1
