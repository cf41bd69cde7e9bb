#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pipe.py -m gpu -q -x > gpurun_out/pipe_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pipe_pytest.txt
grep -q "rc=0" gpurun_out/pipe_pytest.txt || exit 0
S="BLR_PIPE=1 BLR_PIPE_SPLIT=14,16"
timeout 900 python scripts/ab.py C4 "BLR_PIPE=0" "$S BLR_PIPE_HINTS=0" "$S" "$S BLR_PIPE_BP=8 BLR_PIPE_WIN=4" "BLR_PIPE=1 BLR_PIPE_SPLIT=16,12" "BLR_PIPE=1 BLR_PIPE_SPLIT=12,20" --reps 3 --layer 0 > gpurun_out/pipe_ab.txt 2>&1
bash scripts/r02_pipe_ncu.sh
