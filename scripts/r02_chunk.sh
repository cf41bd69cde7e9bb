#!/bin/bash
cd $GRAFT_REPO_ROOT
BLR_S23_CHUNK=256 timeout 600 python -m pytest tests -m gpu -x -q -k "split_s2 or sampled or robustness or fp8" > gpurun_out/q_pytest.txt 2>&1
echo "pytest chunk rc=$?" >> gpurun_out/q_pytest.txt
timeout 900 python scripts/ab.py C4 "" "BLR_S23_CHUNK=512" "BLR_S23_CHUNK=1024" "BLR_S23_CHUNK=1536" "BLR_S23_CHUNK=2048" --reps 7 > gpurun_out/ab_chunk.txt 2>&1
