#!/bin/bash
cd $GRAFT_REPO_ROOT
BLR_S12_CHUNK=384 timeout 600 python -m pytest tests -m gpu -x -q -k "split_s2 or sampled or robustness or fp8" > gpurun_out/q_pytest.txt 2>&1
echo "pytest s12 rc=$?" >> gpurun_out/q_pytest.txt
timeout 900 python scripts/ab.py C4 "" "BLR_S12_CHUNK=1024" "BLR_S12_CHUNK=1536" "BLR_S12_CHUNK=2048" "BLR_S12_CHUNK=4096" --reps 7 > gpurun_out/ab_s12.txt 2>&1
timeout 900 python scripts/ab.py C4F8 "" "BLR_S12_CHUNK=2048" "BLR_S12_CHUNK=4096" --reps 7 >> gpurun_out/ab_s12.txt 2>&1
