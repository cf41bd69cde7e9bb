#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "split_s2 or sampled" > gpurun_out/q_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/q_pytest.txt
BLR_PF=12 timeout 600 python -m pytest tests -m gpu -x -q -k "split_s2 or sampled or pair" >> gpurun_out/q_pytest.txt 2>&1
echo "pytest pf rc=$?" >> gpurun_out/q_pytest.txt
timeout 600 python scripts/ab.py C4 "BLR_PF=0" "BLR_PF=8" "BLR_PF=12" "BLR_PF=20" "BLR_PF=12 BLR_WIDE=1" --reps 9 > gpurun_out/ab_pf.txt 2>&1
timeout 600 python scripts/ab.py C4M "BLR_PF=0" "BLR_PF=12" "BLR_PF=20" --reps 9 >> gpurun_out/ab_pf.txt 2>&1
