#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "split or sampled or robustness or fp8" > gpurun_out/q_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/q_pytest.txt
BLR_PLAN=1 timeout 300 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-variants --no-dense > /dev/null 2> gpurun_out/blk_plan.txt
timeout 900 python scripts/ab.py C4 "" "BLR_BLK_CW_OLD=1" "BLR_BLK_CW_OLD=1 BLR_BN_FILL=0" --reps 11 --layer 0 > gpurun_out/ab_blk.txt 2>&1
timeout 900 python scripts/ab.py C4 "" "BLR_BLK_CW_OLD=1" --reps 11 >> gpurun_out/ab_blk.txt 2>&1
