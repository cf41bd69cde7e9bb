#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "pair or split or sampled or robustness" > gpurun_out/q_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/q_pytest.txt
BLR_PLAN=1 timeout 300 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-variants --no-dense > /dev/null 2> gpurun_out/mc_plan.txt
timeout 600 python scripts/ab.py C4 "BLR_MC=1" "BLR_MC=2" "BLR_MC=4" --reps 9 > gpurun_out/ab_mc.txt 2>&1
timeout 600 python scripts/ab.py C4M "BLR_MC=1" "BLR_MC=2" "BLR_MC=4" --reps 9 >> gpurun_out/ab_mc.txt 2>&1
