#!/bin/bash
cd $GRAFT_REPO_ROOT
BLR_NCL=1 timeout 600 python -m pytest tests -m gpu -x -q -k "split_s2 or sampled or pair or robustness or transposed" > gpurun_out/q_pytest.txt 2>&1
echo "pytest ncl rc=$?" >> gpurun_out/q_pytest.txt
BLR_NCL=1 BLR_PLAN=1 timeout 300 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-variants --no-dense > /dev/null 2> gpurun_out/ncl_plan.txt
timeout 900 python scripts/ab.py C4 "" "BLR_NCL=1" --reps 11 > gpurun_out/ab_ncl.txt 2>&1
timeout 900 python scripts/ab.py C4M "" "BLR_NCL=1" --reps 11 >> gpurun_out/ab_ncl.txt 2>&1
timeout 900 python scripts/ab.py C4 "" "BLR_NCL=1" --reps 11 >> gpurun_out/ab_ncl.txt 2>&1
