#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "pair or split or fp8 or sampled or transposed" > gpurun_out/q_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/q_pytest.txt
BLR_PLAN=1 timeout 300 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-variants --no-dense > /dev/null 2> gpurun_out/wide_plan.txt
for w in 0 1; do
  for c in C4 C4M C4F8; do
    BLR_WIDE=$w timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/wide${w}_$c.json 2>gpurun_out/wide${w}_$c.err
  done
done
