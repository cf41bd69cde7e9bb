#!/bin/bash
# ncu --set full of one bench step of a config (the first N launches of our kernels), then the
# robustness tests.   usage: r02_ncu.sh <config> <count> [pytest -k expr]
cd $GRAFT_REPO_ROOT
CFG=${1:-C4}; CNT=${2:-6}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"blr_|blast_" -c $CNT \
   -o gpurun_out/prof_$CFG -f python bench.py --config $CFG --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-variants --eager > gpurun_out/ncu_$CFG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$CFG.log
if [ -n "$3" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -k "$3" > gpurun_out/q_pytest.txt 2>&1
  echo "pytest rc=$?" >> gpurun_out/q_pytest.txt
fi
