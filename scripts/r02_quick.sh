#!/bin/bash
# quick GPU iteration: selected GPU tests + one workload's bench line
#   usage: r02_quick.sh "<pytest -k expr>" <config> [extra bench args]
cd $GRAFT_REPO_ROOT
K="$1"; CFG="$2"; shift 2
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/q_pytest.txt 2>&1
  echo "pytest rc=$?" >> gpurun_out/q_pytest.txt
fi
if [ -n "$CFG" ]; then
  timeout 900 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-variants "$@" > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
  echo "bench rc=$?" >> gpurun_out/q_bench.err
fi
