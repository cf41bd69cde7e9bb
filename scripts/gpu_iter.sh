#!/bin/bash
# Iteration helper: build, a filtered GPU test subset, then benches with plans.
# usage: bash scripts/gpu_iter.sh "<pytest -k expr>" "CFG..."
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
if [[ -n "$1" ]]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 120 -p no:cacheprovider -k "$1" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
fi
for CFG in $2; do
  timeout 600 python bench.py --config $CFG --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/it_$CFG.json 2> gpurun_out/it_$CFG.err; echo "bench $CFG rc=$?"; python scripts/summarize.py gpurun_out/it_$CFG.json
done
