#!/bin/bash
# tests + C2 bench + optional extra configs (args), summarised
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; grep -E "^E +AssertionError" gpurun_out/pytest_gpu.log | head
for CFG in C2 "$@"; do
  timeout 900 python bench.py --config $CFG $EXTRA > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err; echo "bench $CFG rc=$?"; tail -3 gpurun_out/bench_$CFG.err
  python scripts/summarize.py gpurun_out/bench_$CFG.json
done
