#!/bin/bash
# Refresh the round's profiles: ncu launch list + full capture per config, plus extra bench lines.
# usage: bash scripts/gpu_profiles.sh TAG "CFG..." "BENCHCFG..."
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r01}; PROF=${2:-C2}; BENCH=${3:-}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
for CFG in $BENCH; do
  timeout 900 python bench.py --config $CFG > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err; echo "bench $CFG rc=$?"; tail -3 gpurun_out/bench_$CFG.err
  python scripts/summarize.py gpurun_out/bench_$CFG.json
done
for CFG in $PROF; do
  timeout 1500 bash scripts/profile_round.sh $CFG $TAG > gpurun_out/profile_$CFG.log 2>&1; echo "profile $CFG rc=$?"; head -24 gpurun_out/profile_$CFG.log
done
