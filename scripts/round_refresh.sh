#!/bin/bash
# Round-end refresh: smoke, default bench line (+ reference arm), per-config bench lines, ncu.
# usage: bash scripts/round_refresh.sh TAG "BENCH_CFGS" "PROFILE_CFGS"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
TAG=${1:-r01}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default bench rc=$?"; python scripts/summarize.py gpurun_out/bench_default.json | head -3
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2>&1; echo "reference rc=$?"; tail -c 400 gpurun_out/bench_reference.json
for CFG in $2; do
  timeout 900 python bench.py --config $CFG > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err; echo "bench $CFG rc=$?"; python scripts/summarize.py gpurun_out/bench_$CFG.json | head -2
done
for CFG in $3; do
  timeout 1500 bash scripts/profile_round.sh $CFG $TAG > gpurun_out/profile_$CFG.log 2>&1; echo "profile $CFG rc=$?"; head -22 gpurun_out/profile_$CFG.log | tail -18
done
