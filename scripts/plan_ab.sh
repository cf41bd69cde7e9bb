#!/bin/bash
# A/B a planner switch on whole-config benches: bash scripts/plan_ab.sh "ENV=..." "CFG..."
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
ENVS=${1:-"X=1"}; CFGS=${2:-C4}
for CFG in $CFGS; do
  for E in $ENVS; do
    env ${E//,/ } BLR_PLAN=1 timeout 900 python bench.py --config $CFG --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_${CFG}_${E}.json 2> gpurun_out/ab_${CFG}_${E}.err
    echo "== $CFG $E rc=$?"; grep "blr plan" gpurun_out/ab_${CFG}_${E}.err | sort | uniq | head -12
    python scripts/summarize.py gpurun_out/ab_${CFG}_${E}.json
  done
done
