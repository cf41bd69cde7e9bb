#!/bin/bash
# One gpurun session: build, smoke, GPU parity tests, bench (N=1), ncu launch list + full capture.
# Usage (from the repo root on the GPU box):  bash scripts/gpu_check.sh [tests|bench|ncu|all] [config]
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
WHAT=${1:-all}
CFG=${2:-C2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
if [[ $WHAT == all || $WHAT == tests ]]; then
  timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/smoke.log
  timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 600 python bench.py --config $CFG > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_$CFG.json; tail -5 gpurun_out/bench_$CFG.err
  timeout 300 python bench.py --config $CFG --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$CFG.json 2>&1; echo "ref rc=$?"; cat gpurun_out/bench_ref_$CFG.json | tail -c 600
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:blr_gemm_kernel -c 60 --csv \
     --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 3 --warmup 1 --no-dense --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:blr_gemm_kernel -s 12 -c 12 \
     -o gpurun_out/prof_$CFG -f python bench.py --config $CFG --steps 1 --warmup 1 --no-dense --no-cpu-baseline > gpurun_out/ncu_full_$CFG.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full_$CFG.log
fi
