#!/bin/bash
# Profile one config: ncu launch list + ncu --set full of one step's launches; summaries -> profiles/
# usage: bash scripts/profile_round.sh CFG TAG   (e.g. C2 r01)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
CFG=${1:-C2}; TAG=${2:-r01}
mkdir -p gpurun_out profiles
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
BLR_DUMP_PHASES=gpurun_out/phases_$CFG.json python bench.py --config $CFG --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-variants --eager > /dev/null 2>&1
N=$(python -c "import json;print(len(json.load(open('gpurun_out/phases_$CFG.json'))))")
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"blr_gemm|blast_s2|blr_fused" -c $((3*N)) --csv \
  --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 2 --warmup 0 --no-dense --no-cpu-baseline --no-variants --eager > /dev/null 2>&1
echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"blr_gemm|blast_s2|blr_fused" -c $N \
  -o gpurun_out/prof_$CFG -f python bench.py --config $CFG --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-variants --eager > gpurun_out/ncu_full_$CFG.log 2>&1
echo "full rc=$?"
# summaries go to gpurun_out/ (only that directory comes back from the box); copy them into
# profiles/ locally:  python scripts/profile_summary.py list|full ... profiles/...
python scripts/profile_summary.py list gpurun_out/launches_$CFG.csv gpurun_out/${TAG}_${CFG}_launches.txt
python scripts/profile_summary.py full gpurun_out/prof_$CFG.ncu-rep gpurun_out/${TAG}_${CFG}_ncu_full.txt gpurun_out/phases_$CFG.json gpurun_out/ncu_traffic_$CFG.json
head -30 gpurun_out/${TAG}_${CFG}_ncu_full.txt
# keep gpurun_out/ small (only <= 64 MiB comes back): the report stays only when KEEP_REP=1
[ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/prof_$CFG.ncu-rep
