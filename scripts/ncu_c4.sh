#!/bin/bash
# full ncu capture of one step of a long config (each kernel once), e.g. C4M
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
CFG=${1:-C4M}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"blr_gemm|blast_s2" -s ${2:-0} -c ${3:-6} \
   -o gpurun_out/prof_$CFG -f python bench.py --config $CFG --steps 1 --warmup 0 --no-dense --no-cpu-baseline --eager > gpurun_out/ncu_$CFG.log 2>&1; echo "ncu rc=$?"
