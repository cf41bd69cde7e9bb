#!/bin/bash
# plan knobs A/B on one config: each line "env -> per-launch ms"
cd $GRAFT_REPO_ROOT
CFG=${1:-C4}
BLR_PLAN=1 timeout 300 python bench.py --config $CFG --steps 3 --warmup 1 --no-cpu-baseline --no-variants --no-dense > /dev/null 2> gpurun_out/var_plan.txt
for v in "" "BLR_BUFS=1" "BLR_KBOX=1" "BLR_BUFS=1 BLR_KBOX=1" "BLR_S3_PAIR=0" "BLR_LONGK_PAIR=0" "BLR_NO_PDL=1"; do
  env $v timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-variants --no-dense > gpurun_out/var_tmp.json 2>/dev/null
  python -c "
import json,sys
d=json.loads(open('gpurun_out/var_tmp.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],3), [{k:round(x,3) for k,x in l['launch_ms'].items()} for l in d['per_layer']])
" >> gpurun_out/var_results.txt
done
