#!/bin/bash
# alternate two builds of the library on the same box: "old" = libblr_old.so, "new" = libblr.so
cd $GRAFT_REPO_ROOT
OLDENV=${OLDENV:-}
for rep in 1 2 3; do
  for c in ${CFGS:-C4 C4M}; do
    env BLR_LIB=$PWD/paper_2512_20861_b200/libblr_old.so $OLDENV timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-variants --no-dense > gpurun_out/abb_tmp.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/abb_tmp.json').read().strip().splitlines()[-1])
print('old', '$c', round(d['ms_per_step'],3), [{k:round(x,3) for k,x in l['launch_ms'].items()} for l in d['per_layer']])" >> gpurun_out/abb.txt
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-variants --no-dense > gpurun_out/abb_tmp.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/abb_tmp.json').read().strip().splitlines()[-1])
print('new', '$c', round(d['ms_per_step'],3), [{k:round(x,3) for k,x in l['launch_ms'].items()} for l in d['per_layer']])" >> gpurun_out/abb.txt
  done
done
