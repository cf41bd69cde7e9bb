#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/chunk_layers.txt
for c in C5V-1 C5D-1 C1 C5V-8; do
  for mx in 0 4096; do
    if [ $mx = 0 ]; then E=""; else E="BLR_DECODE_MAXN=$mx"; fi
    env $E timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-variants --no-cpu-baseline --no-dense > gpurun_out/chunk_tmp.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/chunk_tmp.json').read().strip().splitlines()[-1])
print('$c maxn=$mx total', round(d['ms_per_step']*1e3,1))
for l in d['per_layer']: print('   ', l['layer'], round(l['ms']*1e3,1), {k:round(v*1e3,1) for k,v in l['launch_ms'].items()})" >> gpurun_out/chunk_layers.txt 2>&1
  done
done
