#!/bin/bash
# time one config under several library builds (BLR_LIB), same box: bisecting a regression
CFG=${CFG:-C5D-1}
rm -f gpurun_out/bisect.txt
for rep in 1 2; do
for lib in old e6cb207 02c07b6 364661e 354fdbf 5dfc904 3612bfa HEAD; do
  if [ $lib = HEAD ]; then L=$PWD/paper_2512_20861_b200/libblr.so; else L=$PWD/paper_2512_20861_b200/libblr_$lib.so; fi
  BLR_LIB=$L timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-variants --no-dense > gpurun_out/bis_tmp.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bis_tmp.json').read().strip().splitlines()[-1])
print('$lib', '$CFG', round(d['ms_per_step'],4), [{k:round(x,4) for k,x in l['launch_ms'].items()} for l in d['per_layer']])" >> gpurun_out/bisect.txt
done
done
