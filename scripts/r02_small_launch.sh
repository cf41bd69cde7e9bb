#!/bin/bash
# Launch lists (every kernel, ours and cuBLAS's) of the small-batch configs: where the per-layer time goes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in C1 C5V-1 C5V-8 C5D-1; do
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -c 300 --csv \
    --log-file gpurun_out/small_$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-variants --eager > gpurun_out/small_$c.log 2>&1
  echo "$c rc=$?"
done
for c in C1 C5V-1 C5V-8 C5D-1; do
  BLR_PLAN=1 BLR_DTC_VERBOSE=1 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/small_plan_$c.log 2>&1
done
