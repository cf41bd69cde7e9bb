#!/bin/bash
# bench lines of every configured workload at HEAD (one box): profiles/r02_bench_<CFG>.json
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/bench_all
for c in C1 C2 C3 C4M C4X C4F8 C4K C5V-1 C5V-8 C5V-64 C5V-256 C5D-1 C5D-8 C5D-64 C5D-256; do
  timeout 600 python bench.py --config $c --no-variants --no-cpu-baseline > gpurun_out/bench_all/$c.json 2> gpurun_out/bench_all/$c.err
  echo "$c rc=$?" >> gpurun_out/bench_all/rc.txt
done
