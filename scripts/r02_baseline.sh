#!/bin/bash
# round-2 baseline: current C4 / C4M bench lines on a fresh box
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02_smi.txt
for c in C4 C4M; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_base_$c.json 2> gpurun_out/r02_base_$c.err
done
