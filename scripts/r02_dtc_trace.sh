#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in lowrank blast monarch; do for n in 1 16; do echo "== $m n=$n"; timeout 120 python scripts/dtc_trace.py $m $n; done; done > gpurun_out/dtc_trace.txt 2>&1
