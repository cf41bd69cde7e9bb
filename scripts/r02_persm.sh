#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in 1 2; do echo "== MINPERSM=$m"; for meth in lowrank blast monarch; do BLR_DTC_MINPERSM=$m BLR_DTC_VERBOSE=1 python scripts/dtc_one.py $meth 1 1 2>&1 | grep dtc; done; BLR_DTC_MINPERSM=$m timeout 300 python scripts/decode_bench.py 2>&1 | grep Llama; done > gpurun_out/persm.txt 2>&1
