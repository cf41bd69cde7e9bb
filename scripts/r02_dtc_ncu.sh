#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in lowrank blast; do
  timeout 600 ncu --set full --clock-control none -k regex:decode_tc -s 2 -c 2 -o gpurun_out/dtc_$m -f python scripts/dtc_one.py $m 1 2 > gpurun_out/dtc_ncu_$m.log 2>&1
done
for m in lowrank blast; do bash scripts/ncu_brief.sh gpurun_out/dtc_$m.ncu-rep > gpurun_out/dtc_ncu_$m.txt 2>&1; done
