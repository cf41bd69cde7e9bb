#!/bin/bash
# C2 diagnostics: launch plans, per-launch times across n, and intra-kernel traces.
cd /root/repo
for m in lowrank monarch blast; do
  for l in c_fc c_proj; do
    BLR_PLAN=1 SCAN_N=${SCAN_N:-2048,8192,32768} python scripts/scan.py $m GPT2-S $l 2>&1 | sort -u
  done
done > gpurun_out/diag_scan.txt
python scripts/trace.py lowrank GPT2-S c_fc 8192 > gpurun_out/diag_trace.txt 2>&1
python scripts/trace.py lowrank GPT2-S c_proj 8192 >> gpurun_out/diag_trace.txt 2>&1
