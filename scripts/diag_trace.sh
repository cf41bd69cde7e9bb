#!/bin/bash
# trace one layer under debug variants: bash scripts/diag_trace.sh lowrank c_fc "0 12 28 44 60"
cd /root/repo
for v in ${3:-0 12 28 44 60}; do
  echo "=== BLR_DBG=$v"
  TRACE_FLUSH=${FL:-zero} BLR_DBG=$v python scripts/trace.py $1 GPT2-S $2 8192 2>&1 | sed -n '/launch 1/,$p' | grep -E "launch|gdwait|lastmma|drained|MMA-commit|issue|full-ready"
done
