#!/bin/bash
cd /root/repo
for f in zero read none; do for v in 0 12; do
  echo "=== flush=$f BLR_DBG=$v"
  TRACE_FLUSH=$f BLR_DBG=$v python scripts/trace.py lowrank GPT2-S c_fc 8192 2>&1 | grep -E "launch|gdwait|lastmma|drained|MMA-commit|full-ready"
done; done
