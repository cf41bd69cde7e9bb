#!/bin/bash
# Per-launch times of one layer under kernel debug switches (BLR_DBG bits, one launch at a time).
# usage: bash scripts/dbg_sweep.sh method model layer "launch:dbg ..."
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
M=$1; MODEL=$2; LAYER=$3
echo "== baseline"; SCAN_N=65536 python scripts/scan.py $M $MODEL $LAYER 2>&1 | tail -1
for v in $4; do
  L=${v%%:*}; D=${v##*:}
  echo "== launch $L dbg $D"; BLR_DBG=$D BLR_DBG_LAUNCH=$L SCAN_N=65536 python scripts/scan.py $M $MODEL $LAYER 2>&1 | tail -1
done
