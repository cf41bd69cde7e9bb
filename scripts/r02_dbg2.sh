#!/bin/bash
# Debug-knob timing of a small (GPT2-S, n = 8192) layer's launches: usage r02_dbg2.sh method layer "L:dbg ..."
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BLR_NVCC_EXTRA=-DBLR_DEBUG_KNOBS python -c "import paper_2512_20861_b200 as b; b.build(force=True)" || exit 1
out=gpurun_out/dbg2_$1_$2.txt; : > $out
echo "== baseline" >> $out; SCAN_N=8192 timeout 300 python scripts/scan.py $1 GPT2-S $2 2>&1 | tail -1 >> $out
for v in $3; do L=${v%%:*}; D=${v##*:}
  echo "== launch $L dbg $D" >> $out; BLR_DBG=$D BLR_DBG_LAUNCH=$L SCAN_N=8192 timeout 300 python scripts/scan.py $1 GPT2-S $2 2>&1 | tail -1 >> $out
done
