#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BLR_NVCC_EXTRA=-DBLR_DEBUG_KNOBS python -c "import paper_2512_20861_b200 as b; b.build(force=True)" || exit 1
out=gpurun_out/widedbg.txt; : > $out
for e in "X=0" "BLR_WIDE=1"; do for d in 0 4 12; do
  echo "== $e dbg $d" >> $out
  env $e BLR_PLAN=1 BLR_DBG=$d BLR_DBG_LAUNCH=2 SCAN_N=65536 timeout 300 python scripts/scan.py blast Llama-7B gate_up_proj 2>&1 | grep -E "n= |kind=0 pair=2 .*tiles=256x16x" | tail -2 >> $out
done; done
