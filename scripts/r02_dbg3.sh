#!/bin/bash
# gate S3 / down S1 of C4 under debug knobs: as is, without MMAs, without MMAs and epilogue
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BLR_NVCC_EXTRA=-DBLR_DEBUG_KNOBS python -c "import paper_2512_20861_b200 as b; b.build(force=True)" || exit 1
out=gpurun_out/dbg3.txt; : > $out
for L in gate_up_proj:2 down_proj:0; do lay=${L%%:*}; li=${L##*:}
for d in 0 4 8 12; do
  echo "== $lay launch $li dbg $d" >> $out
  BLR_DBG=$d BLR_DBG_LAUNCH=$li SCAN_N=65536 timeout 300 python scripts/scan.py blast Llama-7B $lay 2>&1 | tail -1 >> $out
done; done
