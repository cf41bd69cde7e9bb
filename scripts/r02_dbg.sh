#!/bin/bash
# Debug-knob timing of the C4 gate/down GEMM phases: which part bounds them
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BLR_NVCC_EXTRA=-DBLR_DEBUG_KNOBS python -c "import paper_2512_20861_b200 as b; b.build(force=True)" || exit 1
out=gpurun_out/dbg_sweep.txt; : > $out
for layer in gate_up_proj down_proj; do
  echo "== $layer baseline" >> $out; SCAN_N=65536 timeout 300 python scripts/scan.py blast Llama-7B $layer 2>&1 | tail -1 >> $out
  for d in 1 4 8 12 2; do
    for L in 0 2; do
      echo "== $layer launch $L dbg $d" >> $out
      BLR_DBG=$d BLR_DBG_LAUNCH=$L SCAN_N=65536 timeout 300 python scripts/scan.py blast Llama-7B $layer 2>&1 | tail -1 >> $out
    done
  done
done
