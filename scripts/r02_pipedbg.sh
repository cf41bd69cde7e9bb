#!/bin/bash
# where the pipelined layer's time goes: debug-knob build, gate layer, fixed role split
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BLR_NVCC_EXTRA=-DBLR_DEBUG_KNOBS python -c "import paper_2512_20861_b200 as b; b.build(force=True)" || exit 1
S="BLR_PIPE=1 BLR_PIPE_SPLIT=${1:-14,16}"
timeout 900 python scripts/ab.py C4 "BLR_PIPE=0" "$S" "$S BLR_PIPE_DBG=1" "$S BLR_PIPE_DBG=2" "$S BLR_PIPE_DBG=4" "$S BLR_PIPE_DBG=7" --reps 3 --layer 0 > gpurun_out/pipe_dbg.txt 2>&1
