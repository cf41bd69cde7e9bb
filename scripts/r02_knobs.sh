#!/bin/bash
# usage: r02_knobs.sh CONFIG "KNOB=.." "KNOB=.." ...   (each knob A/B'd against the default, in-process)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CFG=$1; shift
for k in "$@"; do
  timeout 600 python scripts/ab.py $CFG "" "$k" --reps 7 >> gpurun_out/knob_ab.txt 2>&1 || echo "$CFG [$k] failed" >> gpurun_out/knob_ab.txt
done
