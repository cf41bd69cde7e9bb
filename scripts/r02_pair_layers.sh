#!/bin/bash
# per-layer in-process A/B of single-CTA tiles (BLR_PAIR=1) against the CTA-pair default
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rm -f gpurun_out/pair_layers.txt
for c in C2:6 C3:12 C5V-256:6 C5D-256:2; do
  cfg=${c%%:*}; nl=${c##*:}
  for ((j=0; j<nl; j++)); do
    timeout 300 python scripts/ab.py $cfg "" "BLR_PAIR=1" --reps 7 --layer $j >> gpurun_out/pair_layers.txt 2>&1
  done
done
