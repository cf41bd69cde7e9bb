#!/bin/bash
# (produced profiles/r02_wide_splitrel_ab.txt: in-process A/B of the wide tiles with the per-half release)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in C4 C4X C4F8; do
  BLR_PLAN=1 timeout 120 python scripts/ab.py $c "" --reps 1 2>&1 | grep "split=1" | sort | uniq > gpurun_out/wide3_plan_$c.txt
done
timeout 300 python scripts/ab.py C4 "" "BLR_WIDE=0" --reps 16 --layer 1 > gpurun_out/wide3_ab.txt 2>&1
timeout 300 python scripts/ab.py C4 "" "BLR_WIDE=0" --reps 16 >> gpurun_out/wide3_ab.txt 2>&1
timeout 300 python scripts/ab.py C4X "" "BLR_WIDE=0" --reps 10 >> gpurun_out/wide3_ab.txt 2>&1
timeout 300 python scripts/ab.py C4F8 "" "BLR_WIDE=0" --reps 10 >> gpurun_out/wide3_ab.txt 2>&1
timeout 300 python scripts/ab.py C4 "" "BLR_WIDE=0" --reps 16 >> gpurun_out/wide3_ab.txt 2>&1
