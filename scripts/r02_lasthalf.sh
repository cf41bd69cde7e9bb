#!/bin/bash
# wide 512-column tiles with a single-half last tile (KParams::last_half: C4 gate S3 = 512 + 176):
# tests + in-process A/B against the 256-column tiles
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/lh_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/lh_tests.txt
tail -3 gpurun_out/lh_tests.txt | grep -q " passed" || exit 1
BLR_PLAN=1 timeout 120 python scripts/ab.py C4 "" --reps 1 2>&1 | grep "split=1" | sort | uniq > gpurun_out/lh_plan.txt
timeout 300 python scripts/ab.py C4 "" "BLR_WIDE=0" --reps 12 --layer 0 > gpurun_out/lh_ab.txt 2>&1
timeout 300 python scripts/ab.py C4 "" "BLR_WIDE=0" --reps 12 >> gpurun_out/lh_ab.txt 2>&1
for c in C4X C4F8 C4M; do timeout 300 python scripts/ab.py $c "" "BLR_WIDE=0" --reps 10 >> gpurun_out/lh_ab.txt 2>&1; done
