#!/bin/bash
# wide (two-MMA, single-accumulator) pair tiles with / without the per-half accumulator release vs
# the default 256-column tiles: parity, dense shapes, C4 layers
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/wide_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/wide_tests.txt
tail -3 gpurun_out/wide_tests.txt | grep -q "passed" || exit 1
timeout 300 python scripts/dense_probe.py "" "BLR_WIDE=1" "BLR_WIDE=1 BLR_SPLITREL=0" > gpurun_out/wide_dense.txt 2>&1
BLR_PLAN=1 BLR_WIDE=1 timeout 120 python scripts/ab.py C4 "" --reps 1 --layer 1 2>&1 | grep plan | sort | uniq > gpurun_out/wide_plan.txt
timeout 300 python scripts/ab.py C4 "" "BLR_WIDE=1" "BLR_WIDE=1 BLR_SPLITREL=0" --reps 8 --layer 1 > gpurun_out/wide_c4.txt 2>&1
timeout 300 python scripts/ab.py C3 "" "BLR_WIDE=1" --reps 15 >> gpurun_out/wide_c4.txt 2>&1
timeout 300 python scripts/ab.py C2 "" "BLR_WIDE=1" --reps 15 >> gpurun_out/wide_c4.txt 2>&1
