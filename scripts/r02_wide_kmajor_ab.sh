#!/bin/bash
# wide tiles over tile-blocked A (K-major factor storage): tests + A/B
# (produced profiles/r02_wide_kmajor_ab.txt)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_wide.py tests/test_gpu_pipe.py tests/test_gpu_fuzz.py -x -q > gpurun_out/wide4_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/wide4_tests.txt
tail -3 gpurun_out/wide4_tests.txt | grep -q " passed" || exit 1
BLR_PLAN=1 timeout 120 python scripts/ab.py C4K "" --reps 1 2>&1 | grep "plan" | sort | uniq > gpurun_out/wide4_plan.txt
timeout 300 python scripts/ab.py C4K "" "BLR_WIDE=0" --reps 12 --layer 0 > gpurun_out/wide4_ab.txt 2>&1
timeout 300 python scripts/ab.py C4K "" "BLR_WIDE=0" --reps 12 >> gpurun_out/wide4_ab.txt 2>&1
timeout 300 python scripts/ab.py C4 "" "BLR_WIDE=0" --reps 12 >> gpurun_out/wide4_ab.txt 2>&1
