#!/bin/bash
# wide tiles with the per-half release as a default (auto rule) vs BLR_WIDE=0: full GPU suite + A/B
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/wide2_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/wide2_tests.txt
for c in C4 C4X C4K C4F8 C3 C2 C5D-256 C5V-256; do
  BLR_PLAN=1 timeout 120 python scripts/ab.py $c "" --reps 1 2>&1 | grep "split=1" | sort | uniq > gpurun_out/wide2_plan_$c.txt
  timeout 300 python scripts/ab.py $c "" "BLR_WIDE=0" --reps 10 >> gpurun_out/wide2_ab.txt 2>&1
done
