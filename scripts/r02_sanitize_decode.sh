#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small shapes of the tensor-core decode kernels
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/sanitizer_decode.txt; : > $OUT
K="test_decode_lowrank and (1-64 or 3-768) or test_decode_monarch and (3-2-3 or 8-4-4) or test_decode_blast and (1-1-1 or 3-3-2 or 8-6-6 or 11-3 or 12-5) or test_decode_forced_plans and (64-3 or 128-6 or 256-7)"
for tool in memcheck racecheck synccheck; do
  echo "=== $tool" >> $OUT
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_decode.py -m gpu -q -x -k "$K" -p no:cacheprovider > gpurun_out/sand_$tool.log 2>&1
  echo "rc=$?" >> $OUT
  grep -E "ERROR SUMMARY|passed|failed|Error|error:" gpurun_out/sand_$tool.log | tail -8 >> $OUT
done
