#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small shapes of every kernel family
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/sanitizer.txt; : > $OUT
K="test_lowrank_parity and (5-64 or 300-200) or test_monarch_parity and (130-2-2 or 257-3-4) or test_blast_parity and (129-2-3 or 200-16-16 or 100-5-2) or test_blast_split_s2_variants and 257-9-7 or test_lowrank_fused_parity or nonfinite and 136 or transposed_parity and (257 or 5-4) or fp8z_parity and 257"
for tool in memcheck racecheck synccheck; do
  echo "=== $tool" >> $OUT
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests -m gpu -q -x -k "$K" -p no:cacheprovider > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?" >> $OUT
  grep -E "ERROR SUMMARY|passed|failed|Error|error:" gpurun_out/san_$tool.log | tail -8 >> $OUT
done
