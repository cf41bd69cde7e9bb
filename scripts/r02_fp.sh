#!/bin/bash
# lean producer: GPU parity subset + in-process A/B against the generic producer
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_monarch_transposed.py -m gpu -q -x > gpurun_out/fp_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/fp_pytest.txt
timeout 600 python scripts/ab.py C4 "" "BLR_FASTPROD=0" --reps 9 > gpurun_out/fp_ab.txt 2>&1
timeout 600 python scripts/ab.py C4M "" "BLR_FASTPROD=0" --reps 9 >> gpurun_out/fp_ab.txt 2>&1
timeout 600 python scripts/ab.py C2 "" "BLR_FASTPROD=0" --reps 15 >> gpurun_out/fp_ab.txt 2>&1
