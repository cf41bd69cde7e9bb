#!/bin/bash
# decode_mn TMA-slice A/B: parity for the small-token paths, then decode_bench old vs new build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "decode or transposed or robust" > gpurun_out/dec_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/dec_pytest.txt
for rep in 1 2; do
  BLR_LIB=$PWD/paper_2512_20861_b200/libblr_old.so timeout 300 python scripts/decode_bench.py > gpurun_out/dec_old_$rep.txt 2>&1
  timeout 300 python scripts/decode_bench.py > gpurun_out/dec_new_$rep.txt 2>&1
done
