#!/bin/bash
# tensor-core decode path: parity of the small-token paths, then plans, timeline, per-launch profile and decode_bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "decode or transposed" > gpurun_out/dtc_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/dtc_pytest.txt
for m in lowrank blast monarch; do BLR_DTC_VERBOSE=1 python scripts/dtc_one.py $m 1 1; done > gpurun_out/dtc_plans.txt 2>&1
bash scripts/r02_dtc_trace.sh
timeout 300 python scripts/decode_prof.py > gpurun_out/dtc_prof_new.txt 2>&1
timeout 300 python scripts/decode_bench.py > gpurun_out/dtc_bench_new.txt 2>&1
