#!/bin/bash
# full GPU suite + smoke + default bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/full_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/full_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/full_smoke.txt
timeout 900 python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; echo "bench rc=$?" >> gpurun_out/full_bench.err
