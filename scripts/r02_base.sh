#!/bin/bash
# session baseline: full GPU suite, smoke, default bench line (C4 + variants)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/base_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/base_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/base_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/base_smoke.txt
timeout 900 python bench.py > gpurun_out/base_bench.json 2> gpurun_out/base_bench.err; echo "bench rc=$?" >> gpurun_out/base_bench.err
