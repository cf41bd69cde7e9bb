#!/bin/bash
# quick perf check: abi harness (LR c_fc, eager events + trace) and graph layer times for C2
cd $GRAFT_REPO_ROOT/benchmarks/micro && nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/at abi_trace.cu \
  -L../../paper_2512_20861_b200 -lblr -Xlinker -rpath=$GRAFT_REPO_ROOT/paper_2512_20861_b200 || exit 1
cd $GRAFT_REPO_ROOT
timeout 60 /tmp/at 8192 1 | grep -E "event|launch|gdwait|lastmma|drained|issue|full-ready"
timeout 300 python scripts/layer_time.py 8192
