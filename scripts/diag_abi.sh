#!/bin/bash
# bash scripts/diag_abi.sh "0 12" [flush 0/1]  -- abi_trace (LR c_fc) under BLR_DBG variants; env passes through
cd $GRAFT_REPO_ROOT/benchmarks/micro && nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/at abi_trace.cu \
  -L../../paper_2512_20861_b200 -lblr -Xlinker -rpath=$GRAFT_REPO_ROOT/paper_2512_20861_b200 || exit 1
cd $GRAFT_REPO_ROOT
for v in $1; do echo "== DBG $v"; BLR_DBG=$v timeout 60 /tmp/at 8192 ${2:-1} | grep -E "event|launch|gdwait|lastmma|drained|issue|full-ready"; done
