#!/bin/bash
# gutted builds (BLR_GUT=1 plain release, 2 commit release, 3 + accumulator hand-off) vs normal; expand only, Z hot
cd $GRAFT_REPO_ROOT
for g in 1 2 3; do
  mkdir -p /tmp/gut$g && nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -DBLR_GUT=$g -I include \
   -o /tmp/gut$g/libblr.so paper_2512_20861_b200/csrc/*.cu || exit 1
  (cd benchmarks/micro && nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/at_gut$g abi_trace.cu -L/tmp/gut$g -lblr -Xlinker -rpath=/tmp/gut$g) || exit 1
done
(cd benchmarks/micro && nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/at abi_trace.cu -L../../paper_2512_20861_b200 -lblr -Xlinker -rpath=$GRAFT_REPO_ROOT/paper_2512_20861_b200) || exit 1
for b in at_gut1 at_gut2 at_gut3 at; do echo "== $b"; BLR_DBG_LAUNCH=1 BLR_DBG=${DBG:-12} BLR_DBG_SKIP_S1=1 BLR_PAIR=1 timeout 60 /tmp/$b 8192 0 | grep -E "event|gdwait|lastmma|full-ready|issue"; done
