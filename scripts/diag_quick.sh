#!/bin/bash
# quick perf check: graph layer times for C2 (+ env variants given as args, e.g. "BLR_DIRECT=0")
cd $GRAFT_REPO_ROOT
echo "== default"; timeout 300 python scripts/layer_time.py 8192
for v in "$@"; do echo "== $v"; env $v timeout 300 python scripts/layer_time.py 8192; done
