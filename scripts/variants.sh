#!/bin/bash
# time one layer's kernels under plan-variant env overrides
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
M=${1:-monarch}; MODEL=${2:-Llama-7B}; LAYER=${3:-down_proj}
for v in "BLR_PAIR=1" "BLR_PAIR=2" "BLR_PAIR=1 BLR_NO_RESIDENT=1" "BLR_PAIR=2 BLR_NO_RESIDENT=1" "BLR_PAIR=1 BLR_KBOX=1" "BLR_PAIR=2 BLR_NO_RESIDENT=1 BLR_KBOX=1"; do
  echo "== $v"; env $v python scripts/scan.py $M $MODEL $LAYER 2>&1 | tail -1
done
