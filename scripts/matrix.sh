#!/bin/bash
# step time for eager/graph x PDL on/off (C2), plus a trace of one layer
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for mode in "" "--eager"; do for pdl in 0 1; do
  BLR_NO_PDL=$pdl python bench.py --no-cpu-baseline --steps 30 $mode > gpurun_out/m.json 2>gpurun_out/m.err || tail -3 gpurun_out/m.err
  echo "== mode=${mode:-graph} no_pdl=$pdl"; python scripts/summarize.py gpurun_out/m.json | head -9
done; done
