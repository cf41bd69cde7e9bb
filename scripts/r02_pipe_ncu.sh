#!/bin/bash
# DRAM bytes of one C4 gate layer: three launches vs the pipelined one-launch layer (ncu)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for e in "BLR_PIPE=0" "BLR_PIPE=1 BLR_PIPE_SPLIT=14,16"; do
  env $e SCAN_N=65536 timeout 900 ncu -c 3 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"blr_gemm|blast_s2|blast_pipe" --csv python scripts/scan.py blast Llama-7B gate_up_proj > gpurun_out/pipe_ncu_raw.csv 2>/dev/null
  echo "== $e"; python - <<'PY'
import csv, io
rows = [r for r in csv.reader(open('gpurun_out/pipe_ncu_raw.csv')) if len(r) > 10]
hdr = rows[0]; data = rows[1:]
ik = hdr.index("Kernel Name"); im = hdr.index("Metric Name"); iv = hdr.index("Metric Value"); iu = hdr.index("Metric Unit"); iid = hdr.index("ID")
from collections import defaultdict
per = defaultdict(dict)
for r in data:
    per[(r[iid], r[ik][:40])][r[im]] = (r[iv], r[iu])
for k, v in list(per.items())[:8]:
    print(k, {m: v[m] for m in v})
PY
done > gpurun_out/pipe_ncu.txt 2>&1
