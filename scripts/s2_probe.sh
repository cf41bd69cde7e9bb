#!/bin/bash
# BLAST split-path S2 variants: per-launch times (ncu launch list) + one full capture.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -k blast -p no:cacheprovider 2>&1 | tail -15
for v in "BLR_S2=mma" "BLR_S2=cuda"; do
  env $v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"blast_s2|blr_gemm" -c 6 --csv \
    python scripts/one_call.py blast Llama-7B gate_up_proj 65536 2 2>/dev/null | grep -E "gpu__time|dram__" | awk -F'","' -v V="$v" '{print V, $(NF-2), $NF}'
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:blast_s2 -c 1 -o gpurun_out/s2_full -f \
   python scripts/one_call.py blast Llama-7B gate_up_proj 65536 1 > /dev/null 2>&1; echo "full rc=$?"
