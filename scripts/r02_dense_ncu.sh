#!/bin/bash
# ncu --set full of the dense-shape S3 GEMM: ours (256-column tiles), ours (BLR_WIDE=1), cuBLAS;
# clocks, tensor-pipe activity, instruction counts, L2->SM bytes side by side
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
PROBE_ONCE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'blr_gemm|nvjet' \
  -o gpurun_out/dense_ncu -f python scripts/dense_probe.py "" "BLR_WIDE=1" > gpurun_out/dense_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/dense_ncu.ncu-rep --page raw --csv > gpurun_out/dense_ncu.csv 2>/dev/null
for i in 1 3; do
  ncu -i gpurun_out/dense_ncu.ncu-rep --page source --csv --launch-skip $i --launch-count 1 --print-source cuda > gpurun_out/dense_src_$i.csv 2>/dev/null
  python scripts/ncu_stalls.py gpurun_out/dense_src_$i.csv 40 > gpurun_out/dense_stalls_$i.txt 2>&1
done
ls -la gpurun_out/dense_ncu.ncu-rep
[ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/dense_ncu.ncu-rep
