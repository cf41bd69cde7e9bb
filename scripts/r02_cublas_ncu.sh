#!/bin/bash
# ncu full-set captures of the cuBLAS kernels on the C4 grouped shapes (what tile / cluster / pipe
# utilisation a vendor kernel reaches on exactly these GEMMs)
mkdir -p gpurun_out
for s in gateS3 downS1 dense; do
  ncu --set full --clock-control none -k regex:'nvjet|gemm' -c 1 --export gpurun_out/cublas_$s -f \
      python scripts/cublas_probe.py $s > gpurun_out/cublas_$s.log 2>&1
  ncu -i gpurun_out/cublas_$s.ncu-rep --page raw --csv > gpurun_out/cublas_$s.csv 2>/dev/null
  ncu -i gpurun_out/cublas_$s.ncu-rep --page details > gpurun_out/cublas_$s.txt 2>/dev/null
  rm -f gpurun_out/cublas_$s.ncu-rep
done
