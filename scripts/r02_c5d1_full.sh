#!/bin/bash
# ncu --set full of C5D-1's fc1 S3 launch (launch 5 of the step) under the round-2-start build and HEAD
# with the same plan (HEAD: BLR_RESIDENT=1 BLR_KBOX=2 reproduces the old plan): where the cycles went
mkdir -p gpurun_out
for v in old new; do
  if [ $v = old ]; then export BLR_LIB=$PWD/paper_2512_20861_b200/libblr_old.so; unset BLR_RESIDENT BLR_KBOX;
  else unset BLR_LIB; export BLR_RESIDENT=1 BLR_KBOX=2; fi
  timeout 600 ncu --set full --clock-control none -k regex:"blr_gemm" --launch-skip 3 --launch-count 1 -o gpurun_out/c5d1_full_$v -f \
     python bench.py --config C5D-1 --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-variants --eager > /dev/null 2>&1
  ncu -i gpurun_out/c5d1_full_$v.ncu-rep --page raw --csv > gpurun_out/c5d1_full_$v.csv 2>/dev/null
  ncu -i gpurun_out/c5d1_full_$v.ncu-rep --page details > gpurun_out/c5d1_full_$v.txt 2>/dev/null
  rm -f gpurun_out/c5d1_full_$v.ncu-rep
done
