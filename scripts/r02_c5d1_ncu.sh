mkdir -p gpurun_out
for v in old new; do
  if [ $v = old ]; then export BLR_LIB=$PWD/paper_2512_20861_b200/libblr_old.so; else unset BLR_LIB; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic --clock-control none -k regex:"blr_|blast_" --csv --log-file gpurun_out/c5d1_$v.csv python bench.py --config C5D-1 --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-variants --eager > /dev/null 2>&1
done
