#!/bin/bash
# token-chunked weight-streaming path: parity, then small-n configs default vs forced
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py -m gpu -q -x > gpurun_out/chunk_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/chunk_pytest.txt
for c in C1 C5V-1 C5V-8 C5D-1 C5D-8 C2 C3; do
  for mx in 0; do
    if [ $mx = 0 ]; then E=""; else E="BLR_DECODE_MAXN=$mx"; fi
    env $E timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-variants --no-cpu-baseline > gpurun_out/chunk_tmp.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/chunk_tmp.json').read().strip().splitlines()[-1])
print('$c', 'maxn=$mx', round(d['ms_per_step']*1e3,1), 'us  x_cublas', round(d.get('speedup_vs_cublas',0),3))" >> gpurun_out/chunk_bench.txt 2>&1
  done
done
