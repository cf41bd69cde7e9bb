#!/bin/bash
# A/B of the streaming tile order (BLR_ORDER=0 plain round robin vs default N-block runs) + tests
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "transposed or robustness or pair or split" > gpurun_out/q_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/q_pytest.txt
for o in 0 1; do
  for c in C4 C4M; do
    BLR_ORDER=$o timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/ord${o}_$c.json 2>gpurun_out/ord${o}_$c.err
  done
done
