#!/bin/bash
# (produced profiles/r02_lastn_ab.txt)
# narrow last-N-tile MMA (KParams::last_nb): parity/bitwise tests + A/B against BLR_LASTN=0
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_wide.py tests/test_gpu_fuzz.py -x -q > gpurun_out/lastn_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/lastn_tests.txt
tail -3 gpurun_out/lastn_tests.txt | grep -q " passed" || exit 1
timeout 300 python scripts/ab.py C4 "" "BLR_LASTN=0" --reps 12 --layer 0 > gpurun_out/lastn_ab.txt 2>&1
timeout 300 python scripts/ab.py C4 "" "BLR_LASTN=0" --reps 12 >> gpurun_out/lastn_ab.txt 2>&1
for c in C4M C4X C3 C2 C5V-256 C5D-256; do timeout 300 python scripts/ab.py $c "" "BLR_LASTN=0" --reps 10 >> gpurun_out/lastn_ab.txt 2>&1; done
