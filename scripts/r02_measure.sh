#!/bin/bash
# round-2 measurement pass: GPU tests, smoke, default bench line, per-config bench lines, ncu
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/m_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/m_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/m_smoke.txt
timeout 900 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
for c in C1 C2 C3 C5V-1 C5V-8 C5V-64 C5V-256 C5D-1 C5D-8 C5D-64 C5D-256; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-variants --no-cpu-baseline > gpurun_out/m_bench_$c.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m_launches.csv python bench.py --steps 2 --warmup 1 --no-variants --no-cpu-baseline --no-dense > /dev/null 2>&1
BLR_DUMP_PHASES=gpurun_out/m_phases.json timeout 300 python bench.py --steps 1 --warmup 0 --no-variants --no-cpu-baseline --no-dense --eager > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"blr_|blast_" -c 6 -o gpurun_out/m_prof_C4 -f python bench.py --config C4 --steps 1 --warmup 0 --no-dense --no-cpu-baseline --no-variants --eager > gpurun_out/m_ncu.log 2>&1
