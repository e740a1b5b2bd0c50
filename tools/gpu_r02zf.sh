#!/bin/bash
# round-2 re-entry check of HEAD (D <= 64 int8 Gram, 16-CTA K2 cluster): GPU suite, smoke, bench, ProHD timings, launch list, cfg2 ncu
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/g_smi.txt
timeout 3000 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/g_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
for cfg in 1 2 3 4 5; do timeout 300 python tools/time_prohd.py $cfg; done > gpurun_out/g_prohd.txt 2>&1
timeout 300 python tools/time_small.py 1 2 > gpurun_out/g_small.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g_launches_cfg5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gram_i8|eigen_|i8_colmax" -o /tmp/g_cfg2 python tools/prof_prohd.py 2 > /dev/null 2>&1
ncu -i /tmp/g_cfg2.ncu-rep --page raw --csv > gpurun_out/g_prohd_cfg2_raw.csv 2>/dev/null
