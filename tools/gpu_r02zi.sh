#!/bin/bash
# round-2 final check of HEAD (K6 CTA-pair kernel as the default directed sweep): GPU suite, smoke, bench, ProHD timings, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/i_smi.txt
timeout 3000 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/i_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke.log 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err
for cfg in 1 2 3 4 5; do timeout 300 python tools/time_prohd.py $cfg; done > gpurun_out/i_prohd.txt 2>&1
timeout 600 python tools/report_configs.py --json gpurun_out/i_configs.json > gpurun_out/i_configs.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/i_launches_cfg5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
