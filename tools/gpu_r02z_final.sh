#!/bin/bash
# round-2 final: full GPU suite, smoke, bench, per-config report, launch list, ncu captures, 2-rank functional run
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/f_smi.txt
timeout 3000 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/f_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
for cfg in 1 2 3 4 5; do timeout 300 python tools/time_prohd.py $cfg; done > gpurun_out/f_prohd.txt 2>&1
timeout 300 python tools/time_small.py 1 2 > gpurun_out/f_small.txt 2>&1
timeout 300 python tools/time_exact_small.py 1 2 >> gpurun_out/f_small.txt 2>&1
timeout 1500 python tools/report_configs.py --json gpurun_out/f_configs.json > gpurun_out/f_configs.md 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_cfg5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_i8|eigen_|i8_colmax|project_tc|sample_thresh|rank_kernel" -o /tmp/f_cfg5 python tools/prof_prohd.py 5 > /dev/null 2>&1
ncu -i /tmp/f_cfg5.ncu-rep --page raw --csv > gpurun_out/f_prohd_cfg5_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:"gram_i8|eigen_|i8_colmax" -o /tmp/f_cfg2 python tools/prof_prohd.py 2 > /dev/null 2>&1
ncu -i /tmp/f_cfg2.ncu-rep --page raw --csv > gpurun_out/f_prohd_cfg2_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:dist_rowmin --launch-count 1 -o /tmp/f_k6 python tools/prof_k6.py > /dev/null 2>&1
ncu -i /tmp/f_k6.ncu-rep --page raw --csv > gpurun_out/f_k6_raw.csv 2>/dev/null
export PROHD_BENCH_BACKEND=gloo
timeout 900 python bench.py --gpus 2 --config 2 --steps 2 --warmup 1 > gpurun_out/f_mr2.json 2> gpurun_out/f_mr2.err
timeout 1500 python bench.py --gpus 2 --config 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/f_mr5.json 2> gpurun_out/f_mr5.err
