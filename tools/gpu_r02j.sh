#!/bin/bash
# round-2 checkpoint j: full GPU suite, smoke, bench, per-config report, launch list, ncu captures
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/j_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/j_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j_smoke.log 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/j_bench.json 2> gpurun_out/j_bench.err
timeout 1500 python tools/report_configs.py --json gpurun_out/j_configs.json > gpurun_out/j_configs.md 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/j_launches_cfg5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for cfg in 3 5; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_i8|eigen_|i8_colmax|project_tc|sample_thresh|rank_kernel" -o /tmp/j_cfg$cfg python tools/prof_prohd.py $cfg > /dev/null 2>&1
ncu -i /tmp/j_cfg$cfg.ncu-rep --page raw --csv > gpurun_out/j_prohd_cfg${cfg}_raw.csv 2>/dev/null
done
