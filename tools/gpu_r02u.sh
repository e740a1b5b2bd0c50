#!/bin/bash
# round-2 profiles: per-config report, bench launch list, K6 / ProHD ncu captures (raw CSV exports)
mkdir -p gpurun_out
python tools/report_configs.py --json gpurun_out/r02u_configs.json > gpurun_out/r02u_configs.md 2> gpurun_out/r02u_configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02u_launches_cfg5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /tmp/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dist_rowmin_2a --launch-count 1 -o /tmp/r02u_k6 python tools/prof_k6.py 256 > /tmp/k6.log 2>&1
ncu -i /tmp/r02u_k6.ncu-rep --page raw --csv > gpurun_out/r02u_k6_raw.csv 2>/dev/null
ncu -i /tmp/r02u_k6.ncu-rep --page details --csv > gpurun_out/r02u_k6_details.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none -o /tmp/r02u_prohd python tools/prof_prohd.py 5 > /tmp/prohd.log 2>&1
ncu -i /tmp/r02u_prohd.ncu-rep --page raw --csv > gpurun_out/r02u_prohd_raw.csv 2>/dev/null
du -sh gpurun_out
