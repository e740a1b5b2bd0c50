#!/bin/bash
python tools/prof_cov.py 5 5 > gpurun_out/r02h_time.log 2>&1
PROHD_OPT_K1_PATH=0 python tools/prof_cov.py 5 3 >> gpurun_out/r02h_time.log 2>&1
python tools/prof_cov.py 4 5 >> gpurun_out/r02h_time.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches.csv python tools/prof_cov.py 5 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gram_i8_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r02h_k1 python tools/prof_cov.py 5 2 > gpurun_out/r02h_ncu.log 2>&1
