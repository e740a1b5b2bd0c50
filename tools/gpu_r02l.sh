#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_moments.py -x -q -s -k "covariance" 2>&1 | tail -12 > gpurun_out/r02l_cov.log
python tools/prof_cov.py 5 5 > gpurun_out/r02l_time.log 2>&1
python tools/prof_cov.py 4 5 >> gpurun_out/r02l_time.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_launches.csv python tools/prof_cov.py 5 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gram_i8_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r02l_k1 python tools/prof_cov.py 5 2 > gpurun_out/r02l_ncu.log 2>&1
