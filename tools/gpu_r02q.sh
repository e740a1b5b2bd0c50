#!/bin/bash
for ab in 0 4; do PROHD_OPT_K1_ABLATE=$ab ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02q_l$ab.csv python tools/prof_cov.py 5 2 > /dev/null 2>&1; done
python tools/prof_cov.py 5 4 > gpurun_out/r02q_time.log 2>&1
timeout 600 python -m pytest tests/test_gpu_moments.py -x -q -s -k "covariance" 2>&1 | tail -3 > gpurun_out/r02q_cov.log
