#!/bin/bash
# round-2: sampled-threshold K4 (K3 on the sample, smem-staged selects): tests, timing, K3 profile
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_prohd.py -x -q -k "sampled or guard or reduced" > gpurun_out/r02z_tests.txt 2>&1
python tools/time_prohd.py 5 4 3 2 > gpurun_out/r02z_prohd.txt 2>&1
PROHD_OPT_K4_SAMPLED=0 python tools/time_prohd.py 5 >> gpurun_out/r02z_prohd.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z_launches_cfg5.csv python tools/prof_prohd.py 5 > /tmp/ncu5.log 2>&1



