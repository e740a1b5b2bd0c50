#!/bin/bash
# round-2: coalesced int8 drains, 682-chunk drain window: timing, moments/prohd tests
mkdir -p gpurun_out
python tools/prof_cov.py 5 6 > gpurun_out/r02y_cov.txt 2>&1
python tools/prof_cov.py 4 6 >> gpurun_out/r02y_cov.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_shard.py tests/test_gpu_prohd.py -x -q -s > gpurun_out/r02y_tests.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/r02y_cov_launches.csv python tools/prof_cov.py 5 2 > /tmp/ncu_cov.log 2>&1
