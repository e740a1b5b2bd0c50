#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_prohd.py -x -q -k "wide_d or separated or asym or cfg4_like or tight or rank" > gpurun_out/k5_tests.log 2>&1
echo "exit $?" >> gpurun_out/k5_tests.log
for st in 1 0; do PROHD_OPT_EIG_STOP=$st timeout 300 python tools/time_eigen.py; done > gpurun_out/k5_te.txt 2>&1
timeout 300 python tools/time_eigen.py 512 16 >> gpurun_out/k5_te.txt 2>&1
