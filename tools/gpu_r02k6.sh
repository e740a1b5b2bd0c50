#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_eigen.py -x -q > gpurun_out/k6_eig.log 2>&1
echo "exit $?" >> gpurun_out/k6_eig.log
for st in 1 0; do PROHD_OPT_EIG_STOP=$st timeout 300 python tools/time_eigen.py; done > gpurun_out/k6_te.txt 2>&1
PROHD_OPT_EIG_CL=8 PROHD_OPT_EIG_STOP=1 timeout 300 python tools/time_eigen.py >> gpurun_out/k6_te.txt 2>&1
timeout 300 python tools/time_small.py 1 2 > gpurun_out/k6_small.txt 2>&1
timeout 300 python tools/time_prohd.py 3 >> gpurun_out/k6_small.txt 2>&1
timeout 2400 python -m pytest tests/test_gpu_prohd.py tests/test_gpu_shard.py tests/test_gpu_next.py -x -q > gpurun_out/k6_tests.log 2>&1
echo "exit $?" >> gpurun_out/k6_tests.log
