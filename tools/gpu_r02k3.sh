#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_shard.py -x -q > gpurun_out/k3_eig.log 2>&1
echo "exit $?" >> gpurun_out/k3_eig.log
for st in 1 2 3 0; do PROHD_OPT_EIG_STOP=$st timeout 300 python tools/time_eigen.py; done > gpurun_out/k3_te.txt 2>&1
timeout 300 python tools/time_small.py 1 2 > gpurun_out/k3_small.txt 2>&1
PROHD_OPT_GRAPH=0 timeout 300 python tools/time_small.py 1 2 > gpurun_out/k3_small_nograph.txt 2>&1
for cfg in 3 4 5; do timeout 300 python tools/time_prohd.py $cfg; done > gpurun_out/k3_t.txt 2>&1
