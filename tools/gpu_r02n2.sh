#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_shard.py -x -q > gpurun_out/n2_eig.log 2>&1
echo "exit $?" >> gpurun_out/n2_eig.log
for st in 1 0; do PROHD_OPT_EIG_STOP=$st timeout 300 python tools/time_eigen.py; done > gpurun_out/n2_te.txt 2>&1
for cfg in 2 3; do timeout 300 python tools/time_prohd.py $cfg; done >> gpurun_out/n2_te.txt 2>&1
