#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_eigen.py -x -q > gpurun_out/k8_eig.log 2>&1
echo "exit $?" >> gpurun_out/k8_eig.log
for st in 1 0; do PROHD_OPT_EIG_STOP=$st timeout 300 python tools/time_eigen.py; done > gpurun_out/k8_te.txt 2>&1
timeout 300 python tools/time_eigen.py 512 16 >> gpurun_out/k8_te.txt 2>&1
