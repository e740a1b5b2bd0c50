#!/bin/bash
# K2 single-CTA register tail + pairwise back-transform + rsqrt; CUDA-graph replay of prohd_estimate
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eigen.py -x -q > gpurun_out/k2_eig.log 2>&1
echo "exit $?" >> gpurun_out/k2_eig.log
for st in 1 2 3 0; do PROHD_OPT_EIG_STOP=$st timeout 300 python tools/time_eigen.py; done > gpurun_out/k2_te.txt 2>&1
timeout 300 python tools/time_small.py 1 2 > gpurun_out/k2_small.txt 2>&1
for cfg in 3 4 5; do timeout 300 python tools/time_prohd.py $cfg; done > gpurun_out/k2_t.txt 2>&1
timeout 2400 python -m pytest tests/test_gpu_prohd.py tests/test_gpu_shard.py tests/test_gpu_fullsize.py tests/test_gpu_next.py tests/test_gpu_moments.py -x -q -k "not exact_full_size_sampled" > gpurun_out/k2_tests.log 2>&1
echo "exit $?" >> gpurun_out/k2_tests.log
