#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/time_exact_small.py 1 2 > gpurun_out/k4_exact_small.txt 2>&1
timeout 300 python tools/time_small.py 1 2 > gpurun_out/k4_small.txt 2>&1
timeout 2400 python -m pytest tests/test_gpu_exact.py tests/test_gpu_next.py tests/test_gpu_prohd.py tests/test_gpu_shard.py -x -q > gpurun_out/k4_tests.log 2>&1
echo "exit $?" >> gpurun_out/k4_tests.log
