#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/time_small.py 1 2 > gpurun_out/h9_small.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_prohd.py tests/test_gpu_next.py tests/test_gpu_shard.py tests/test_gpu_select.py -x -q > gpurun_out/h9_tests.log 2>&1
echo "exit $?" >> gpurun_out/h9_tests.log
