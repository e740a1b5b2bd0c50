#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_shard.py tests/test_gpu_moments.py tests/test_gpu_prohd.py tests/test_gpu_fullsize.py tests/test_gpu_next.py -x -q -k "not exact_full_size_sampled" > gpurun_out/h8_tests.log 2>&1
echo "exit $?" >> gpurun_out/h8_tests.log
for st in 1 0; do PROHD_OPT_EIG_STOP=$st timeout 300 python tools/time_eigen.py; done > gpurun_out/h8_te.txt 2>&1
for cfg in 1 2 3 4 5; do timeout 300 python tools/time_prohd.py $cfg; done > gpurun_out/h8_t.txt 2>&1
