#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_shard.py tests/test_gpu_prohd.py tests/test_gpu_fullsize.py tests/test_gpu_next.py -x -q -k "not exact_full_size_sampled" > gpurun_out/h5_tests.log 2>&1
echo "exit $?" >> gpurun_out/h5_tests.log
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_shard.py tests/test_gpu_eigen.py -x -q >> gpurun_out/h5_rep.log 2>&1; done
for st in 1 0; do PROHD_OPT_EIG_STOP=$st timeout 300 python tools/time_eigen.py; done > gpurun_out/h5_te.txt 2>&1
