#!/bin/bash
# K2 register-resident column (no CTA barriers per step) + small-D int8 reduce
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_moments.py -x -q > gpurun_out/h3_eig.log 2>&1
echo "exit $?" >> gpurun_out/h3_eig.log
for st in 1 0; do PROHD_OPT_EIG_STOP=$st timeout 300 python tools/time_eigen.py; done > gpurun_out/h3_te.txt 2>&1
for cfg in 1 2 3 4 5; do timeout 300 python tools/time_prohd.py $cfg; done > gpurun_out/h3_t.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_prohd.py tests/test_gpu_fullsize.py tests/test_gpu_next.py tests/test_gpu_shard.py -x -q -k "not exact_full_size_sampled" > gpurun_out/h3_prohd.log 2>&1
echo "exit $?" >> gpurun_out/h3_prohd.log
