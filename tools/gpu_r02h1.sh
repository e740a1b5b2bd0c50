#!/bin/bash
# D <= 128 int8 Gram (gram_i8s_kernel) + sharded int8 moments: tests and timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_shard.py -x -q > gpurun_out/h1_mom.log 2>&1
echo "exit $?" >> gpurun_out/h1_mom.log
for cfg in 1 2 3 5; do
  PROHD_OPT_K1_PATH=0 timeout 300 python tools/time_prohd.py $cfg | sed "s/^/dmma /"
  timeout 300 python tools/time_prohd.py $cfg | sed "s/^/i8   /"
done > gpurun_out/h1_t.txt 2>&1
timeout 300 python tools/time_small.py 1 2 > gpurun_out/h1_small.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_prohd.py tests/test_gpu_fullsize.py tests/test_gpu_next.py -x -q -k "not exact_full_size_sampled" > gpurun_out/h1_prohd.log 2>&1
echo "exit $?" >> gpurun_out/h1_prohd.log
