#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_shard.py -x -q > gpurun_out/m2_mom.log 2>&1
echo "exit $?" >> gpurun_out/m2_mom.log
for cfg in 1 2 3; do
  PROHD_OPT_K1_PATH=0 timeout 300 python tools/time_prohd.py $cfg | sed "s/^/dmma /"
  timeout 300 python tools/time_prohd.py $cfg | sed "s/^/i8   /"
done > gpurun_out/m2_t.txt 2>&1
timeout 300 python tools/time_small.py 1 2 > gpurun_out/m2_small.txt 2>&1
for cfg in 2 3; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m2_launches_cfg$cfg.csv python tools/prof_prohd.py $cfg > /dev/null 2>&1; done
timeout 1800 python -m pytest tests/test_gpu_prohd.py tests/test_gpu_fullsize.py -x -q -k "not exact_full_size_sampled and not undirected_full" > gpurun_out/m2_prohd.log 2>&1
echo "exit $?" >> gpurun_out/m2_prohd.log
