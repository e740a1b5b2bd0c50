#!/bin/bash
# K6 fp16x3 split: probe, parity tests, bench
timeout 300 python tools/split_probe.py > gpurun_out/r02c_probe.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_exact.py tests/test_gpu_prohd.py tests/test_gpu_next.py tests/test_gpu_shard.py -x -q -s 2>&1 | tail -60 > gpurun_out/r02c_tests.log
timeout 400 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
