#!/bin/bash
# round 2 check: K6 RN split (exact tests incl. the adversarial mantissas), prohd/select smoke
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_prohd.py -x -q -s 2>&1 | tail -40 > gpurun_out/r02a_tests.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
tail -3 gpurun_out/r02a_bench.err
