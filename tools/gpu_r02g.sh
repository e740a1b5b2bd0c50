#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_exact.py -x -q -s -k "covariance or wide_dynamic" 2>&1 | tail -30 > gpurun_out/r02g_cov.log
timeout 1500 python -m pytest tests/test_gpu_prohd.py tests/test_gpu_fullsize.py -x -q -s -k "not undirected and not exact_full" 2>&1 | tail -40 > gpurun_out/r02g_prohd.log
timeout 400 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
