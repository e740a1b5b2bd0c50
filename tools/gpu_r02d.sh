#!/bin/bash
# full GPU suite after the fp16 K6, band-select fallback, full-size parity at 20k rows
nproc; lscpu | grep "Model name"
timeout 600 python -m pytest tests/test_gpu_prohd.py -x -q -s -k "overflow" 2>&1 | tail -15 > gpurun_out/r02d_overflow.log
timeout 3000 python -m pytest tests -m gpu -q -s --durations=15 2>&1 | tail -80 > gpurun_out/r02d_tests.log
