#!/bin/bash
# round-2: K2 split cluster barrier: timing + eigen tests
mkdir -p gpurun_out
python tools/time_eigen.py > gpurun_out/r02z_eigen.txt 2>&1
PROHD_OPT_EIG_STOP=1 python tools/time_eigen.py >> gpurun_out/r02z_eigen.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_eigen.py -x -q > gpurun_out/r02z_tests.txt 2>&1
