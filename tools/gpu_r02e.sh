#!/bin/bash
timeout 300 python tools/dbg_perrow.py > gpurun_out/r02e_dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_moments.py -x -q -s -k "covariance" 2>&1 | tail -30 > gpurun_out/r02e_cov.log
