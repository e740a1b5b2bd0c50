#!/bin/bash
PROHD_OPT_K1_ABLATE=4 ncu --set full --import-source on --clock-control none -k regex:gram_i8_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r02p_k1ab4 python tools/prof_cov.py 5 2 > gpurun_out/r02p_ncu.log 2>&1
