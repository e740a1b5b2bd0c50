#!/bin/bash
mkdir -p gpurun_out
for cl in -1 8 16; do PROHD_OPT_EIG_CL=$cl PROHD_OPT_EIG_STOP=1 timeout 300 python tools/time_eigen.py | sed "s/^/cl=$cl /"; done > gpurun_out/n_cl.txt 2>&1
