#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eigen_reduce_cluster --launch-count 1 -o /tmp/k7 python tools/time_eigen.py 256 16 > /tmp/k7.log 2>&1
ncu -i /tmp/k7.ncu-rep --page source --csv --print-source sass > gpurun_out/k7_eig_sass.csv 2>/dev/null
ncu -i /tmp/k7.ncu-rep --page raw --csv > gpurun_out/k7_eig_raw.csv 2>/dev/null
ncu -i /tmp/k7.ncu-rep --page details --csv > gpurun_out/k7_eig_details.csv 2>/dev/null
