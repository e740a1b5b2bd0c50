#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sample_thresh --launch-count 1 -o /tmp/r02zy python tools/prof_prohd.py 5 > /tmp/st.log 2>&1
ncu -i /tmp/r02zy.ncu-rep --page source --csv --print-source sass > gpurun_out/r02zy_st_sass.csv 2>/dev/null
ncu -i /tmp/r02zy.ncu-rep --page raw --csv > gpurun_out/r02zy_st_raw.csv 2>/dev/null
