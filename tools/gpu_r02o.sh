#!/bin/bash
for ab in 3 4 5; do PROHD_OPT_K1_ABLATE=$ab ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r02o_l$ab.csv python tools/prof_cov.py 5 2 > /dev/null 2>&1; done
