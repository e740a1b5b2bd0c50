#!/bin/bash
python tools/prof_cov.py 5 4 > gpurun_out/r02m_time.log 2>&1
PROHD_OPT_K1_ABLATE=1 python tools/prof_cov.py 5 4 >> gpurun_out/r02m_time.log 2>&1
PROHD_OPT_K1_ABLATE=2 python tools/prof_cov.py 5 4 >> gpurun_out/r02m_time.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_l0.csv python tools/prof_cov.py 5 2 > /dev/null 2>&1
PROHD_OPT_K1_ABLATE=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_l1.csv python tools/prof_cov.py 5 2 > /dev/null 2>&1
PROHD_OPT_K1_ABLATE=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_l2.csv python tools/prof_cov.py 5 2 > /dev/null 2>&1
