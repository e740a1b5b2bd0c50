#!/bin/bash
# round-2: fused K3 ablations (k4_sampled 2: no tests, 3: no appends)
mkdir -p gpurun_out
for v in 1; do
PROHD_OPT_K4_SAMPLED=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:project_tc --log-file gpurun_out/r02zz_abl$v.csv python tools/prof_prohd.py 5 > /tmp/a$v.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_prohd.py -x -q -k "sampled or guard or reduced or ties or w3 or w5 or cfg1" > gpurun_out/r02zz_tests.txt 2>&1
python tools/time_prohd.py 5 4 3 > gpurun_out/r02zz_t.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02zz_launches.csv python tools/prof_prohd.py 5 > /tmp/ncu5.log 2>&1
