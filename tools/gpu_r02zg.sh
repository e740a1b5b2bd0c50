#!/bin/bash
# K6 two-A kernel: software-pipelined TMEM drain vs the serial drain (build/libprohd_serial.so), pairs per SM clock
mkdir -p gpurun_out
L=paper_2511_18207_b200/libprohd.so
cp $L /tmp/libprohd_pipe.so
run() { timeout 300 python tools/time_k6_clock.py 256 128; }
{ echo "== pipelined"; run; cp build/libprohd_serial.so $L; echo "== serial"; run; cp /tmp/libprohd_pipe.so $L; echo "== pipelined"; run;
  cp build/libprohd_serial.so $L; echo "== serial"; run; cp /tmp/libprohd_pipe.so $L; } > gpurun_out/zg_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_exact.py -q -x > gpurun_out/zg_tests.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:dist_rowmin --launch-count 1 -o /tmp/zg_k6 python tools/prof_k6.py > /dev/null 2>&1
ncu -i /tmp/zg_k6.ncu-rep --page raw --csv > gpurun_out/zg_k6_raw.csv 2>/dev/null
