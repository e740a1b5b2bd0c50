#!/bin/bash
# K6 CTA-pair kernel (option k6_variant 2): parity tests, then interleaved A/B against the two-A kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_exact.py -q -x -k "cta_pair" > gpurun_out/zh_tests.txt 2>&1
echo "exit $?" >> gpurun_out/zh_tests.txt
if grep -q "passed" gpurun_out/zh_tests.txt && ! grep -q "failed\|error" gpurun_out/zh_tests.txt; then
  { for i in 1 2; do
      echo "== two-A (default)"; timeout 300 python tools/time_k6_clock.py 256 128
      echo "== pair"; PROHD_OPT_K6_VARIANT=2 timeout 300 python tools/time_k6_clock.py 256 128
    done; } > gpurun_out/zh_ab.txt 2>&1
  PROHD_OPT_K6_VARIANT=2 timeout 600 ncu --set full --clock-control none -k regex:dist_rowmin --launch-count 1 -o /tmp/zh_k6 python tools/prof_k6.py > /dev/null 2>&1
  ncu -i /tmp/zh_k6.ncu-rep --page raw --csv > gpurun_out/zh_k6_raw.csv 2>/dev/null
fi
