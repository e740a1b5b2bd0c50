#!/bin/bash
# fused bidirectional sweep on the CTA-pair K6 (option k6_bidir_2a = 2): parity, A/B timing, then the
# suites that run hausdorff()/subset HD with the option forced as a candidate default
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exact.py -q -x -k "bidirectional_cta_pair" > gpurun_out/j_tests.txt 2>&1
echo "exit $?" >> gpurun_out/j_tests.txt
if grep -q "passed" gpurun_out/j_tests.txt && ! grep -q "failed\|error" gpurun_out/j_tests.txt; then
  timeout 600 python tools/time_bidir_pair.py > gpurun_out/j_ab.txt 2>&1
  for v in 0 2; do for cfg in 3 4 5; do echo "== k6_bidir_2a=$v cfg$cfg"; PROHD_OPT_K6_BIDIR_2A=$v timeout 300 python tools/time_prohd.py $cfg; done; done > gpurun_out/j_prohd.txt 2>&1
  PYTHONPATH=tools PROHD_OPT_K6_BIDIR_2A=2 timeout 2400 python -m pytest -p pytest_force_opts -q -x -m gpu \
    tests/test_gpu_exact.py tests/test_gpu_prohd.py tests/test_gpu_next.py tests/test_gpu_shard.py \
    "tests/test_gpu_fullsize.py::test_undirected_full_size_sampled" "tests/test_gpu_fullsize.py::test_prohd_full_size" \
    > gpurun_out/j_forced_tests.txt 2>&1
  echo "exit $?" >> gpurun_out/j_forced_tests.txt
fi
