#!/bin/bash
# check of HEAD with the fused bidirectional sweep on the CTA-pair K6 by default: the suites that run
# hausdorff()/subset HD, smoke, bench, bench launch list, ncu --set full of one bidirectional pair launch
mkdir -p gpurun_out
timeout 2400 python -m pytest -q -x -m gpu tests/test_gpu_exact.py tests/test_gpu_prohd.py tests/test_gpu_next.py \
  tests/test_gpu_shard.py tests/test_gpu_select.py "tests/test_gpu_fullsize.py::test_undirected_full_size_sampled" \
  "tests/test_gpu_fullsize.py::test_prohd_full_size" > gpurun_out/k_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/k_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/k_smoke.log 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/k_launches_cfg5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:dist_rowmin --launch-count 1 -o /tmp/k_k6 python tools/prof_k6.py 256 bidir > /dev/null 2>&1
ncu -i /tmp/k_k6.ncu-rep --page raw --csv > gpurun_out/k_k6_bidir_raw.csv 2>/dev/null
