#!/bin/bash
# check of the bidirectional kernel rule (pair up to nA nB D = 1e14, single-block above): exact/ProHD suites, full-size undirected, smoke, per-config report
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/n_smoke.log 2>&1
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_exact.py tests/test_gpu_prohd.py tests/test_gpu_next.py \
  "tests/test_gpu_fullsize.py::test_undirected_full_size_sampled" > gpurun_out/n_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/n_tests.log
timeout 400 python tools/report_configs.py --json gpurun_out/n_configs.json > gpurun_out/n_configs.txt 2>&1
