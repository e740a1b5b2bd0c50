#!/bin/bash
# final check of HEAD (pair K6 for directed and bidirectional sweeps): full GPU suite, smoke, per-config report, small-D pair probe
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/l_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/l_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/l_smoke.log 2>&1
timeout 600 python tools/report_configs.py --json gpurun_out/l_configs.json > gpurun_out/l_configs.txt 2>&1
timeout 300 python tools/probe_pair_small_d.py > gpurun_out/l_small_d.txt 2>&1
