#!/bin/bash
# round-2 re-entry: full GPU suite + smoke + bench + launch list at HEAD
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/h0_smi.txt
timeout 3000 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/h0_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/h0_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h0_smoke.log 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/h0_bench.json 2> gpurun_out/h0_bench.err
python tools/time_prohd.py 5 4 3 > gpurun_out/h0_prohd.txt 2>&1
