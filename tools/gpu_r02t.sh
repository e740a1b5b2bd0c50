#!/bin/bash
# full GPU suite + bench after the int8 K1
timeout 3000 python -m pytest tests -m gpu -q -s --durations=10 2>&1 | tail -60 > gpurun_out/r02t_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02t_bench.json 2> gpurun_out/r02t_bench.err
