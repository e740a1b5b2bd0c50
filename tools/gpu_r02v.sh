#!/bin/bash
# functional multi-rank bench (2 ranks sharing the one GPU over gloo; timings meaningless)
export PROHD_BENCH_BACKEND=gloo
timeout 900 python bench.py --gpus 2 --config 2 --steps 2 --warmup 1 > gpurun_out/r02v_mr2.json 2> gpurun_out/r02v_mr2.err
timeout 1200 python bench.py --gpus 2 --config 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02v_mr5.json 2> gpurun_out/r02v_mr5.err
tail -5 gpurun_out/r02v_mr2.err
