mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 3 > gpurun_out/gb_bench.json 2> gpurun_out/gb_bench.err; echo "rc=$?" >> gpurun_out/gb_bench.err
PROHD_K6_BIDIR_2A=1 timeout 600 python tools/report_configs.py 3 4 5 > gpurun_out/gb_bidir2a.md 2>&1
