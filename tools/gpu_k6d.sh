mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_exact.py tests/test_gpu_next.py tests/test_gpu_fullsize.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_k6d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k6d.log
timeout 600 python tools/time_exact.py > gpurun_out/time_k6d.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
