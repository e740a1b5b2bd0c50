mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_exact.py tests/test_gpu_next.py tests/test_gpu_prohd.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_k6e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k6e.log
timeout 300 python tools/time_bidir.py > gpurun_out/time_bidir.txt 2>&1
PROHD_K6_VARIANT=1 timeout 300 python tools/time_bidir.py > gpurun_out/time_bidir1.txt 2>&1
timeout 300 python tools/time_prohd.py 5 4 3 > gpurun_out/time_prohd.txt 2>&1
