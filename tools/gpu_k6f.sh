mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_exact.py tests/test_gpu_next.py tests/test_gpu_prohd.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_k6f.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k6f.log
timeout 300 python tools/time_bidir.py > gpurun_out/time_bidir.txt 2>&1
timeout 300 python tools/time_exact.py > gpurun_out/time_k6f.txt 2>&1
timeout 300 python tools/time_prohd.py 5 4 3 2 > gpurun_out/time_prohd.txt 2>&1
