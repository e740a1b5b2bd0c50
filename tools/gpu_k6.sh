mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exact.py tests/test_gpu_prohd.py -x -q > gpurun_out/pytest_k6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k6.log
timeout 600 python tools/time_exact.py > gpurun_out/time_k6.txt 2>&1
