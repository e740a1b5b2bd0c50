mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_moments.py -x -q > gpurun_out/pytest_k1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k1.log
timeout 300 python tools/time_prohd.py 5 4 > gpurun_out/time_k1.txt 2>&1
