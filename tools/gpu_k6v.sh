V=${V:-2a}
PROHD_K6_VARIANT=$V timeout 900 python -m pytest tests/test_gpu_exact.py -x -q > gpurun_out/pytest_k6v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k6v.log
PROHD_K6_VARIANT=$V timeout 600 python tools/time_exact.py > gpurun_out/time_k6v.txt 2>&1
