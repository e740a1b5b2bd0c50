PROHD_K6_VARIANT=2sm timeout 600 python tools/time_exact.py > gpurun_out/time_k6_2sm.txt 2>&1
PROHD_K6_VARIANT=2sm timeout 900 python -m pytest tests/test_gpu_exact.py -x -q > gpurun_out/pytest_k6_2sm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k6_2sm.log
