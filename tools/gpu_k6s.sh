mkdir -p gpurun_out
PROHD_K6_SPLITS=2x timeout 900 python tools/report_configs.py 2 3 4 5 > gpurun_out/k6s_old.md 2>&1
timeout 900 python tools/report_configs.py 2 3 4 5 > gpurun_out/k6s_new.md 2>&1
timeout 1200 python -m pytest tests/test_gpu_exact.py tests/test_gpu_prohd.py tests/test_gpu_next.py -m gpu -q -x > gpurun_out/k6s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k6s_pytest.log
