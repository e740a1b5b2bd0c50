mkdir -p gpurun_out
timeout 900 python tools/report_configs.py 3 4 > gpurun_out/k6b_configs.md 2>&1
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_next.py tests/test_gpu_prohd.py -m gpu -q -x > gpurun_out/k6b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k6b_pytest.log
