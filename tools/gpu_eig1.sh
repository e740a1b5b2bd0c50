mkdir -p gpurun_out
PROHD_EIG_STOP=1 timeout 200 python tools/time_eigen.py > gpurun_out/eig1.log 2>&1
timeout 200 python tools/time_eigen.py >> gpurun_out/eig1.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_prohd.py tests/test_gpu_shard.py -m gpu -q -x > gpurun_out/eig1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/eig1_pytest.log
timeout 600 python tools/report_configs.py 2 3 5 > gpurun_out/eig1_configs.md 2>&1
