mkdir -p gpurun_out
for v in 1 2 3; do timeout 120 python tools/time_project.py >> gpurun_out/k3d.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_prohd.py -m gpu -q -x > gpurun_out/k3d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k3d_pytest.log
