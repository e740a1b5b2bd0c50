mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_moments.py -x -q > gpurun_out/pytest_mom.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mom.log
