mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_next.py -x -q > gpurun_out/pytest_next.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_next.log
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_next.py -x -q -k "rc4" > gpurun_out/sanitize_rc4.log 2>&1
