mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_prohd.py tests/test_gpu_next.py tests/test_gpu_fullsize.py tests/test_gpu_select.py -x -q > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sel.log
timeout 300 python tools/time_prohd.py 5 4 3 2 > gpurun_out/time_sel.txt 2>&1
