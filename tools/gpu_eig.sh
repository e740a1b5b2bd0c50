mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eigen.py tests/test_gpu_prohd.py -x -q > gpurun_out/pytest_eig.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_eig.log
for st in 1 2 3 0; do PROHD_EIG_STOP=$st timeout 120 python tools/time_eigen.py; done > gpurun_out/time_eig.txt 2>&1
timeout 300 python tools/time_prohd.py 5 4 3 2 > gpurun_out/time_eig2.txt 2>&1
