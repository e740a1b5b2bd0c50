mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prohd.py tests/test_gpu_exact.py -x -q > gpurun_out/pytest_k2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k2.log
for st in 1 2 3 0; do PROHD_EIG_STOP=$st timeout 120 python tools/time_eigen.py; done > gpurun_out/time_eig.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"shift" python tools/prof_prohd.py 5 > gpurun_out/shift_launch.csv 2>&1
timeout 300 python tools/time_prohd.py 5 4 > gpurun_out/time_k2.txt 2>&1
