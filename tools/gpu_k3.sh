mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_select.py -x -q -s > gpurun_out/pytest_k3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k3.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"project" python tools/prof_prohd.py 5 > gpurun_out/proj_launch.csv 2>&1
timeout 300 python tools/time_prohd.py 5 4 > gpurun_out/time_k3.txt 2>&1
