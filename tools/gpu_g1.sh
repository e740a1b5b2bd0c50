mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/time_prohd.py 5 4 > gpurun_out/time_row.txt 2>&1
PROHD_K3_TILE=1 timeout 300 python tools/time_prohd.py 5 4 > gpurun_out/time_tile.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"project" python tools/time_prohd.py 5 > gpurun_out/proj_launch.csv 2>&1
