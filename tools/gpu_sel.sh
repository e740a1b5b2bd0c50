mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_prohd.py tests/test_gpu_shard.py tests/test_gpu_next.py tests/test_gpu_select.py -x -q > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sel.log
timeout 300 python tools/time_prohd.py 5 4 3 2 > gpurun_out/time_sel.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"radix|collect|rank|compact|cand" python tools/prof_prohd.py 5 > gpurun_out/sel_launch.csv 2>&1
