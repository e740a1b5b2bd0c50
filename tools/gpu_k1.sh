mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_moments.py -x -q > gpurun_out/pytest_k1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k1.log
timeout 300 python tools/time_prohd.py 5 4 3 2 > gpurun_out/time_k1.txt 2>&1
for c in 5 3 2; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"gram|colsum|shift|finalize|covariance" python tools/prof_prohd.py $c > gpurun_out/k1_launch_cfg$c.csv 2>&1
done
