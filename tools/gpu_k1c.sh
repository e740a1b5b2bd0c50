mkdir -p gpurun_out
for c in 5 4 3 2 5; do timeout 200 python tools/time_moments.py $c >> gpurun_out/k1c.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_prohd.py -m gpu -q -x > gpurun_out/k1c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k1c_pytest.log
timeout 600 ncu --clock-control none -k regex:gram_kernel --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active python tools/prof_prohd.py 5 > gpurun_out/k1c_ncu.log 2>&1
