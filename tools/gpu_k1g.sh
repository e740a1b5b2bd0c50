# K1 column sums inside the Gram launch (D >= 224): timings per config (cs = 7 default vs others)
mkdir -p gpurun_out
for c in 5 4; do timeout 200 python tools/time_moments.py $c >> gpurun_out/k1g.log 2>&1; done
for v in 0 8; do PROHD_K1_CS_SMS=$v timeout 200 python tools/time_moments.py 4 | sed "s/^/cs=$v /" >> gpurun_out/k1g.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_prohd.py -m gpu -q -x > gpurun_out/k1g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k1g_pytest.log
