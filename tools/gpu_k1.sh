# K1 (diagonal-tile skip, load-balanced groups) and K3 (6 TMA boxes + 4 xl tiles) check:
# parity of moments / selection / ProHD, K3 ring A/B, per-config timings
mkdir -p gpurun_out
for r in 8 6 8 6; do PROHD_K3_RING=$r timeout 120 python tools/time_project.py >> gpurun_out/k3_ring.log 2>&1; echo "ring=$r" >> gpurun_out/k3_ring.log; done
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_select.py tests/test_gpu_prohd.py -m gpu -q -x > gpurun_out/k1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k1_pytest.log
timeout 600 python tools/report_configs.py 2 3 4 5 > gpurun_out/k1_configs.md 2> gpurun_out/k1_configs.err
