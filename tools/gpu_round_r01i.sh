mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01i_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01i_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r01i_smoke.log
timeout 900 python bench.py > gpurun_out/r01i_bench.json 2> gpurun_out/r01i_bench.err; echo "bench rc=$?" >> gpurun_out/r01i_bench.err
timeout 600 python tools/report_configs.py > gpurun_out/r01i_configs.md 2> gpurun_out/r01i_configs.err
SKIP_K6=1 TAG=r01i bash tools/gpu_profile.sh > gpurun_out/r01i_profile.log 2>&1
