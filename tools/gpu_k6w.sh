# K6 warp-wide elected MMA issue: sustained bench (clock) + exact parity
mkdir -p gpurun_out
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/k6w_$i.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/k6w_$i.json')); print('run $i', round(d['value'],1), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],4), round(d['prohd_ms'],2))" >> gpurun_out/k6w.log; done
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_next.py -m gpu -q -x > gpurun_out/k6w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k6w_pytest.log
timeout 600 python tools/report_configs.py 2 3 4 > gpurun_out/k6w_configs.md 2>&1
