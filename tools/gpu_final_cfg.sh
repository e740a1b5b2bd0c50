bash tools/gpu_final.sh
timeout 600 python tools/report_configs.py > gpurun_out/configs.md 2> gpurun_out/configs.err
