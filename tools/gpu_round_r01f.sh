mkdir -p gpurun_out
TAG=r01f bash tools/gpu_profile.sh > gpurun_out/r01f_profile.log 2>&1
timeout 1200 python tools/report_configs.py > gpurun_out/report_configs.md 2> gpurun_out/report_configs.err
