mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r01g_bench.json 2> gpurun_out/r01g_bench.err; echo "bench rc=$?" >> gpurun_out/r01g_bench.err
TAG=r01g bash tools/gpu_profile.sh > gpurun_out/r01g_profile.log 2>&1
