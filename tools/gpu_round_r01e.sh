mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python tools/time_prohd.py 5 4 3 2 > gpurun_out/time_prohd.txt 2>&1
TAG=r01e bash tools/gpu_profile.sh > gpurun_out/r01e_profile.log 2>&1
