#!/bin/bash
# Profiling pass (run only after bench.py exits 0 without ncu): launch list of the bench
# command, then ncu --set full captures of the ProHD kernels and of K6, exported to text on
# the box (the .ncu-rep files are too large to bring back whole).
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01b}
if [ -z "$SKIP_LAUNCH" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/${TAG}_launch_bench.log 2>&1; echo "launch rc=$?"
fi
R=/tmp/ncu_${TAG}; mkdir -p $R
timeout 900 ncu --set full --clock-control none --import-source on -f -o $R/prohd \
  python tools/prof_prohd.py ${PROHD_CFG:-5} > gpurun_out/${TAG}_prohd.log 2>&1; echo "prohd rc=$?"
ncu -i $R/prohd.ncu-rep --page raw --csv > gpurun_out/${TAG}_prohd_raw.csv 2>&1
ncu -i $R/prohd.ncu-rep --page details > gpurun_out/${TAG}_prohd_details.txt 2>&1
if [ -z "$SKIP_K6" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -f -o $R/k6 \
  -k regex:dist_rowmin python tools/prof_k6.py > gpurun_out/${TAG}_k6.log 2>&1; echo "k6 rc=$?"
ncu -i $R/k6.ncu-rep --page raw --csv > gpurun_out/${TAG}_k6_raw.csv 2>&1
ncu -i $R/k6.ncu-rep --page details > gpurun_out/${TAG}_k6_details.txt 2>&1
fi
ls -la gpurun_out
