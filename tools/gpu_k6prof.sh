mkdir -p gpurun_out
R=/tmp/ncu_r01i; mkdir -p $R
timeout 600 ncu --set full --clock-control none --import-source on -f -o $R/k6 -k regex:dist_rowmin python tools/prof_k6.py > gpurun_out/r01i_k6.log 2>&1; echo "k6 rc=$?"
ncu -i $R/k6.ncu-rep --page raw --csv > gpurun_out/r01i_k6_raw.csv 2>&1
ncu -i $R/k6.ncu-rep --page details > gpurun_out/r01i_k6_details.txt 2>&1
