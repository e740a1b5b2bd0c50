set -x
R=/tmp/ncu_k1; mkdir -p $R gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -f -o $R/k1 -k regex:"gram_kernel|moments_kernel" python tools/prof_prohd.py 5 > gpurun_out/k1_prof.log 2>&1
ncu -i $R/k1.ncu-rep --page details > gpurun_out/k1_details.txt 2>&1
ncu -i $R/k1.ncu-rep --page raw --csv > gpurun_out/k1_raw.csv 2>&1
ncu -i $R/k1.ncu-rep --page source --csv > gpurun_out/k1_source.csv 2>&1
ls -la gpurun_out/k1*
