R=/tmp/ncu_k6; mkdir -p $R gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -f -o $R/k6 -k regex:dist_rowmin -c 1 python tools/prof_k6.py > gpurun_out/k6m_prof.log 2>&1
ncu -i $R/k6.ncu-rep --page details > gpurun_out/k6m_details.txt 2>&1
ncu -i $R/k6.ncu-rep --page raw --csv > gpurun_out/k6m_raw.csv 2>&1
ncu -i $R/k6.ncu-rep --page source --csv > gpurun_out/k6m_source.csv 2>&1
