set -x
R=/tmp/ncu_eig; mkdir -p $R gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -f -o $R/eig -k regex:"eigen_" python tools/eig_once.py > gpurun_out/eig_prof.log 2>&1
ncu -i $R/eig.ncu-rep --page details > gpurun_out/eig_details.txt 2>&1
ncu -i $R/eig.ncu-rep --page raw --csv > gpurun_out/eig_raw.csv 2>&1
ncu -i $R/eig.ncu-rep --page source --csv > gpurun_out/eig_source.csv 2>&1
