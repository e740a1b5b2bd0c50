mkdir -p gpurun_out
PROHD_K3_RAWHI=1 timeout 600 python -m pytest tests/test_gpu_select.py -x -q -s -k "configs or variants" > gpurun_out/pytest_k3raw.log 2>&1
PROHD_K3_RAWHI=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"project" python tools/prof_prohd.py 5 > gpurun_out/proj_launch_raw.csv 2>&1
R=/tmp/ncu_k3; mkdir -p $R
timeout 600 ncu --set full --clock-control none --import-source on -f -o $R/k3 -k regex:"project_tc" -c 1 python tools/prof_prohd.py 5 > gpurun_out/k3_prof.log 2>&1
ncu -i $R/k3.ncu-rep --page details > gpurun_out/k3_details.txt 2>&1
ncu -i $R/k3.ncu-rep --page raw --csv > gpurun_out/k3_raw.csv 2>&1
ncu -i $R/k3.ncu-rep --page source --csv > gpurun_out/k3_source.csv 2>&1
