ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv python tools/prof_prohd.py 5 > gpurun_out/prohd_launch.csv 2>&1
PROHD_K3_SCALAR=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:project --csv python tools/prof_prohd.py 5 > gpurun_out/prohd_launch_scalar.csv 2>&1
