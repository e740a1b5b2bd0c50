ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv -k regex:"colmax|colsum|slice|gram_i8" python tools/prof_prohd.py 5 > gpurun_out/i8_launch.csv 2>&1
R=/tmp/ncu_i8; mkdir -p $R
timeout 600 ncu --set full --clock-control none --import-source on -f -o $R/i8 -k regex:"gram_i8_kernel|slice_kernel" -c 2 python tools/prof_prohd.py 5 > gpurun_out/i8_prof.log 2>&1
ncu -i $R/i8.ncu-rep --page details > gpurun_out/i8_details.txt 2>&1
ncu -i $R/i8.ncu-rep --page source --csv > gpurun_out/i8_source.csv 2>&1
