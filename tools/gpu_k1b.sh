# K1 group-allocation sweep (PROHD_K1_BETA) + per-CTA DMMA view of the default
mkdir -p gpurun_out
for b in 0 4 8 16 1000 0; do PROHD_K1_BETA=$b timeout 200 python tools/time_moments.py 5 >> gpurun_out/k1b.log 2>&1; done
for b in 0 8; do PROHD_K1_BETA=$b timeout 200 python tools/time_moments.py 4 >> gpurun_out/k1b.log 2>&1; done
timeout 600 ncu --clock-control none -k regex:gram_kernel --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.max.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.min.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_sector_hit_rate.pct python tools/prof_prohd.py 5 > gpurun_out/k1b_ncu.log 2>&1
