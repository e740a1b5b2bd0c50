for c in 5 3 2; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"gram|colsum|shift|finalize|covariance" python tools/prof_prohd.py $c > gpurun_out/k1_launch_cfg$c.csv 2>&1
done
