timeout 300 python tools/time_prohd.py 5 4 3 2 > gpurun_out/time_sel.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"radix|collect|rank|compact|cand" python tools/prof_prohd.py 5 > gpurun_out/sel_launch.csv 2>&1
