timeout 300 python tools/dbg_perrow.py > gpurun_out/r02f_dbg.log 2>&1
