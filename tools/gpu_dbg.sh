mkdir -p gpurun_out
timeout 600 python tools/dbg_iter2.py > gpurun_out/dbg_iter2.log 2>&1
cat gpurun_out/dbg_iter2.log
