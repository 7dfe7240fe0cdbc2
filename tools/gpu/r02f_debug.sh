mkdir -p gpurun_out
timeout 600 python tools/debug_k2.py 0 4096 20000 > gpurun_out/debug_k2.log 2>&1
cat gpurun_out/debug_k2.log
