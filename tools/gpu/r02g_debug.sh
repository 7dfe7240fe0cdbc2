mkdir -p gpurun_out
timeout 600 python tools/debug_k2b.py 466 > gpurun_out/debug_k2b.log 2>&1
cat gpurun_out/debug_k2b.log
