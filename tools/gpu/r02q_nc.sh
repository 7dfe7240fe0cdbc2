mkdir -p gpurun_out
timeout 1500 python tools/ab_k2.py nc5 nc6 nc8 nc12 > gpurun_out/ab_k2_r02q.txt 2>&1; tail -6 gpurun_out/ab_k2_r02q.txt
