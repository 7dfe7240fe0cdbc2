mkdir -p gpurun_out
timeout 1500 python tools/ab_k2.py nc4 nc3 nc2 nc1 > gpurun_out/ab_k2_r02p.txt 2>&1; tail -6 gpurun_out/ab_k2_r02p.txt
