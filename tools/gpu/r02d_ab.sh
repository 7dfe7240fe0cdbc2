mkdir -p gpurun_out
timeout 1200 python tools/ab_k2.py base new new_mb6 new_mb4 > gpurun_out/ab_k2_r02d.txt 2>&1
cat gpurun_out/ab_k2_r02d.txt | tail -8
