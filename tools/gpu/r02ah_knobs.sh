mkdir -p gpurun_out
timeout 2400 python tools/ab_k2.py blk minb6 minb7 retry1 retry16 > gpurun_out/ab_k2_knobs.txt 2>&1; tail -7 gpurun_out/ab_k2_knobs.txt
