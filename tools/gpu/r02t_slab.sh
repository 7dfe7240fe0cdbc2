mkdir -p gpurun_out
timeout 600 python tools/config3_slab_time.py > gpurun_out/slab_time.json 2> gpurun_out/slab_time.err; cat gpurun_out/slab_time.json; tail -3 gpurun_out/slab_time.err
