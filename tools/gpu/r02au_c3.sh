mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullscale.py -m gpu -x -q -k "coupled or config3 or slab or split" > gpurun_out/pytest_c3.log 2>&1; tail -4 gpurun_out/pytest_c3.log
timeout 600 python tools/config3_job.py --steps 6000 > gpurun_out/c3_overlap.txt 2>&1; tail -4 gpurun_out/c3_overlap.txt
