mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_build.py -q -x 2>&1 | tail -5
