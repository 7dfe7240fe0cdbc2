mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stencil.py -q -x 2>&1 | tail -40 > gpurun_out/parity_r02e.log
cat gpurun_out/parity_r02e.log
