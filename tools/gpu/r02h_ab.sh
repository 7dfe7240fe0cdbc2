mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stencil.py -q -x 2>&1 | tail -5
timeout 1200 python tools/ab_k2.py base new new_mb6 > gpurun_out/ab_k2_r02h.txt 2>&1
tail -5 gpurun_out/ab_k2_r02h.txt
