mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 1500 python tools/ab_k2.py noreord reord > gpurun_out/ab_k2_r02u.txt 2>&1; tail -4 gpurun_out/ab_k2_r02u.txt
