mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 900 python tools/ab_k2.py cur > gpurun_out/ab_k2_r02o.txt 2>&1; tail -3 gpurun_out/ab_k2_r02o.txt
timeout 900 python -m pytest tests/test_gpu_fullscale.py -q -x -k "config4 or config2 or large" 2>&1 | tail -3
