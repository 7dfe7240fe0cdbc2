mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_initiation.py -m gpu -x -q > gpurun_out/pytest_scr.log 2>&1; tail -3 gpurun_out/pytest_scr.log
timeout 1800 python tools/ab_k2.py base scr > gpurun_out/ab_k2_scr.txt 2>&1; tail -3 gpurun_out/ab_k2_scr.txt
timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw_scr.log 2>&1; cat gpurun_out/pbw_scr.log
