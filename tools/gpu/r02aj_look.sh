mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_initiation.py -m gpu -x -q > gpurun_out/pytest_look.log 2>&1; tail -5 gpurun_out/pytest_look.log
timeout 1200 python tools/ab_k2.py nolook look > gpurun_out/ab_k2_look.txt 2>&1; tail -4 gpurun_out/ab_k2_look.txt
timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw_look.log 2>&1; cat gpurun_out/pbw_look.log
