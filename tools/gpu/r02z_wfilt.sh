mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_initiation.py -m gpu -x -q > gpurun_out/pytest_wfilt.log 2>&1; tail -3 gpurun_out/pytest_wfilt.log
timeout 1200 python tools/ab_k2.py head wfilt > gpurun_out/ab_k2_wfilt.txt 2>&1; tail -4 gpurun_out/ab_k2_wfilt.txt
timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw_wfilt.log 2>&1; cat gpurun_out/pbw_wfilt.log
