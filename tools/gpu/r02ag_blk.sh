mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_initiation.py tests/test_gpu_acceptance.py -m gpu -x -q > gpurun_out/pytest_blk.log 2>&1; tail -5 gpurun_out/pytest_blk.log
timeout 1200 python tools/ab_k2.py noblk blk > gpurun_out/ab_k2_blk.txt 2>&1; tail -4 gpurun_out/ab_k2_blk.txt
timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw_blk.log 2>&1; cat gpurun_out/pbw_blk.log
