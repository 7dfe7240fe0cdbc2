mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_initiation.py -m gpu -x -q > gpurun_out/pytest_look2.log 2>&1; tail -3 gpurun_out/pytest_look2.log
timeout 1800 python tools/ab_k2.py look look2 look2_100 look2_400 > gpurun_out/ab_k2_look2.txt 2>&1; tail -5 gpurun_out/ab_k2_look2.txt
timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw_look2.log 2>&1; cat gpurun_out/pbw_look2.log
TI64_VARIANT_LIB=$PWD/paper_2402_17580_b200/_lib/variants/lib_look2_100.so timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw_look2_100.log 2>&1; cat gpurun_out/pbw_look2_100.log
