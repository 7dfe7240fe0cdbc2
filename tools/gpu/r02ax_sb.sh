mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_initiation.py -m gpu -x -q > gpurun_out/pytest_sb.log 2>&1; tail -3 gpurun_out/pytest_sb.log
timeout 1800 python tools/ab_k2.py sb1 sb2 sb3 > gpurun_out/ab_k2_sb.txt 2>&1; tail -4 gpurun_out/ab_k2_sb.txt
for v in sb1 sb2 sb3; do TI64_VARIANT_LIB=$PWD/paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 600 python tools/prof_bench_window.py --windows 2 2>&1 | tail -1; done > gpurun_out/pbw_sb.log; cat gpurun_out/pbw_sb.log
