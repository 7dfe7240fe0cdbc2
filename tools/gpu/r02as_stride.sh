mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_initiation.py -m gpu -x -q > gpurun_out/pytest_st.log 2>&1; tail -3 gpurun_out/pytest_st.log
timeout 1800 python tools/ab_k2.py st1 st4 st8 st16 > gpurun_out/ab_k2_st.txt 2>&1; tail -5 gpurun_out/ab_k2_st.txt
for v in st1 st4 st8 st16; do TI64_VARIANT_LIB=$PWD/paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 600 python tools/prof_bench_window.py --windows 2 2>&1 | tail -1; done > gpurun_out/pbw_st.log; cat gpurun_out/pbw_st.log
