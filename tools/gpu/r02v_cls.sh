mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 1500 python tools/ab_k2.py c4 c6 > gpurun_out/ab_k2_r02v.txt 2>&1; tail -4 gpurun_out/ab_k2_r02v.txt
for v in c4 c6; do TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 600 python tools/prof_bench_window.py --windows 2 2>/dev/null | tail -1; done
