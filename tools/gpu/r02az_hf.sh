mkdir -p gpurun_out
timeout 1800 python tools/ab_k2.py hf0 hf1 > gpurun_out/ab_k2_hf.txt 2>&1; tail -3 gpurun_out/ab_k2_hf.txt
for v in hf0 hf1; do TI64_VARIANT_LIB=$PWD/paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 600 python tools/prof_bench_window.py --windows 2 2>&1 | tail -1; done > gpurun_out/pbw_hf.log; cat gpurun_out/pbw_hf.log
