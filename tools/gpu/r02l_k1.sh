mkdir -p gpurun_out
for rep in 1 2; do for v in base k1scalar k1p1 k1p4; do echo "== $v"; TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 300 python tools/bench_hbm.py 2>/dev/null | head -1; done; done > gpurun_out/ab_k1_r02l.txt
cat gpurun_out/ab_k1_r02l.txt
