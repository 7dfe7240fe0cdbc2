mkdir -p gpurun_out
for v in base k1scalar k1p1 k1p4; do echo "== $v"; TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 300 python tools/bench_hbm.py 2>&1 | head -1; done > gpurun_out/ab_k1_r02k.txt
cat gpurun_out/ab_k1_r02k.txt
timeout 1500 python tools/ab_k2.py base creg_mb6 creg_mb5 creg_mb4 creg_mb3 > gpurun_out/ab_k2_r02k.txt 2>&1
tail -7 gpurun_out/ab_k2_r02k.txt
