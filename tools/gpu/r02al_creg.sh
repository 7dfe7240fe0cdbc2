mkdir -p gpurun_out
timeout 1800 python tools/ab_k2.py look2 creg5 creg4 creg3 > gpurun_out/ab_k2_creg.txt 2>&1; tail -5 gpurun_out/ab_k2_creg.txt
for v in look2 creg4; do TI64_VARIANT_LIB=$PWD/paper_2402_17580_b200/_lib/variants/lib_$v.so python tools/cold_only_probe.py --windows 3 2>&1 | tail -1; done
