mkdir -p gpurun_out
timeout 1200 python tools/ab_k2.py lean call callnolean > gpurun_out/ab_k2_call.txt 2>&1; tail -5 gpurun_out/ab_k2_call.txt
export TI64_VARIANT_LIB=$PWD/paper_2402_17580_b200/_lib/variants/lib_call.so
timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw_call.log 2>&1; cat gpurun_out/pbw_call.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 100 -c 1 -o gpurun_out/prof_call -f python tools/prof_advance.py --config 4 --n 8388608 --pre 20000 --steps 200 --snap 200 --reps 1 > gpurun_out/ncu_call.log 2>&1; tail -2 gpurun_out/ncu_call.log
