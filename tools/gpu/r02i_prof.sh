mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil.py -q -x 2>&1 | tail -5
export TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_base.so
python tools/prof_advance.py --config 4 --n 2097152 --pre 20000 --steps 600 --reps 2 > gpurun_out/adv4w.plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_cfg4_win_base -f \
  python tools/prof_advance.py --config 4 --n 2097152 --pre 20000 --steps 600 --reps 2 > gpurun_out/ncu_adv4w.log 2>&1
export TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_new.so
ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_cfg4_win_new -f \
  python tools/prof_advance.py --config 4 --n 2097152 --pre 20000 --steps 600 --reps 2 > gpurun_out/ncu_adv4w_new.log 2>&1
ls -la gpurun_out/*.ncu-rep
