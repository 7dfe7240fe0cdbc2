mkdir -p gpurun_out
for v in lean nolean; do
  export TI64_VARIANT_LIB=$PWD/paper_2402_17580_b200/_lib/variants/lib_$v.so
  timeout 600 python tools/prof_advance.py --config 4 --n 8388608 --pre 20000 --steps 200 --snap 200 > gpurun_out/pa_$v.log 2>&1; tail -2 gpurun_out/pa_$v.log
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 100 -c 1 -o gpurun_out/prof_$v -f python tools/prof_advance.py --config 4 --n 8388608 --pre 20000 --steps 200 --snap 200 --reps 1 > gpurun_out/ncu_$v.log 2>&1; tail -2 gpurun_out/ncu_$v.log
done
