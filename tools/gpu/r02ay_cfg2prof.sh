mkdir -p gpurun_out
timeout 600 python tools/prof_advance.py --config 2 --n 16777216 --pre 10200 --steps 200 --snap 200 > gpurun_out/pa_cfg2.log 2>&1; tail -2 gpurun_out/pa_cfg2.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 51 -c 1 -o gpurun_out/prof_r02ay_cfg2_window -f python tools/prof_advance.py --config 2 --n 16777216 --pre 10200 --steps 200 --snap 200 --reps 1 > gpurun_out/ncu_cfg2.log 2>&1; tail -2 gpurun_out/ncu_cfg2.log
