set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20
python tools/window_rates.py --config 4 --n 2097152 > gpurun_out/win4.json 2> gpurun_out/win4.err
python tools/window_rates.py --config 2 --n 2097152 > gpurun_out/win2.json 2>> gpurun_out/win4.err
python tools/prof_advance.py --config 4 --n 1048576 --pre 50000 --steps 2000 --reps 2 > gpurun_out/adv4.plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_adv_cfg4_r02a -f \
  python tools/prof_advance.py --config 4 --n 1048576 --pre 50000 --steps 2000 --reps 2 > gpurun_out/ncu_adv4.log 2>&1
ls -la gpurun_out
