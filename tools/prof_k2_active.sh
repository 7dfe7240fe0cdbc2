set -u
mkdir -p gpurun_out
python tools/prof_advance.py --config 2 --n 4194304 --step0 10000 --pre 200 --steps 2000 --reps 2 > gpurun_out/adv2.plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_adv_cfg2b -f \
  python tools/prof_advance.py --config 2 --n 4194304 --step0 10000 --pre 200 --steps 2000 --reps 2 > gpurun_out/ncu_adv2.log 2>&1
python tools/prof_advance.py --config 4 --n 1048576 --pre 50000 --steps 2000 --reps 2 > gpurun_out/adv4.plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_adv_cfg4 -f \
  python tools/prof_advance.py --config 4 --n 1048576 --pre 50000 --steps 2000 --reps 2 > gpurun_out/ncu_adv4.log 2>&1
ls -la gpurun_out/*.ncu-rep
