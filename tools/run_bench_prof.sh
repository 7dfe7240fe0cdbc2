set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo bench=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 1 -c 1 -o gpurun_out/r01b_adv_cfg1_job -f \
  python tools/prof_advance.py --steps 10000 --snap 1000 --reps 2 > gpurun_out/ncu_job.log 2>&1; echo job=$?
