# Round profiling refresh (run under gpurun): full bench line, launch list of the
# bench, ncu --set full of the headline K2 launch and of the K4 stencil.  Each
# command first runs without ncu and must exit 0.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo bench=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --quick > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01c.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --quick > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
python tools/prof_advance.py --steps 10000 --snap 1000 --reps 2 > gpurun_out/job.plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 1 -c 1 -o gpurun_out/r01c_adv_cfg1_job -f \
  python tools/prof_advance.py --steps 10000 --snap 1000 --reps 2 > gpurun_out/ncu_job.log 2>&1; echo job=$?
python tools/prof_stencil.py > gpurun_out/stencil.plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:built_tma_kernel \
      --launch-skip 21 -c 4 -o gpurun_out/r01c_stencil -f python tools/prof_stencil.py > gpurun_out/ncu_stencil.log 2>&1; echo stencil=$?
