#!/bin/bash
# Round profiling pass (run under gpurun): each command first runs without ncu
# and must exit 0; then one ncu capture.  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
run() { local name=$1; shift; "$@" > gpurun_out/$name.plain.log 2>&1 || { echo "$name: plain run failed"; return 1; }; }
run bench python bench.py --steps 2 --warmup 1 --no-cpu-baseline && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
      > gpurun_out/ncu_launches.log 2>&1
run stencil python tools/prof_stencil.py && \
  ncu --set full --import-source on --clock-control none -k regex:built_tma_kernel \
      --launch-skip 21 -c 4 -o gpurun_out/prof_stencil -f python tools/prof_stencil.py \
      > gpurun_out/ncu_stencil.log 2>&1
run k1 python tools/k1_probe.py && \
  ncu --set full --import-source on --clock-control none -k regex:run_range_kernel \
      --launch-skip 1 -c 1 -o gpurun_out/prof_k1 -f python tools/k1_probe.py \
      > gpurun_out/ncu_k1.log 2>&1
run cn python tools/cn_probe.py && \
  ncu --set full --import-source on --clock-control none -k regex:run_range_cn \
      --launch-skip 1 -c 1 -o gpurun_out/prof_cn -f python tools/cn_probe.py \
      > gpurun_out/ncu_cn.log 2>&1
run adv1 python tools/prof_advance.py --steps 10000 --snap 1000 --reps 1 && \
  ncu --set full --import-source on --clock-control none -k regex:advance_kernel \
      -c 1 -o gpurun_out/prof_adv_cfg1 -f \
      python tools/prof_advance.py --steps 10000 --snap 1000 --reps 1 > gpurun_out/ncu_adv1.log 2>&1
run adv2 python tools/prof_advance.py --config 2 --n 4194304 --pre 200 --reps 1 && \
  ncu --set full --import-source on --clock-control none -k regex:advance_kernel \
      --launch-skip 1 -c 1 -o gpurun_out/prof_adv_cfg2 -f \
      python tools/prof_advance.py --config 2 --n 4194304 --pre 200 --reps 1 \
      > gpurun_out/ncu_adv2.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches.csv
