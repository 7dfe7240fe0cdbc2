#!/bin/bash
# ncu source-level captures of the fused advance (K2): config-1 job (one
# launch = the bench's job) and config 4 mid-job (all points active).
# Each command first runs without ncu.  Usage: tools/prof_k2.sh TAG
set -u
tag=${1:-k2}
mkdir -p gpurun_out
python tools/prof_advance.py --steps 10000 --snap 1000 --reps 2 > gpurun_out/${tag}_c1.plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 1 -c 1 -o gpurun_out/${tag}_c1 -f \
  python tools/prof_advance.py --steps 10000 --snap 1000 --reps 2 > gpurun_out/${tag}_c1.ncu.log 2>&1
python tools/prof_advance.py --config 4 --n 1048576 --pre 50000 --steps 2000 --reps 2 > gpurun_out/${tag}_c4.plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 2 -c 1 -o gpurun_out/${tag}_c4 -f \
  python tools/prof_advance.py --config 4 --n 1048576 --pre 50000 --steps 2000 --reps 2 > gpurun_out/${tag}_c4.ncu.log 2>&1
ls -la gpurun_out/${tag}_*.ncu-rep
