mkdir -p gpurun_out
timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw2.plain.log 2>&1
cat gpurun_out/pbw2.plain.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 5 -c 1 -o gpurun_out/prof_r02b_cfg4_window -f python tools/prof_bench_window.py --windows 1 > gpurun_out/ncu_pbw2.log 2>&1
tail -2 gpurun_out/ncu_pbw2.log
ls -la gpurun_out/*.ncu-rep
