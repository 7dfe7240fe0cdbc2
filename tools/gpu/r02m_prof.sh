mkdir -p gpurun_out
timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw.plain.log 2>&1
cat gpurun_out/pbw.plain.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 5 -c 1 -o gpurun_out/prof_r02_cfg4_window -f python tools/prof_bench_window.py --windows 1 > gpurun_out/ncu_pbw.log 2>&1
tail -3 gpurun_out/ncu_pbw.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:run_range_vec --launch-skip 1 -c 1 -o gpurun_out/prof_r02_k1vec -f python tools/bench_hbm.py > gpurun_out/ncu_k1.log 2>&1
tail -3 gpurun_out/ncu_k1.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 2 --warmup 1 --quick --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/ncu_bench.log
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
