# HEAD full run: GPU tests, both bench arms (driver flags), smoke, bench launch list, ncu of the window launch
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu_r02aw.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02aw.log
tail -12 gpurun_out/pytest_gpu_r02aw.log
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/b_ref_r02aw.json 2> gpurun_out/b_ref_r02aw.err
tail -3 gpurun_out/b_ref_r02aw.err
mkdir -p gpurun_out/numba_cache && cp -r baseline/_ref/.numba_cache/. gpurun_out/numba_cache/
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/b_r02aw.json 2> gpurun_out/b_r02aw.err
tail -12 gpurun_out/b_r02aw.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02aw.log 2>&1; tail -2 gpurun_out/smoke_r02aw.log
timeout 900 python bench.py --steps 2 --warmup 1 --quick --no-cpu-baseline > gpurun_out/b_quick_r02aw.json 2> gpurun_out/b_quick_r02aw.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/r02aw_bench_launches.csv python bench.py --steps 2 --warmup 1 --quick --no-cpu-baseline > gpurun_out/ncu_bench_r02aw.log 2>&1
tail -2 gpurun_out/ncu_bench_r02aw.log
timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw_r02aw.log 2>&1
cat gpurun_out/pbw_r02aw.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 101 -c 1 -o gpurun_out/prof_r02aw_cfg4_window -f python tools/prof_bench_window.py --windows 1 > gpurun_out/ncu_pbw_r02aw.log 2>&1
tail -3 gpurun_out/ncu_pbw_r02aw.log
ls -la gpurun_out/*.ncu-rep
