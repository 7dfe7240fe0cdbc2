mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu_r02s.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02s.log
tail -12 gpurun_out/pytest_gpu_r02s.log
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/b_ref_r02s.json 2> gpurun_out/b_ref_r02s.err
tail -3 gpurun_out/b_ref_r02s.err
mkdir -p gpurun_out/numba_cache && cp -r baseline/_ref/.numba_cache/. gpurun_out/numba_cache/
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/b_r02s.json 2> gpurun_out/b_r02s.err
tail -12 gpurun_out/b_r02s.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02s.log 2>&1; tail -2 gpurun_out/smoke_r02s.log
