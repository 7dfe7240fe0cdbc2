mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_gpu_r02j.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02j.log
tail -15 gpurun_out/pytest_gpu_r02j.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/b_ref_r02j.json 2> gpurun_out/b_ref_r02j.err
tail -3 gpurun_out/b_ref_r02j.err
mkdir -p gpurun_out/numba_cache && cp -r baseline/_ref/.numba_cache/. gpurun_out/numba_cache/
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/b_r02j.json 2> gpurun_out/b_r02j.err
tail -12 gpurun_out/b_r02j.err
