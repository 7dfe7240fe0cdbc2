set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 1 --quick > gpurun_out/b_quick.json 2> gpurun_out/b_quick.err
tail -5 gpurun_out/b_quick.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
tail -5 gpurun_out/b_ref.err
mkdir -p gpurun_out/numba_cache && cp -r baseline/_ref/.numba_cache/* gpurun_out/numba_cache/ 2>/dev/null
ls gpurun_out/numba_cache | head
