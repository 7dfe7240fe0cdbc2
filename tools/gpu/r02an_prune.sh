mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_initiation.py tests/test_gpu_acceptance.py -m gpu -x -q > gpurun_out/pytest_prune.log 2>&1; tail -3 gpurun_out/pytest_prune.log
timeout 1800 python tools/ab_k2.py prune prune2 > gpurun_out/ab_k2_prune.txt 2>&1; tail -3 gpurun_out/ab_k2_prune.txt
timeout 600 python tools/prof_bench_window.py --windows 2 > gpurun_out/pbw_prune.log 2>&1; cat gpurun_out/pbw_prune.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"classify|residue|task_sums" --launch-skip 404 -c 10 --csv --log-file gpurun_out/prune_cls.csv python tools/prof_bench_window.py --windows 1 > /dev/null 2>&1; grep -o '"[a-z_:<>A-Z0-9 ,()]*kernel[^"]*".*' gpurun_out/prune_cls.csv | awk -F'","' '{print $1, $NF}' | tail -10
