mkdir -p gpurun_out
stat -c '%Y %s %n' baseline/_ref/ti64micro/batch.py > gpurun_out/stat_box.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
