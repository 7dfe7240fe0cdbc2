mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" > gpurun_out/pytest_host.log 2>&1; tail -5 gpurun_out/pytest_host.log
timeout 900 python tools/e2e_chunks.py > gpurun_out/e2e_chunks.txt 2>&1; cat gpurun_out/e2e_chunks.txt
