mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 1500 python tools/ab_k2.py c6 c7 > gpurun_out/ab_k2_r02w.txt 2>&1; tail -3 gpurun_out/ab_k2_r02w.txt
for v in c6 c7; do TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 600 python tools/prof_bench_window.py --windows 2 2>/dev/null | tail -1; done
for v in c7 c7r500; do TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 600 python tools/window_rates.py --config 4 --n 2097152 --window 5000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['job_ms'], d['job_rate'])"; done
