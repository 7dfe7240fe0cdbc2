mkdir -p gpurun_out
timeout 1200 python tools/ab_k2.py r500 r1000 > gpurun_out/ab_k2_r02x.txt 2>&1; tail -3 gpurun_out/ab_k2_r02x.txt
for v in r200 r300 r500 r1000; do TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 600 python tools/window_rates.py --config 4 --n 2097152 --window 5000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 job 2^21 $v', d['job_ms'], d['job_rate'])"; done
for v in r300 r1000; do TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 600 python tools/window_rates.py --config 2 --n 4194304 --window 5000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 job 2^22 $v', d['job_ms'], d['job_rate'])"; done
