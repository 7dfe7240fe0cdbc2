# A/B of the split coupled step's stencil instance across library variants (config-3 job
# chunks and an ncu launch-time list). Usage: tools/ab_split_k4.sh A B ...
for rep in 1 2; do for v in "$@"; do
TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so timeout 120 python tools/config3_job.py --steps 2000 > gpurun_out/k4ab_$v.json 2>&1
echo $v $(python -c "import json;d=json.loads(open('gpurun_out/k4ab_$v.json').read().strip().splitlines()[-1]);print(d['us_per_step_by_chunk'])")
done; done
for v in "$@"; do TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"built_tma" --launch-skip 1500 -c 3 --csv --log-file gpurun_out/k4ab_$v.csv python tools/config3_job.py --steps 2000 > /dev/null 2>&1; echo $v $(grep duration gpurun_out/k4ab_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '); done
