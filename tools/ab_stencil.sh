#!/bin/bash
# interleaved A/B of stencil/coupled timings across library variants
for rep in 1 2 3; do
  for v in "$@"; do
    TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so python tools/bench_hbm.py 2>/dev/null | python -c "
import sys,json
out=[]
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    if d['kernel'] in ('K4 stencil_built','fused coupled step'): out.append(round(d['s']*1e6,1))
print('$v', *out)"
  done
done
