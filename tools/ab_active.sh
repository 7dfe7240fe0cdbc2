#!/bin/bash
# interleaved A/B of the fused advance on the ALL-ACTIVE workloads: config 2
# (2^22 shard, steps 10000-12000, every point transforming every step) and
# config 4 (2^20 shard, steps 50000-52000 from the state after 50000 steps),
# plus the config-1 job (bench --quick).  Usage: tools/ab_active.sh A B ...
for rep in 1 2; do
  for v in "$@"; do
    TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so python - <<PY
import json, subprocess, sys, torch
import sys; sys.path.insert(0, "tools"); import _variant  # noqa
import paper_2402_17580_b200 as pkg
from paper_2402_17580_b200.batch import gen_temperature
dev = torch.device("cuda", 0)
out = []
for c, n, s0, pre in ((2, 1 << 22, 10000, 0), (4, 1 << 20, 50000, 50000)):
    src = pkg.source_for_config(c)
    f = pkg.init_from_source(src, n, device=dev)
    if pre:
        pkg.advance(f, pre, src, step0=0)
    else:
        f.temperature_old.copy_(gen_temperature(src, n, s0))
    best = 0.0
    for r in range(3):
        g = f.copy()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); pkg.advance(g, 2000, src, step0=s0); e1.record(); e1.synchronize()
        best = max(best, n * 2000 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    out.append(round(best, 2))
r = subprocess.run([sys.executable, "bench.py", "--quick", "--no-cpu-baseline", "--steps", "5"],
                   capture_output=True, text=True)
d = json.loads(r.stdout.strip().splitlines()[-1])
print("$v", "cfg1 ms/job", round(d["ms_per_step"], 2), "cfg2/cfg4 active G upd/s", out, flush=True)
PY
  done
done
# single-task step latency of config 1 (the 32 surface points 0..31 alone)
for v in "$@"; do
  echo -n "$v cfg1 single task: "
  TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so python tools/prof_advance.py --config 1 --n 32 --steps 10000 --reps 3 | tail -1
done
