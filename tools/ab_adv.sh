#!/bin/bash
# interleaved A/B of the fused advance across library variants: config-1 job
# (bench --quick) and the config 2/4 2^22-point shards
for rep in 1 2; do
  for v in "$@"; do
    TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so python - <<PY
import json, subprocess, sys, torch
import sys; sys.path.insert(0, "tools"); import _variant  # noqa
import paper_2402_17580_b200 as pkg
dev = torch.device("cuda", 0)
out = []
for c in (2, 4):
    src = pkg.source_for_config(c)
    f = pkg.init_from_source(src, 1 << 22, device=dev)
    pkg.advance(f, 200, src, snapshot_every=1000)
    g = f.copy()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); pkg.advance(g, 2000, src, step0=200, snapshot_every=1000); e1.record(); e1.synchronize()
    out.append(round((1 << 22) * 2000 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2))
r = subprocess.run([sys.executable, "bench.py", "--quick", "--no-cpu-baseline", "--steps", "5"],
                   capture_output=True, text=True)
d = json.loads(r.stdout.strip().splitlines()[-1])
print("$v", "cfg1 ms/job", round(d["ms_per_step"], 2), "cfg2/4 G upd/s", out)
PY
  done
done
