#!/bin/bash
# interleaved A/B of the implicit step_all (block-100 layout, 2^22 points)
for rep in 1 2; do
  for v in "$@"; do
    TI64_VARIANT_LIB=paper_2402_17580_b200/_lib/variants/lib_$v.so python - <<PY
import torch, bench
import sys; sys.path.insert(0, "tools"); import _variant  # noqa
import paper_2402_17580_b200 as pkg
dev = torch.device("cuda", 0)
cfg = pkg.IntegratorConfig(scheme="crank_nicolson", dt_sub_max=0.01)
out = []
for blk in (1, 100):
    p = pkg.GlobalFields(*bench.branch_layout(blk, 1 << 22), device=dev)
    ts = []
    for r in range(6):
        w = p.copy()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); pkg.step_all(w, 0.01, config=cfg, n_lanes=8); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    out.append(round(sorted(ts[1:])[2], 3))
print("$v", "CN ms (block 1, 100):", out)
PY
  done
done
