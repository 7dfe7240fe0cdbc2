"""Single-warp step latency of the fused advance: one 32-point task run alone
on the GPU (no co-resident warps), so the time per step is the latency of one
step's dependency chain.  python tools/step_latency.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402
from paper_2402_17580_b200.batch import gen_temperature  # noqa: E402

dev = torch.device("cuda", 0)
for c, s0, pre in ((2, 0, 0), (2, 10000, 10000), (4, 50000, 50000)):
    src = pkg.source_for_config(c)
    for n in (32, 148 * 32 * 4):
        f = pkg.init_from_source(src, n, device=dev)
        if pre:
            pkg.advance(f, pre, src)
        steps = 2000
        best = 1e9
        for r in range(3):
            g = f.copy()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); pkg.advance(g, steps, src, step0=s0); e1.record(); e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"config {c} steps {s0}-{s0 + steps} n={n}: {best * 1e6 / steps:8.1f} ns per step "
              f"({best * 1e6 / steps * 1.965:7.0f} cycles at 1965 MHz)", flush=True)
