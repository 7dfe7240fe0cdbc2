"""Throughput of the fused advance on every pure-ODE BASELINE config at its
per-GPU size (single GPU): config 0 full; config 1 full; configs 2 and 4 on
their per-GPU shard (2^24 points = config 2 on 1 GPU, config 4 / 8 GPUs) for a
window of steps.  Prints one JSON line per config."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="0,1,2,4")
ap.add_argument("--window", type=int, default=0, help="steps per config (0 = preset)")
ap.add_argument("--full", action="store_true", help="the config's whole step count")
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
preset = {0: (4096, 20000, 0), 1: (1 << 20, 10000, 0), 2: (1 << 24, 5000, 0),
          4: (1 << 24, 5000, 0)}
for c in [int(x) for x in a.configs.split(",")]:
    n, steps, step0 = preset[c]
    if a.n:
        n = a.n
    if a.window:
        steps = a.window
    if a.full:
        steps = {0: 20000, 1: 10000, 2: 50000, 4: 100000}[c] - 200
    src = pkg.source_for_config(c)
    f = pkg.init_from_source(src, n)
    # warm (first 200 steps), then time the window
    pkg.advance(f, 200, src, snapshot_every=1000)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pkg.advance(f, steps, src, step0=200, snapshot_every=1000)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"config": c, "points": n, "steps": steps, "ms": ms,
                      "point_updates_per_s": n * steps / (ms * 1e-3)}), flush=True)
