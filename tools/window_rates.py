"""Per-window throughput over a whole pure-ODE job on one shard (to choose
the bench's measurement window and relate it to the whole-job rate).
Usage: python tools/window_rates.py [--config 4] [--n 2097152] [--window 1000]"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--n", type=int, default=1 << 21)
ap.add_argument("--window", type=int, default=1000)
ap.add_argument("--steps", type=int, default=0)
a = ap.parse_args()
src = pkg.source_for_config(a.config)
total = a.steps or {0: 20000, 1: 10000, 2: 50000, 4: 100000}[a.config]
f = pkg.init_from_source(src, a.n)
scratch = pkg.batch._scratch(a.n, f.device)
rates = []
tot_ms = 0.0
for s0 in range(0, total, a.window):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pkg.advance(f, a.window, src, step0=s0, scratch=scratch)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    tot_ms += ms
    rates.append(a.n * a.window / ms * 1e3)
print(json.dumps({"config": a.config, "n": a.n, "window": a.window, "job_steps": total,
                  "job_ms": tot_ms, "job_rate": a.n * total / tot_ms * 1e3,
                  "window_rates": rates}))
