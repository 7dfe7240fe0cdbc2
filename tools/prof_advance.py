"""Profiling driver: one warm + one measured launch of the fused advance
kernel on a BASELINE config (default 1), for ncu.  Usage:
    python tools/prof_advance.py [--config 1] [--steps 1000] [--n N]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--steps", type=int, default=1000)
ap.add_argument("--step0", type=int, default=0)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--pre", type=int, default=0, help="untimed steps before the measured launches")
ap.add_argument("--snap", type=int, default=0, help="snapshot_every of the measured launches")
a = ap.parse_args()
src = pkg.source_for_config(a.config)
n = a.n or (src.n_points if a.config == 1 else {0: 4096, 2: 1 << 24, 4: 1 << 24}[a.config])
f0 = pkg.init_from_source(src, n)
if a.step0:
    from paper_2402_17580_b200.batch import gen_temperature
    f0.temperature_old.copy_(gen_temperature(src, n, a.step0))
if a.pre:
    pkg.advance(f0, a.pre, src, step0=a.step0)
    a.step0 += a.pre
for r in range(a.reps):
    f = f0.copy()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pkg.advance(f, a.steps, src, step0=a.step0, snapshot_every=a.snap)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"rep {r}: {a.steps} steps x {n} points: {ms:.3f} ms, "
          f"{n * a.steps / ms / 1e6:.3f} G upd/s", flush=True)
