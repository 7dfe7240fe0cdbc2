"""Profiling driver for the bench headline: config 4 at N points (default
2^27) prepared to step 20 000 in 5000-step launches (4 advance launches),
one warm-up window (advance launch 101: launches cover at most 200 steps), then `--windows` timed 200-step windows (the
bench's K2 launches).  For ncu: -k regex:advance_kernel --launch-skip 101 -c 1
captures the first bench window launch."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 27)
ap.add_argument("--windows", type=int, default=2)
ap.add_argument("--window", type=int, default=200, help="steps per timed window")
a = ap.parse_args()
src = pkg.source_for_config(4)
f = pkg.init_from_source(src, a.n)
scr = pkg.batch._scratch(a.n, f.device)
s = 0
while s < 20000:
    pkg.advance(f, 5000, src, step0=s, scratch=scr)
    s += 5000
pkg.advance(f, 200, src, step0=s, snapshot_every=200, scratch=scr)
s += 200
W = a.window
for w in range(a.windows):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pkg.advance(f, W, src, step0=s, snapshot_every=W, scratch=scr)
    e1.record()
    e1.synchronize()
    s += W
    print(f"window {w}: steps {s - W}-{s}: {e0.elapsed_time(e1):.2f} ms "
          f"({a.n * W / e0.elapsed_time(e1) / 1e6:.3f} G upd/s)", flush=True)
