"""Probe: the cold loop's step rate when every warp stays in it.  Config-4
generator with peaks U(100, 600) K (T never reaches T_alpha_s,end) on points
that all start transformed (0.5, 0.2, 0.3), so every point fires its rate
branches at every step and no seed or hot path runs.  Used to compare the
product kernel with code-footprint experiments (TI64_VARIANT_LIB)."""
import argparse
import dataclasses
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 23)
ap.add_argument("--windows", type=int, default=4)
ap.add_argument("--amp", type=float, nargs=2, default=[100.0, 600.0])
a = ap.parse_args()
src = dataclasses.replace(pkg.source_for_config(4), amp=tuple(a.amp))
f = pkg.init_from_source(src, a.n)
f.x_alpha_s.fill_(0.5)
f.x_alpha_m.fill_(0.2)
f.x_beta.fill_(0.3)
s = 20000
f.temperature_old.copy_(pkg.batch.gen_temperature(src, a.n, s))
for w in range(a.windows):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pkg.advance(f, 200, src, step0=s, snapshot_every=200)
    e1.record()
    e1.synchronize()
    s += 200
    ms = e0.elapsed_time(e1)
    print(f"window {w}: {ms:.2f} ms ({a.n * 200 / ms / 1e6:.3f} G upd/s) "
          f"sums {[round(float(x), 6) for x in pkg.phase_sums(f).cpu()]}", flush=True)
