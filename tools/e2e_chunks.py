"""End-to-end window time of the headline (config 4, N points prepared to
step 20 000) with the state in pinned host memory, for several staged chunk
sizes of ti64_advance_host and for the zero-copy access (-1), next to the
device-resident window.  Each e2e window starts from the same host state and
is timed on the host (perf_counter around advance + sums read-back + sync)."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 27)
ap.add_argument("--chunks", type=int, nargs="*", default=[1 << 21, 1 << 22, 1 << 23, 1 << 24, -1])
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
NAMES = pkg.batch.NAMES
src = pkg.source_for_config(4)
f = pkg.init_from_source(src, a.n)
scr = pkg.batch._scratch(a.n, f.device)
s = 0
while s < 20000:
    pkg.advance(f, 5000, src, step0=s, scratch=scr)
    s += 5000
start = f.copy()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
pkg.advance(f, 200, src, step0=s, snapshot_every=200, scratch=scr)
for k in NAMES:
    getattr(f, k).copy_(getattr(start, k))
e0.record()
r = pkg.advance(f, 200, src, step0=s, snapshot_every=200, scratch=scr)
e1.record()
e1.synchronize()
print(f"device-resident window: {e0.elapsed_time(e1):.2f} ms", flush=True)
host = {k: torch.empty(getattr(f, k).shape, dtype=getattr(f, k).dtype, pin_memory=True)
        for k in NAMES}
for hc in a.chunks:
    for rep in range(a.reps):
        for k in NAMES:
            host[k].copy_(getattr(start, k))
        torch.cuda.synchronize()
        c0 = time.perf_counter()
        fh = pkg.GlobalFields(*[host[k] for k in NAMES], device="host")
        rh = pkg.advance(fh, 200, src, step0=s, snapshot_every=200, host_chunk_points=hc)
        sums = rh.sums.cpu()
        torch.cuda.synchronize()
        dt = time.perf_counter() - c0
        same = all(torch.equal(host[k], getattr(f, k).cpu()) for k in NAMES)
        print(f"chunk {hc:>9}: rep {rep}: {1e3 * dt:.2f} ms ({a.n * 200 / dt / 1e9:.3f} G upd/s) "
              f"bitwise_equal_to_device={same}", flush=True)
