"""Break down the e2e (host-buffer) path of bench.py into its parts."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402

src = pkg.source_for_config(1)
n = src.n_points
dev = torch.device("cuda", 0)
pristine = pkg.init_from_source(src, n, device=dev)
host = {k: torch.from_numpy(pristine.host(k)).pin_memory() for k in pkg.batch.NAMES}
scratch = pkg.batch._scratch(n, dev)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = pkg.GlobalFields(*[host[k] for k in pkg.batch.NAMES], device=dev)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pkg.advance(f, 10000, src, snapshot_every=1000, scratch=scratch)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st = f.states()
    t3 = time.perf_counter()
    print(f"h2d+fields {1e3*(t1-t0):.2f} ms  advance {1e3*(t2-t1):.2f} ms  d2h {1e3*(t3-t2):.2f} ms")
