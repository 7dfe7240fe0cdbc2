"""Config 0 at full size (4096 points x 20 000 steps, one launch): ms per job."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402
src = pkg.source_for_config(0)
f0 = pkg.init_from_source(src, 4096)
best = 1e9
for r in range(4):
    f = f0.copy()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); pkg.advance(f, 20000, src, snapshot_every=1000); e1.record(); e1.synchronize()
    if r:
        best = min(best, e0.elapsed_time(e1))
print(f"config0 job {best:.3f} ms")
