"""Probe for ncu: a few explicit step_all calls (K1) on 2^26 points."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402

n = 1 << 26
rng = np.random.default_rng(0)
xs = rng.uniform(0.0, 0.9, n)
f = pkg.GlobalFields(xs, np.zeros(n), 1.0 - xs, rng.uniform(300, 1500, n), rng.uniform(300, 1500, n))
for _ in range(3):
    pkg.step_all(f, 2e-5)
torch.cuda.synchronize()
print("ok")
