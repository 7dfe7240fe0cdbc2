"""Probe: a few implicit step_all calls on the benchmark layouts (for ncu)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import bench  # noqa: E402
import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402

dev = torch.device("cuda", 0)
cfg = pkg.IntegratorConfig(scheme="crank_nicolson", dt_sub_max=0.01)
for block in (1, 100):
    f = pkg.GlobalFields(*bench.branch_layout(block, 1 << 22), device=dev)
    for _ in range(2):
        pkg.step_all(f.copy(), 0.01, config=cfg, n_lanes=8)
torch.cuda.synchronize()
print("ok")
