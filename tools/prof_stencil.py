"""ncu driver: the built stencil and the fused coupled step at config-3 size."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
from paper_2402_17580_b200 import thermal as th, scanpath  # noqa: E402

nz, ny, nx = 256, 512, 512
dom = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=20e-6)
src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=20e-6)
segs = scanpath.serpentine((1e-3, 1e-3, 9.24e-3, 9.24e-3), 80e-6, 1.0, 0.35 * 250.0)
beams = scanpath.beam_schedule(segs, 50, 1e-6)
dom.run(20, 1e-6, beams, src, fused=True)
for k in range(3):
    th.step_thermal(dom.field, 1e-6, th.DEFAULT_THERMAL, src, beams[k], losses=False,
                    bottom_dirichlet=353.0, all_built=True)
dom.run(3, 1e-6, beams[20:], src, fused=True)
torch.cuda.synchronize()
print("ok")
