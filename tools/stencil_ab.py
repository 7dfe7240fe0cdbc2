"""Helper for tests/test_gpu_stencil.py: run K4 and the fused coupled step on
an odd-sized grid and save the results (the pipeline is chosen by TI64_NO_TMA,
the coupled-step mode by the second argument: split (default) or fused)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
from paper_2402_17580_b200 import scanpath, thermal as th  # noqa: E402

nz, ny, nx, h, dt = 21, 37, 64, 20e-6, 1e-6
src = th.HeatSource(w_eff=87.5, radius=50e-6, h_powder=h)
segs = scanpath.serpentine((0.2e-3, 0.2e-3, 1.0e-3, 0.6e-3), 80e-6, 1.0, 87.5)
beams = scanpath.beam_schedule(segs, 300, dt)
a = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h)
split = len(sys.argv) < 3 or sys.argv[2] != "fused"
a.run(300, dt, beams, src, fused=True, split=split)
b = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h)
b.field.temperature_old.copy_(a.field.temperature_old)
for k in range(5):
    th.step_thermal(b.field, dt, th.DEFAULT_THERMAL, src, beams[k], losses=False,
                    bottom_dirichlet=353.0, all_built=True)
    b.field.temperature_old.copy_(b.field.temperature_new)
h1 = a.fields.to_host()
np.savez(sys.argv[1], stencil=b.field.temperature_new.cpu().numpy(),
         coupled_T=a.field.temperature_old.cpu().numpy(), **h1)
