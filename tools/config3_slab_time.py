"""Config-3 step times: the whole-grid CoupledDomain vs SlabCoupledGPU at
world size 1 (the slab-form split step), and, for a 32-plane block (one
rank's slab at 8 GPUs), the directly launched step loop vs the replayed
CUDA graph.  Prints one JSON line."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
from paper_2402_17580_b200 import scanpath, thermal as th  # noqa: E402
from paper_2402_17580_b200.distributed import SlabCoupledGPU  # noqa: E402

h, dt = 20e-6, 1e-6
src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=h)
segs = scanpath.serpentine((1e-3, 1e-3, 9.24e-3, 9.24e-3), 80e-6, 1.0, 0.35 * 250.0)
steps = 2000
beams = scanpath.beam_schedule(segs, 2 * steps + 1, dt)


def per_step(run, n):
    run(1, 0)  # warm-up / first-step initialisation
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run(n, 1)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n


out = {}
nz, ny, nx = 256, 512, 512
d = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h)
out["whole_grid_ms"] = per_step(lambda n, k0: d.run(n, dt, beams[k0:], src), steps)
del d
s = SlabCoupledGPU(nz, ny, nx, h)
out["slab_world1_ms"] = per_step(lambda n, k0: s.run(n, dt, beams[k0:], src), steps)
del s
for nzs in (32,):
    d = th.CoupledDomain(nx=nx, ny=ny, nz=nzs, h=h)
    out[f"nz{nzs}_direct_ms"] = per_step(lambda n, k0: d.run(n, dt, beams[k0:], src), steps)
    d2 = th.CoupledDomain(nx=nx, ny=ny, nz=nzs, h=h)
    out[f"nz{nzs}_graph_ms"] = per_step(
        lambda n, k0: d2.run(n, dt, beams[k0:], src, graph=n >= 3), steps)
print(json.dumps(out))
