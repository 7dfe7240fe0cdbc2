"""Config-3 determinism: the fused coupled run (512x512x256, 3000 steps) twice
from the same start, every state array compared bit for bit."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg
from paper_2402_17580_b200 import scanpath, thermal as th
dev = torch.device("cuda", 0)
res = []
for r in range(2):
    dom = th.CoupledDomain(nx=512, ny=512, nz=256, h=20e-6, device=dev)
    src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=20e-6)
    segs = scanpath.serpentine((1e-3, 1e-3, 9.24e-3, 9.24e-3), 80e-6, 1.0, 0.35 * 250.0)
    beams = scanpath.beam_schedule(segs, 3000, 1e-6)
    dom.run(3000, 1e-6, beams, src, fused=True)
    torch.cuda.synchronize()
    res.append({k: getattr(dom.fields, k).cpu().numpy().copy() for k in ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old", "seed_active")})
    del dom
for k in res[0]:
    print(k, np.array_equal(res[0][k].view(np.uint8), res[1][k].view(np.uint8)))
