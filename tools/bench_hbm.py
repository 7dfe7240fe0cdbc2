"""HBM-bound kernels at config-3 size (512 x 512 x 256 = 2^26 cells):
K1 step_all (73 B/point-update model) and K4 built stencil (16 B/cell), plus
one coupled step (stencil + step_all).  Prints JSON lines with GB/s."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402
from paper_2402_17580_b200 import thermal as th, scanpath  # noqa: E402

nz, ny, nx = 256, 512, 512
n = nz * ny * nx
dom = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=20e-6)
src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=20e-6)
segs = scanpath.serpentine((1e-3, 1e-3, 9.24e-3, 9.24e-3), 80e-6, 1.0, 0.35 * 250.0)
beams = scanpath.beam_schedule(segs, 200, 1e-6)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


dom.run(5, 1e-6, beams, src)  # warm + heat a little
f = dom.fields
t = timed(lambda: pkg.step_all(f, 1e-6))
print(json.dumps({"kernel": "K1 run_range (step_all)", "cells": n, "s": t,
                  "model_bytes": 73 * n, "GB/s": 73 * n / t / 1e9,
                  "point_updates_per_s": n / t}))
k = [0]


def stencil():
    th.step_thermal(dom.field, 1e-6, th.DEFAULT_THERMAL, src, beams[k[0] % 200], losses=False,
                    bottom_dirichlet=353.0, all_built=True)
    k[0] += 1


t = timed(stencil)
print(json.dumps({"kernel": "K4 stencil_built", "cells": n, "s": t, "model_bytes": 16 * n,
                  "GB/s": 16 * n / t / 1e9, "cell_updates_per_s": n / t}))
t = timed(lambda: dom.run(1, 1e-6, beams[k[0] % 200:], src), reps=10)
print(json.dumps({"kernel": "coupled step (K4 + K1)", "cells": n, "s": t,
                  "model_bytes": (16 + 73) * n, "GB/s": 89 * n / t / 1e9,
                  "cell_steps_per_s": n / t}))
dom2 = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=20e-6)
dom2.run(5, 1e-6, beams, src, fused=True)
t = timed(lambda: dom2.run(10, 1e-6, beams[k[0] % 150:], src, fused=True), reps=5) / 10
print(json.dumps({"kernel": "fused coupled step", "cells": n, "s": t,
                  "stencil_bytes": 16 * n, "GB/s_stencil_model": 16 * n / t / 1e9,
                  "cell_steps_per_s": n / t}))
if "--job" in sys.argv:
    steps = 20000
    segs3 = scanpath.serpentine((1e-3, 1e-3, 9.24e-3, 9.24e-3), 80e-6, 1.0, 0.35 * 250.0)
    b3 = scanpath.beam_schedule(segs3, steps, 1e-6)
    dom3 = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=20e-6)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dom3.run(steps, 1e-6, b3, src, fused=True)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3
    h = dom3.fields.to_host()
    print(json.dumps({"job": "config 3 full (512x512x256, 20000 steps)", "s": s,
                      "cell_steps_per_s": n * steps / s,
                      "T_max": float(h["temperature_old"].max()),
                      "mean_xs": float(h["x_alpha_s"].mean()),
                      "mean_xm": float(h["x_alpha_m"].mean())}))
