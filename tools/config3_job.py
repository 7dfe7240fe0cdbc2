"""The whole config-3 job on one GPU: 512x512x256 cells, 20 000 coupled steps
(stencil + kinetics of every cell, fused kernel), dt = 1e-6 s, serpentine 1 m/s
80 um hatch, 250 W x 0.35.  Times every 1000-step chunk (the transformed trail
behind the beam grows over the job, and with it the kinetics work), then the
whole job.  python tools/config3_job.py [--steps 20000]"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402
from paper_2402_17580_b200 import scanpath, thermal as th  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20000)
ap.add_argument("--chunk", type=int, default=1000)
a = ap.parse_args()
dev = torch.device("cuda", 0)
nx, ny, nz = 512, 512, 256
dom = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=20e-6, device=dev)
src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=20e-6)
segs = scanpath.serpentine((1e-3, 1e-3, 9.24e-3, 9.24e-3), 80e-6, 1.0, 0.35 * 250.0)
beams = scanpath.beam_schedule(segs, a.steps, 1e-6)
chunks = []
k = 0
e_all0 = torch.cuda.Event(enable_timing=True)
e_all1 = torch.cuda.Event(enable_timing=True)
e_all0.record()
while k < a.steps:
    m = min(a.chunk, a.steps - k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dom.run(m, 1e-6, beams[k:k + m], src, fused=True)
    e1.record()
    e1.synchronize()
    chunks.append(round(e0.elapsed_time(e1) / m * 1e3, 1))
    k += m
e_all1.record()
e_all1.synchronize()
s = e_all0.elapsed_time(e_all1) * 1e-3
f = dom.fields
sums = pkg.phase_sums(f).cpu().numpy() / (nx * ny * nz)
Tmax = float(dom.field.temperature_old.max().item()) if hasattr(dom, "field") else None
print(json.dumps({"config": 3, "cells": nx * ny * nz, "steps": a.steps, "job_s": s,
                  "cell_steps_per_s": nx * ny * nz * a.steps / s,
                  "us_per_step_by_chunk": chunks, "mean_fractions": sums.tolist(),
                  "T_max": Tmax}), flush=True)
