"""Debug helper: config-0 advance in chunks of C steps vs the oracle loop;
prints, per chunk size, the first step where any point differs."""
import sys
sys.path.insert(0, "tools")
import _variant  # noqa
import numpy as np
import torch
import paper_2402_17580_b200 as pkg
from oracle import oracle as orc

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 0
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
total = int(sys.argv[3]) if len(sys.argv) > 3 else 4000
src = pkg.source_for_config(cfg_id)
kp = pkg.DEFAULT_PARAMS.kernel_tuple()
cfg = pkg.IntegratorConfig().kernel_tuple()
g = src.tempgen(point_offset=0)
for chunk in (1, 7, 100, total):
    f = pkg.init_from_source(src, n)
    h = orc.gen_initial_state(g, n)
    h.temperature_old[:] = orc.gen_temperature(g, n, 0)
    h.temperature_new[:] = h.temperature_old
    bad = None
    for s0 in range(0, total, chunk):
        k = min(chunk, total - s0)
        pkg.advance(f, k, src, step0=s0)
        orc.advance(h, g, s0, k, kp, cfg, lanes=8)
        got = f.to_host()
        for name in ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old"):
            a = got[name].view(np.int64)
            b = getattr(h, name).view(np.int64)
            if not np.array_equal(a, b):
                i = int(np.flatnonzero(a != b)[0])
                bad = (s0 + k, name, i, got[name][i], getattr(h, name)[i],
                       int((a != b).sum()))
                break
        if bad:
            break
    print(f"chunk {chunk}: first mismatch {bad}", flush=True)
    if bad:
        i = bad[2]
        print("  point", i, {k2: got[k2][i] for k2 in pkg.batch.NAMES},
              {k2: getattr(h, k2)[i] for k2 in pkg.batch.NAMES}, flush=True)
