import sys
sys.path.insert(0, "tools")
import _variant  # noqa
import numpy as np
import paper_2402_17580_b200 as pkg
from oracle import oracle as orc
src = pkg.source_for_config(0)
n, P = 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 466
kp = pkg.DEFAULT_PARAMS.kernel_tuple()
cfg = pkg.IntegratorConfig().kernel_tuple()
g = src.tempgen(point_offset=0)
f = pkg.init_from_source(src, n)
h = orc.gen_initial_state(g, n)
h.temperature_old[:] = orc.gen_temperature(g, n, 0)
h.temperature_new[:] = h.temperature_old
pkg.advance(f, 1990, src, step0=0)
orc.advance(h, g, 0, 1990, kp, cfg, lanes=8)
for s in range(1990, 2025):
    pkg.advance(f, 1, src, step0=s)
    orc.advance(h, g, s, 1, kp, cfg, lanes=8)
    got = f.to_host()
    row = lambda d, get: " ".join(f"{k[:6]}={get(d, k)!r}" for k in
                                  ("x_alpha_s", "x_beta", "temperature_old", "seed_tracked",
                                   "seed_active", "seed_direction"))
    print(s + 1, "GPU", row(got, lambda d, k: d[k][P]))
    print(s + 1, "ORC", row(h, lambda d, k: getattr(d, k)[P]))
