import sys, ctypes as C
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import _variant
import torch
import paper_2402_17580_b200 as pkg
from paper_2402_17580_b200 import _lib
lib = _lib.require()
n = 1 << 24
src = pkg.source_for_config(4)
f = pkg.init_from_source(src, n)
s = 0
while s < 20000:
    pkg.advance(f, 5000, src, step0=s); s += 5000
pkg.advance(f, 200, src, step0=s, snapshot_every=200); s += 200
buf = (C.c_ulonglong * 8)()
torch.cuda.synchronize()
lib.ti64_path_times(buf)
pkg.advance(f, 200, src, step0=s, snapshot_every=200)
torch.cuda.synchronize()
lib.ti64_path_times(buf)
v = list(buf)
tot = sum(v[:6])
names = ["init", "rest(all idle)", "cold loop", "generic: seeding warp", "generic: hot lane", "generic: other", "cold steps", "seed-warp steps"]
for k, x in zip(names, v):
    print(f"{k:24s} {x:16d} {100*x/tot if k not in ('cold steps','seed-warp steps') else 0:6.2f}%")
print("warp-updates", n * 200 // 32)
