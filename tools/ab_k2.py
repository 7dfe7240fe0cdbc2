"""A/B of fused-advance (K2) library variants: per variant (a subprocess
with TI64_VARIANT_LIB), the config-4 window (2^21 shard, 600 steps from step
20000), the config-2 window (2^22, 600 steps from 10000), the config-1 job
and config 0; prints ms and a digest of the final states (must agree
across variants: every variant is bit-exact).
    python tools/ab_k2.py VARIANT [VARIANT ...]   (names under _lib/variants)"""
import hashlib
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r'''
import hashlib, json, sys
sys.path.insert(0, "tools")
import _variant  # noqa
import torch
import paper_2402_17580_b200 as pkg
out = {}
for cfg, n, s0, steps, reps in ((4, 1 << 21, 20000, 600, 3), (2, 1 << 22, 10000, 600, 3),
                                 (1, 1 << 20, 0, 10000, 3), (0, 4096, 0, 20000, 2)):
    src = pkg.source_for_config(cfg)
    f0 = pkg.init_from_source(src, n)
    if s0:
        pkg.advance(f0, s0, src)
    ts = []
    for r in range(reps):
        f = f0.copy()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pkg.advance(f, steps, src, step0=s0, snapshot_every=steps)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    h = hashlib.sha256()
    for k in pkg.batch.NAMES:
        t = getattr(f, k)
        if k == "seed_tracked":
            t = torch.where(f.seed_active != 0, t, torch.zeros_like(t))
        h.update(t.cpu().numpy().tobytes())
    out[f"cfg{cfg}"] = {"ms": min(ts), "upd_per_s": n * steps / min(ts) * 1e3,
                        "digest": h.hexdigest()[:16]}
print(json.dumps(out))
'''

res = {}
for rep in range(2):
    for v in sys.argv[1:]:
        env = dict(os.environ, TI64_VARIANT_LIB=str(ROOT / "paper_2402_17580_b200" / "_lib" /
                                                    "variants" / f"lib_{v}.so"))
        p = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env,
                           capture_output=True, text=True)
        if p.returncode:
            print(v, "FAILED", p.stderr[-2000:], flush=True)
            continue
        d = json.loads(p.stdout.strip().splitlines()[-1])
        print(v, rep, json.dumps(d), flush=True)
        for c, x in d.items():
            r = res.setdefault(v, {}).setdefault(c, x)
            r["ms"] = min(r["ms"], x["ms"])
            if r["digest"] != x["digest"]:
                r["digest"] = "NONDETERMINISTIC"
print("== summary (best of reps)")
names = sorted({c for v in res.values() for c in v})
for v, d in res.items():
    print(v.ljust(14), "  ".join(f"{c}: {d[c]['ms']:9.2f} ms {d[c]['digest'][:8]}" for c in names))
