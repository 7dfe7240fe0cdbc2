"""Per-task timing of the fused advance (diagnostic): needs the variant built
with  python tools/build_variant.py tt -DADV_TASK_TIMES=1  and
TI64_LIB=paper_2402_17580_b200/_lib/variants/lib_tt.so.
Prints the distribution of 32-point task durations of one config-1 job and the
job's timeline (how many tasks are running over time)."""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_17580_b200 as pkg  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
src = pkg.source_for_config(cfg)
n = src.n_points if cfg == 1 else 1 << 20
steps = 10000 if cfg == 1 else 2000
f0 = pkg.init_from_source(src, n)
pkg.advance(f0.copy(), steps, src, snapshot_every=1000)
pkg.advance(f0.copy(), steps, src, snapshot_every=1000)
torch.cuda.synchronize()
lib = ctypes.CDLL(os.environ["TI64_LIB"])
ntask = (n + 31) // 32
buf = (ctypes.c_ulonglong * (8 * ntask))()
assert lib.ti64_debug_task_times(buf, ctypes.c_int64(ntask)) == 0
raw = np.frombuffer(buf, dtype=np.uint64)
t = raw[:2 * ntask].reshape(-1, 2).astype(np.int64)
cs = raw[2 * ntask:4 * ntask].view(np.uint32).reshape(-1, 4).astype(np.int64)
ph = raw[4 * ntask:8 * ntask].reshape(-1, 4).astype(np.int64)
t0 = t[:, 0].min()
st, en = (t[:, 0] - t0) / 1e6, (t[:, 1] - t0) / 1e6
dur = en - st
print(f"job span {en.max():.3f} ms; tasks {ntask}; total task-ms {dur.sum():.1f}")
q = np.percentile(dur, [50, 90, 99, 99.9, 100])
print("task duration ms p50/p90/p99/p99.9/max:", np.round(q, 4))
order = np.argsort(-dur)[:10]
for k in order:
    print(f"  task {k:6d} (layer {k * 32 // 16384:2d}) start {st[k]:7.3f} end {en[k]:7.3f} dur {dur[k]:7.3f}"
          f"  warp-steps computed {cs[k, 0]}, lane-steps base {cs[k, 1]} off-base {cs[k, 2]} skipped {cs[k, 3]}"
          f"  -> {dur[k] * 1e6 / max(cs[k, 0], 1):.0f} ns per computed warp-step; cycles per computed step:"
          f" T/screens {ph[k, 0] / max(cs[k, 0], 1):.0f} update {ph[k, 1] / max(cs[k, 0], 1):.0f}"
          f" tail {ph[k, 2] / max(cs[k, 0], 1):.0f}")
heavy = dur > 5.0
print(f"heavy tasks (>5 ms): {heavy.sum()}, mean computed warp-steps {cs[heavy, 0].mean():.0f}, "
      f"lane-steps base {cs[heavy, 1].mean():.0f} off {cs[heavy, 2].mean():.0f} skip {cs[heavy, 3].mean():.0f}")
for tt in np.linspace(0, en.max(), 16):
    print(f"t={tt:7.3f} ms running={(np.sum((st <= tt) & (en > tt)))}")
by_layer = np.bincount((np.arange(ntask) * 32 // 16384), weights=dur) if cfg == 1 else None
if by_layer is not None:
    print("task-ms by layer:", np.round(by_layer[:16], 1))
