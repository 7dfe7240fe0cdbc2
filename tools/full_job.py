"""A whole pure-ODE job on one GPU, as one rank of a sharded run: config 2
(all 2^24 points, 50 000 steps) and config 4 (rank 0 of 8: its 2^24-point
shard, 100 000 steps), with snapshots every 1000 steps, event counters and the
256-bin phase histograms.  Prints one JSON line per config.
    python tools/full_job.py [--configs 2,4] [--world 8]"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402
from paper_2402_17580_b200.distributed import ShardedAdvance  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,4")
ap.add_argument("--world", type=int, default=8, help="ranks of the config-4 job (this is rank 0)")
a = ap.parse_args()
jobs = {2: (1 << 24, 50000, 1), 4: (1 << 27, 100000, a.world)}
for c in [int(x) for x in a.configs.split(",")]:
    n_total, steps, world = jobs[c]
    src = pkg.source_for_config(c)
    job = ShardedAdvance(src, n_total, rank=0, world=world)
    n = job.hi - job.lo
    cnt = pkg.EventCounters(n, torch.device("cuda", 0))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    sums = job.run(steps, snapshot_every=1000, counters=cnt, reduce=False)
    hist = job.histogram(256, reduce=False)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    s = e0.elapsed_time(e1) * 1e-3
    tot = cnt.totals_dict()
    h = hist.cpu().numpy().reshape(3, -1)
    print(json.dumps({
        "config": c, "points_total": n_total, "shard_points": n, "world": world, "steps": steps,
        "device_s": s, "wall_s": wall, "point_updates_per_s": n * steps / s,
        "job_estimate_s_at_world": s if world > 1 else None,
        "final_mean_fractions": (sums[-1].double().cpu().numpy() / n).tolist(),
        "totals": tot, "hist_nonzero_bins": [int((h[k] > 0).sum()) for k in range(3)],
        "hist_checksum": int(h.sum())}), flush=True)
