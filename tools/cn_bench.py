"""Implicit-scheme throughput on the reference's CPU-benchmark layouts
(bench.py:131-155 measure_throughput: dt = dt_sub_max = 0.01, pristine state
restored outside the timed region) with its analytic flop count
(bench.py:158-205) against the measured FP64 DFMA peak."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
import paper_2402_17580_b200 as pkg  # noqa: E402
from paper_2402_17580_b200 import _lib  # noqa: E402


def main(n=1 << 22, lanes_list=(8, 1), reps=7):
    dev = torch.device("cuda", 0)
    lib = _lib.require()
    peak = bench.measure_fp64_peak(torch, lib, torch.cuda.current_stream())
    rows = []
    for scheme in ("crank_nicolson", "explicit"):
        cfg = pkg.IntegratorConfig(scheme=scheme, dt_sub_max=0.01)
        for block in (1, 10, 100):
            lay = bench.branch_layout(block, n)
            pristine = pkg.GlobalFields(*lay, device=dev)
            for lanes in lanes_list:
                ts = []
                iters = None
                for r in range(reps + 2):
                    w = pristine.copy()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    it = pkg.step_all(w, 0.01, config=cfg, n_lanes=lanes,
                                      record_iters=(r == 0))
                    e1.record()
                    e1.synchronize()
                    if r == 0 and it is not None:
                        iters = it.double().mean().item()
                    if r >= 2:
                        ts.append(e0.elapsed_time(e1) * 1e-3)
                t = float(np.median(ts))
                fl = bench.reference_flops(lay[0], lay[1], lay[3], lay[4], lanes, scheme,
                                           iters)
                rows.append({"scheme": scheme, "block": block, "lanes": lanes, "n": n,
                             "ms": t * 1e3, "GDoF/s": 3 * n / t / 1e9,
                             "mean_iters": iters, "ref_flops_per_point": fl / n,
                             "TF/s": fl / t / 1e12, "frac_fp64_peak": fl / t / peak})
                print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"fp64_peak_TF/s": peak / 1e12}))


if __name__ == "__main__":
    main()
