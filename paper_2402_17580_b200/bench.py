"""Throughput and roofline harness of the step_all path, on the GPU.

Mirrors ti64micro/bench.py (the reference's own benchmark API):
``BLOCK_SIZES``, the analytic per-branch flop constants (bench.py:45-59),
``generate_layout`` (:61-80), ``measure_bandwidth`` (:83-108),
``measure_peak_flops`` (:111-128), ``measure_throughput`` (:131-155),
``count_flops`` (:158-205), ``RooflineReport`` (:208-257) and ``roofline``
(:260-275).  The machine baselines become device measurements — a DAXPY
stream (``ti64_bench_daxpy``) and a DFMA stream (``ti64_bench_dfma``) timed
with CUDA events — and ``measure_throughput`` times step_all on the device
(events around the call, pristine state restored outside the timed region).
``count_flops`` and ``RooflineReport`` are host arithmetic, identical to
the reference (pinned by tests/golden/report.npz).

(The repo-root bench.py is the driver's benchmark contract; this module is
the package's drop-in for ``ti64micro.bench``.)
"""

from dataclasses import dataclass, field

import numpy as np

from .batch import BYTES_PER_POINT, DOF_PER_POINT, GlobalFields, step_all
from .integrator import IntegratorConfig
from .kinetics import DEFAULT_PARAMS

__all__ = ["BLOCK_SIZES", "MIX_FACTOR_PRESETS", "generate_layout", "measure_bandwidth",
           "measure_peak_flops", "measure_throughput", "count_flops", "RooflineReport",
           "roofline"]

MIX_FACTOR_PRESETS = {"none": 1.0, "intel-server": 0.43, "amd-epyc": 0.57}
BLOCK_SIZES = (1, 10, 100)

# analytic per-lane operation counts (mul/add/sub/div = 1, fma = 2)
FLOPS_EXP = 19
FLOPS_LN = 26
FLOPS_POW = FLOPS_LN + FLOPS_EXP + 1
FLOPS_TFUNCS = 2 + 1 + (FLOPS_EXP + 3) + (FLOPS_EXP + 4)
FLOPS_XMEQ_BASE = FLOPS_EXP + 3
FLOPS_BRANCH_SHARED = FLOPS_POW
FLOPS_BRANCH_GROW = FLOPS_POW + 3
FLOPS_BRANCH_AM = FLOPS_POW + 3
FLOPS_BRANCH_DISSOLVE = 2 * FLOPS_POW + 6
FLOPS_RATES_BASE = 4
FLOPS_EULER = 4
FLOPS_CORRECTIONS = 10
FLOPS_WRMS = 12


def _layout_arrays(block_size, n_points, seed=0):
    """bench.py:61-80: even blocks cool mid-transformation (beta -> alpha_s
    growth near 1000 K), odd blocks heat above equilibrium (dissolution near
    1150 K); numpy's seeded generator, as there."""
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    rng = np.random.default_rng(seed)
    odd = (np.arange(n_points) // block_size) % 2 == 1
    t_old = np.where(odd, 1150.0, 1000.0) + rng.uniform(-20.0, 20.0, n_points)
    t_new = t_old + np.where(odd, 1.0, -1.0)
    xs = np.where(odd, 0.80, 0.20) + rng.uniform(-0.02, 0.02, n_points)
    xm = np.zeros(n_points)
    return xs, xm, 1.0 - xs - xm, t_old, t_new


def generate_layout(block_size, n_points, seed=0, params=DEFAULT_PARAMS, device=None):
    """Deterministic device-resident fields whose branch conditions alternate
    per block (bench.py:61-80)."""
    return GlobalFields(*_layout_arrays(block_size, n_points, seed), device=device)


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def measure_bandwidth(n=20_000_000, repetitions=8, threads=1):
    """Stream-update (DAXPY) bandwidth in GB/s, 24 B per element, on the
    device (bench.py:83-108; `threads` is ignored)."""
    import torch
    from . import _lib
    lib = _lib.require()
    x = torch.full((n,), 1.0, dtype=torch.float64, device="cuda")
    y = torch.full((n,), 2.0, dtype=torch.float64, device="cuda")
    st = _lib.stream_handle()
    _lib.check(lib.ti64_bench_daxpy(_lib.ptr(y), _lib.ptr(x), 0.999999, n, st),
               "ti64_bench_daxpy")
    best = np.inf
    for _ in range(repetitions):
        e0, e1 = _events(torch)
        e0.record()
        _lib.check(lib.ti64_bench_daxpy(_lib.ptr(y), _lib.ptr(x), 1.000001, n, st),
                   "ti64_bench_daxpy")
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return 24.0 * n / best / 1e9


def measure_peak_flops(lanes=4096, reps=4096, repetitions=8):
    """Peak FP64 FMA throughput in GFlop/s (2 flops per FMA) from the device
    DFMA stream (bench.py:111-128; lanes/reps size the CPU loop there and are
    ignored here)."""
    import torch
    from . import _lib
    lib = _lib.require()
    sc = torch.zeros(1, dtype=torch.float64, device="cuda")
    dev = torch.cuda.current_device()
    blocks = torch.cuda.get_device_properties(dev).multi_processor_count * 8
    st = _lib.stream_handle()
    lib.ti64_bench_dfma(_lib.ptr(sc), 2000, blocks, st)
    best = 0.0
    for _ in range(repetitions):
        e0, e1 = _events(torch)
        e0.record()
        fl = _lib.check(lib.ti64_bench_dfma(_lib.ptr(sc), 20000, blocks, st), "ti64_bench_dfma")
        e1.record()
        e1.synchronize()
        best = max(best, fl / (e0.elapsed_time(e1) * 1e-3))
    return best / 1e9


def measure_throughput(layout, scheme="explicit", n_lanes=8, repetitions=20, warmup=10,
                       dt=0.01, params=DEFAULT_PARAMS, threads=1):
    """Median DoF/s of step_all on the layout (bench.py:131-155), timed on
    the device; each repetition starts from a copy of the pristine layout
    made outside the timed region.  Returns (dof_per_s, median_seconds,
    iters_per_point or None) — iters as a numpy int64 array."""
    import torch
    config = IntegratorConfig(scheme=scheme, dt_sub_max=dt)
    pristine = layout.copy()
    times = []
    for rep in range(warmup + repetitions):
        work = pristine.copy()
        e0, e1 = _events(torch)
        e0.record()
        step_all(work, dt, params, config, n_lanes=n_lanes, threads=threads)
        e1.record()
        e1.synchronize()
        if rep >= warmup:
            times.append(e0.elapsed_time(e1) * 1e-3)
    iters = None
    if scheme == "crank_nicolson":
        work = pristine.copy()
        iters = step_all(work, dt, params, config, n_lanes=n_lanes, threads=threads,
                         record_iters=True).cpu().numpy()
    med = float(np.median(times))
    return DOF_PER_POINT * layout.n_points / med, med, iters


def _host(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def count_flops(layout, scheme="explicit", n_lanes=8, dt=0.01, params=DEFAULT_PARAMS,
                iters=None):
    """Analytic flop count of one step_all on the layout (bench.py:158-205):
    a branch any lane of a batch needs is charged to all n_lanes lanes."""
    from .batch import fast_exp
    xs_h = _host(layout.x_alpha_s)
    xm_h = _host(layout.x_alpha_m)
    t0_h = _host(layout.temperature_old)
    t1_h = _host(layout.temperature_new)
    n = len(xs_h)
    nbat = (n + n_lanes - 1) // n_lanes
    pad = nbat * n_lanes

    def batched(a, fill):
        out = np.full(pad, fill)
        out[:n] = a
        out[n:] = a[-1] if n else fill
        return out.reshape(nbat, n_lanes)

    xs = batched(xs_h, 0.0)
    xm = batched(xm_h, 0.0)
    t0 = batched(t0_h, 1000.0)
    t1 = batched(t1_h, 1000.0)
    xa = xs + xm
    flops = 2 * FLOPS_TFUNCS * pad
    form = (t1 < params.t_alpha_m_start).any(axis=1)
    flops += FLOPS_XMEQ_BASE * n_lanes * int(form.sum())
    tf = t0.ravel()
    ramp = 1.0 - np.asarray(fast_exp(-params.k_alpha_eq * (params.t_alpha_s_start - tf)))
    xaeq0 = np.where(tf < params.t_alpha_s_end, 0.9,
                     np.where(tf > params.t_alpha_s_start, 0.0, ramp)).reshape(nbat, n_lanes)
    grow = (xa < xaeq0) & (xs > 0.0)
    am = (xm > 0.0) & (xs > 0.0)
    dis = (xa > xaeq0) & (xa < 0.9)
    n_shared = int((grow.any(axis=1) | am.any(axis=1)).sum())
    flops += FLOPS_BRANCH_SHARED * n_lanes * n_shared
    flops += FLOPS_BRANCH_GROW * n_lanes * int(grow.any(axis=1).sum())
    flops += FLOPS_BRANCH_AM * n_lanes * int(am.any(axis=1).sum())
    flops += FLOPS_BRANCH_DISSOLVE * n_lanes * int(dis.any(axis=1).sum())
    flops += (FLOPS_RATES_BASE + FLOPS_EULER + FLOPS_CORRECTIONS) * pad
    if scheme == "crank_nicolson":
        mean_iters = float(np.mean(iters)) if iters is not None else 2.0
        per_iter = (FLOPS_BRANCH_SHARED + FLOPS_BRANCH_GROW + FLOPS_BRANCH_DISSOLVE
                    + FLOPS_RATES_BASE + FLOPS_CORRECTIONS + FLOPS_WRMS)
        flops += int((1.0 + mean_iters) * per_iter * pad)
    return flops


@dataclass
class RooflineReport:
    """Measured runs against the device's memory and compute ceilings
    (bench.py:208-257)."""

    measured_bandwidth: float          # GB/s
    peak_flops: float                  # GFlop/s
    instruction_mix_factor: float = 1.0
    rows: list = field(default_factory=list)

    def add_run(self, label, flops, bytes_modeled, seconds):
        intensity = flops / bytes_modeled
        achieved = flops / seconds / 1e9
        ceiling = min(self.peak_flops * self.instruction_mix_factor,
                      intensity * self.measured_bandwidth)
        self.rows.append({"label": label, "flops": flops, "bytes": bytes_modeled,
                          "seconds": seconds, "gflops": achieved, "intensity": intensity,
                          "ceiling": ceiling})

    @property
    def memory_bound_dof_rate(self):
        """Modeled memory-bound throughput: bandwidth / 24 B per DoF (GDoF/s)."""
        return self.measured_bandwidth / (BYTES_PER_POINT / DOF_PER_POINT)

    def respects_ceilings(self, slack=0.05):
        return all(r["gflops"] <= r["ceiling"] * (1.0 + slack) for r in self.rows)

    def to_csv(self):
        lines = ["label,flops,bytes,seconds,gflops,intensity,ceiling_gflops"]
        for r in self.rows:
            lines.append(f"{r['label']},{r['flops']},{r['bytes']},{r['seconds']!r},"
                         f"{r['gflops']!r},{r['intensity']!r},{r['ceiling']!r}")
        return "\n".join(lines) + "\n"

    def to_gnuplot(self):
        lines = ["# intensity_flop_per_byte achieved_gflops ceiling_gflops label"]
        for r in self.rows:
            lines.append(f"{r['intensity']!r} {r['gflops']!r} {r['ceiling']!r} {r['label']}")
        lines.append("")
        lines.append("# ceilings: memory = intensity * bandwidth; compute = peak * mix")
        lines.append(f"# bandwidth_gb_s = {self.measured_bandwidth!r}")
        lines.append(f"# peak_gflops = {self.peak_flops!r}")
        lines.append(f"# mix_factor = {self.instruction_mix_factor!r}")
        return "\n".join(lines) + "\n"


def roofline(runs, measured_bandwidth=None, peak_flops=None, instruction_mix_factor=1.0,
             threads=1):
    """RooflineReport from runs (dicts: label, flops, bytes, seconds); the
    device baselines are measured unless supplied (bench.py:260-275)."""
    bw = measured_bandwidth if measured_bandwidth is not None else measure_bandwidth()
    pk = peak_flops if peak_flops is not None else measure_peak_flops()
    rep = RooflineReport(bw, pk, instruction_mix_factor)
    for r in runs:
        rep.add_run(r["label"], r["flops"], r["bytes"], r["seconds"])
    return rep
