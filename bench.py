#!/usr/bin/env python
"""bench.py — microstructure point-updates/s (fp64) on B200.

Headline workload: BASELINE.json configs[4], the largest configuration that
fits one GPU (the metric string names no config, so the largest one is the
one it is quoted on): N = 2^27 points, per-point seeded histories of 1-20
Gaussian pulses (peaks U(600, 3000) K, widths log-uniform on [1e-4, 1e-2] s,
centres U(0, 1) s, base 300 K), dt = 1e-5 s, a 100 000-step job; every point
is advanced by the explicit update each step.

One bench "step" = one WINDOW of 200 consecutive time steps of that job over
all 2^27 points (5.4e9 point-updates), run by one launch of the fused
advance kernel K2 (+ the snapshot phase-sum kernel).  The state is prepared
untimed up to step 20 000 (where the per-window rate has reached the
whole-job average to within a few %, tools/window_rates.py), then W warm-up
windows, then K timed windows: steps 20 000 + 200 W ... of the real job.
The timed region ends with the 3x256-bin phase-fraction histogram and the
cross-rank all-reduce of sums, histogram and counters.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--gpus N without torchrun spawns N ranks itself (one process per GPU,
127.0.0.1 rendezvous); the 2^27 points are sharded in contiguous blocks
(strong scaling: total work fixed); max-over-ranks device time.

--impl reference times the reference's own CPU implementation (ti64micro's
numba step_all from baseline/_ref, n_lanes=8, all host threads) on a bounded
sample of the same windows: every 1024th point of the 2^27, state prepared
by the oracle (bit-identical to the reference, checked on the sample), the
per-step temperatures generated outside the timed region.
"""

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "microstructure point-updates/s (fp64)"
UNIT = "point-updates/s"
HEADLINE = 4
# per config: total points, job steps, window steps (one bench step), start
# step of the warm-up windows, stride of the CPU sample (global indices)
CONFIGS = {
    4: dict(n=1 << 27, job=100_000, window=200, start=20_000, stride=1024),
    2: dict(n=1 << 24, job=50_000, window=200, start=10_000, stride=128),
    1: dict(n=1 << 20, job=10_000, window=10_000, start=0, stride=8),
    0: dict(n=4096, job=20_000, window=20_000, start=0, stride=1),
}
WORKLOADS = {
    4: "config4: 1-20 Gaussian pulses/point, peaks U(600,3000) K, widths log-U[1e-4,1e-2] s, "
       "centres U(0,1) s, base 300 K; N=2^27 points, dt=1e-5 s, 100000-step job",
    2: "config2: 10 re-scan pulses on 353 K, seeded xs0 U(0.8,0.95); N=2^24, dt=1e-5 s, "
       "50000-step job",
    1: "config1: Rosenthal raster (200 W, eta 0.35, 1 m/s, 100 um hatch) on a 128x128x64 "
       "lattice h=20um; N=2^20, dt=2e-5 s, 10000-step job",
    0: "config0: one Gaussian pulse/point; N=4096, dt=1e-5 s, 20000-step job",
}
# Algorithmic flops per point-update (the reference's count_flops
# constants bench.py:45-58 at n_lanes=1, minus the carried T_n functions):
# F = 48 + 22[T1<848] + 46[grow|am] + 49[grow] + 49[am] + 98[dissolve] + 18
F_BASE, F_FORM, F_GA, F_GROW, F_AM, F_DIS, F_TAIL = 48, 22, 46, 49, 49, 98, 18
# executed view and DRAM traffic of the headline launch, from the committed
# ncu capture of the bench workload (profiles/README.md, round 2)
K2_PROFILE = {
    "file": "profiles/r02l_advance_cfg4_window.txt (ncu --set full of the first timed window "
            "launch at HEAD, 2^27 points, steps 20200-20400)",
    "dram_bytes_per_launch": 33_225_701_000 + 22_913_592_000,  # read + write
    "fp64_pipe_active": 0.5934, "issue_active": 0.7855,
    # FP64-pipe warp instructions per 32 point-updates (DFMA+DADD+DMUL+DSETP+FRND) of that launch
    "fp64_inst_per_update": 130.9,
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def config_dict(cfg_id, n_gpus, K, W):
    c = CONFIGS[cfg_id]
    t0 = c["start"] + W * c["window"]
    d = {"workload": WORKLOADS[cfg_id], "config_id": cfg_id, "points": c["n"],
         "job_steps": c["job"], "window_steps": c["window"],
         "timed_steps": [t0, t0 + K * c["window"]],
         "step": f"{c['window']} consecutive time steps of the job over all points",
         "l2": "inputs larger than L2 (state 50 B/point)" if c["n"] * 50 > (256 << 20)
         else "L2 flushed between timed iterations (256 MiB write)",
         "parallelism": f"points sharded in contiguous blocks over {n_gpus} GPU(s), "
                        "no communication until the final all-reduce"}
    return d


# ---------------------------------------------------------------------------
# launching: one process per GPU
# ---------------------------------------------------------------------------

def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n, argv):
    """Run this script as n ranks (RANK/LOCAL_RANK/WORLD_SIZE/MASTER_*), as
    torchrun would; rank 0's stdout is this process's stdout."""
    port = free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()), *argv],
                                      env=env, stdout=None if r == 0 else subprocess.DEVNULL))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                s, m = float(p[1]), float(p[2])
            except ValueError:
                continue
            sm.append(s)
            smax = max(smax, m)
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def flops_from_totals(t):
    return (F_BASE + F_TAIL) * t["point_updates"] + F_FORM * t["n_form"] + \
        F_GA * t["n_grow_or_am"] + F_GROW * t["n_grow"] + F_AM * t["n_am"] + \
        F_DIS * t["n_dissolve"]


# The reference's analytic flop count of one step_all on a layout
# (bench.py:158-205 count_flops, its per-branch constants bench.py:45-59):
# a branch any lane of a batch needs is charged to all lanes of the batch;
# the implicit scheme adds (1 + mean iterations) x the per-iteration work.
R_EXP, R_LN = 19, 26
R_POW = R_LN + R_EXP + 1
R_TFUNCS = 2 + 1 + (R_EXP + 3) + (R_EXP + 4)
R_XMEQ = R_EXP + 3
R_SHARED, R_GROW, R_AM, R_DIS = R_POW, R_POW + 3, R_POW + 3, 2 * R_POW + 6
R_RATES, R_EULER, R_CORR, R_WRMS = 4, 4, 10, 12


def reference_flops(xs, xm, t0, t1, n_lanes, scheme="explicit", mean_iters=None,
                    params=None):
    from paper_2402_17580_b200.kinetics import DEFAULT_PARAMS
    p = params or DEFAULT_PARAMS
    n = len(xs)
    nbat = (n + n_lanes - 1) // n_lanes
    pad = nbat * n_lanes

    def batched(a, fill):
        out = np.full(pad, fill)
        out[:n] = a
        out[n:] = a[-1] if n else fill
        return out.reshape(nbat, n_lanes)

    xs, xm = batched(xs, 0.0), batched(xm, 0.0)
    t0, t1 = batched(t0, 1000.0), batched(t1, 1000.0)
    xa = xs + xm
    fl = 2 * R_TFUNCS * pad
    fl += R_XMEQ * n_lanes * int((t1 < p.t_alpha_m_start).any(axis=1).sum())
    ramp = 1.0 - np.exp(-p.k_alpha_eq * (p.t_alpha_s_start - t0))
    xaeq0 = np.where(t0 < p.t_alpha_s_end, 0.9, np.where(t0 > p.t_alpha_s_start, 0.0, ramp))
    grow = (xa < xaeq0) & (xs > 0.0)
    am = (xm > 0.0) & (xs > 0.0)
    dis = (xa > xaeq0) & (xa < 0.9)
    fl += R_SHARED * n_lanes * int((grow.any(axis=1) | am.any(axis=1)).sum())
    fl += R_GROW * n_lanes * int(grow.any(axis=1).sum())
    fl += R_AM * n_lanes * int(am.any(axis=1).sum())
    fl += R_DIS * n_lanes * int(dis.any(axis=1).sum())
    fl += (R_RATES + R_EULER + R_CORR) * pad
    if scheme == "crank_nicolson":
        mi = 2.0 if mean_iters is None else float(mean_iters)
        per_iter = R_SHARED + R_GROW + R_DIS + R_RATES + R_CORR + R_WRMS
        fl += int((1.0 + mi) * per_iter * pad)
    return fl


def branch_layout(block, n, seed=0):
    """The reference's CPU-benchmark layout (bench.py:62-80 generate_layout)."""
    rng = np.random.default_rng(seed)
    odd = (np.arange(n) // block) % 2 == 1
    t_old = np.where(odd, 1150.0, 1000.0) + rng.uniform(-20.0, 20.0, n)
    t_new = t_old + np.where(odd, 1.0, -1.0)
    xs = np.where(odd, 0.80, 0.20) + rng.uniform(-0.02, 0.02, n)
    xm = np.zeros(n)
    return xs, xm, 1.0 - xs - xm, t_old, t_new


# ---------------------------------------------------------------------------
# CPU legs (the oracle port and the reference itself) on a strided sample
# ---------------------------------------------------------------------------

NAMES = ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old", "temperature_new",
         "seed_tracked", "seed_active", "seed_direction")


def cpu_threads():
    return os.cpu_count() or 1


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_windows(step_fn, fields, gen, pts, t0, window, max_windows, budget_s, threads):
    """Run whole windows of step_fn(fields) from step t0 with the sample's
    temperatures generated outside the timed region; returns (seconds,
    windows)."""
    from oracle import oracle as orc
    timed, done = 0.0, 0
    while done < max_windows and (done == 0 or timed < budget_s):
        T = orc.gen_temperature_points(gen, pts, t0 + done * window + 1, window, threads)
        for s in range(window):
            fields.temperature_new[:] = T[s]
            c0 = time.perf_counter()
            step_fn(fields)
            timed += time.perf_counter() - c0
        done += 1
    return timed, done


def oracle_sample_rate(cfg_id, state, pts, t0, max_windows, budget_s):
    """The oracle port's step_all (lanes=8, OpenMP over all host threads) on
    the sample, from `state` (numpy arrays of the sample at step t0)."""
    from oracle import oracle as orc
    from paper_2402_17580_b200 import sources
    from paper_2402_17580_b200.integrator import IntegratorConfig
    from paper_2402_17580_b200.kinetics import DEFAULT_PARAMS
    c = CONFIGS[cfg_id]
    src = sources.source_for_config(cfg_id)
    gen = src.tempgen(point_offset=0, **_beam_kw(src, c["job"] + 1))
    threads = cpu_threads()
    kp = DEFAULT_PARAMS.kernel_tuple()
    cfg = IntegratorConfig().kernel_tuple()
    f = orc.HostFields(*[state[k] for k in NAMES])
    secs, wins = cpu_windows(lambda fl: orc.step_all(fl, src.dt, kp, cfg, n_lanes=8,
                                                     threads=threads),
                             f, gen, pts, t0, c["window"], max_windows, budget_s, threads)
    upd = len(pts) * c["window"] * wins
    return {"value": upd / secs, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"every {c['stride']}th point ({len(pts)} points) x {wins} window(s) of "
                      f"{c['window']} steps from step {t0}; oracle/ti64_oracle.c step_all "
                      f"(lanes=8, OpenMP {threads} threads on {cpu_model()}), T generated "
                      f"outside the timed region; {secs:.1f} s timed",
            "seconds": secs, "windows": wins, "fields": f}


_BEAMS = {}


def _beam_kw(src, rows):
    """Host beam table for the oracle's Rosenthal generator (config 1)."""
    tab_fn = getattr(src, "beam_table", None)
    if tab_fn is None:
        return {}
    tab = _BEAMS.get((src, rows))
    if tab is None:
        tab = tab_fn(rows)
        if tab is None:
            return {}
        tab = np.ascontiguousarray(tab)
        _BEAMS[(src, rows)] = tab
    return {"beam_ptr": tab.ctypes.data, "beam_steps": rows}


def import_reference():
    """ti64micro (the unmodified reference) from baseline/_ref, or None."""
    # the unresolved /root/repo path (a symlink to the run directory on the
    # GPU box): numba keys its on-disk cache by the source path, so a stable
    # path lets a cache made on one box serve the next
    stable = Path("/root/repo/baseline/_ref")
    ref = stable if (stable / "ti64micro").exists() else ROOT / "baseline" / "_ref"
    if not (ref / "ti64micro").exists():
        return None, "baseline/_ref/ti64micro missing"
    cache = ref / ".numba_cache"
    try:
        cache.mkdir(exist_ok=True)
        os.environ.setdefault("NUMBA_CACHE_DIR", str(cache))
    except OSError:
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ti64_numba_cache")
    os.environ.setdefault("NUMBA_NUM_THREADS", str(cpu_threads()))
    sys.path.insert(0, str(ref))
    try:
        import ti64micro  # noqa: F401
        from ti64micro import batch, integrator, kinetics
        return (batch, integrator, kinetics), None
    except Exception as e:  # numba missing on the box, etc.
        return None, f"{type(e).__name__}: {e}"


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg_id = HEADLINE
    c = CONFIGS[cfg_id]
    from oracle import oracle as orc
    from paper_2402_17580_b200 import sources
    from paper_2402_17580_b200.integrator import IntegratorConfig
    from paper_2402_17580_b200.kinetics import DEFAULT_PARAMS
    src = sources.source_for_config(cfg_id)
    gen = src.tempgen(point_offset=0)
    threads = cpu_threads()
    pts = np.arange(0, c["n"], c["stride"], dtype=np.int64)
    t_start = c["start"] + args.warmup * c["window"]
    kp = DEFAULT_PARAMS.kernel_tuple()
    icfg = IntegratorConfig().kernel_tuple()
    # state of the sample at the first timed step: the oracle (bit-identical
    # to the reference, checked below on the timed windows)
    c0 = time.perf_counter()
    h = orc.gen_initial_points(gen, pts)
    orc.advance_points(h, pts, gen, 0, t_start, kp, icfg, threads=threads)
    prep_s = time.perf_counter() - c0
    start_state = {k: getattr(h, k).copy() for k in NAMES}
    mods, why = import_reference()
    kind, jit_s, check = "reference", None, None
    if mods is not None:
        rbatch, rinteg, rkin = mods
        import numba
        rf = rbatch.GlobalFields(*[start_state[k].copy() for k in NAMES[:5]],
                                 seed_tracked=start_state["seed_tracked"].copy(),
                                 seed_active=start_state["seed_active"].copy(),
                                 seed_direction=start_state["seed_direction"].copy())
        rcfg = rinteg.IntegratorConfig(scheme="explicit")
        c0 = time.perf_counter()
        warm = rbatch.GlobalFields(*[start_state[k][:64].copy() for k in NAMES[:5]])
        rbatch.step_all(warm, src.dt, rkin.DEFAULT_PARAMS, rcfg, n_lanes=8, threads=threads)
        jit_s = time.perf_counter() - c0
        secs, wins = cpu_windows(
            lambda fl: rbatch.step_all(fl, src.dt, rkin.DEFAULT_PARAMS, rcfg, n_lanes=8,
                                       threads=threads),
            rf, gen, pts, t_start, c["window"], args.steps, 1e30, threads)
        layer = numba.threading_layer()
        desc = (f"ti64micro.batch.step_all (the unmodified reference, baseline/_ref, numba "
                f"{numba.__version__} threading layer {layer}, n_lanes=8, threads={threads}) on "
                f"{cpu_model()}")
        if not args.no_ref_check:  # the oracle on the same windows: bitwise equal states
            o = orc.HostFields(*[start_state[k] for k in NAMES])
            orc.advance_points(o, pts, gen, t_start, wins * c["window"], kp, icfg,
                               threads=threads)
            check = all(np.array_equal(np.asarray(getattr(rf, k)).view(np.uint8),
                                       getattr(o, k).view(np.uint8))
                        for k in ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old"))
    else:
        kind = "port"
        f = orc.HostFields(*[start_state[k] for k in NAMES])
        secs, wins = cpu_windows(lambda fl: orc.step_all(fl, src.dt, kp, icfg, n_lanes=8,
                                                         threads=threads),
                                 f, gen, pts, t_start, c["window"], args.steps, 1e30, threads)
        desc = (f"oracle/ti64_oracle.c step_all (port; the reference could not be imported: "
                f"{why}), lanes=8, OpenMP {threads} threads on {cpu_model()}")
    cfg3 = None
    if mods is not None and not args.no_config3:
        try:
            cfg3 = reference_config3_step(mods, threads)
        except Exception as e:  # keep the headline line even if this extra fails
            cfg3 = {"error": f"{type(e).__name__}: {e}"}
    upd = len(pts) * c["window"] * wins
    value = upd / secs
    sample = (f"every {c['stride']}th point of the 2^27 ({len(pts)} points) x {wins} window(s) "
              f"of {c['window']} steps from step {t_start}: {desc}; T generated outside the "
              f"timed region; sample state prepared by the oracle in {prep_s:.1f} s")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": wins, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / wins, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg_id, args.gpus, args.steps, args.warmup),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "reference_extra": {"jit_seconds": jit_s, "prep_seconds": prep_s,
                                "timed_seconds": secs,
                                "ms_per_step_note": "one step = one window of the bounded "
                                                    "sample (not of all 2^27 points)",
                                "reference_equals_oracle_bitwise": check,
                                "config3_full_grid_step": cfg3}}
    print(json.dumps(line), flush=True)
    return 0


def reference_config3_step(mods, threads):
    """BASELINE.md §3 for config 3: one full-grid 512x512x256 coupled step of
    the reference on the host — thermal.step_thermal(field, 1e-6,
    losses=False, bottom_dirichlet=353) (serial numba _stencil_step) then
    step_all (n_lanes=8, all threads) on the aliased temperature buffers, as
    run_build's couple does (thermal.py:541-555); JIT excluded."""
    import importlib
    rbatch, rinteg, rkin = mods
    rth = importlib.import_module("ti64micro.thermal")
    nz, ny, nx, h = 256, 512, 512, 20e-6
    src = rth.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=h)
    beam = (5e-3, 5e-3, 0.35 * 250.0, True)
    rcfg = rinteg.IntegratorConfig(scheme="explicit")

    def domain(nz_, ny_, nx_):
        n = nz_ * ny_ * nx_
        t_old, t_new = np.full(n, 353.0), np.full(n, 353.0)
        f = rbatch.GlobalFields(np.full(n, 0.9), np.zeros(n), np.full(n, 0.1), t_old, t_new)
        field = rth.ThermalField(f.temperature_old.reshape(nz_, ny_, nx_),
                                 f.temperature_new.reshape(nz_, ny_, nx_),
                                 np.ones((nz_, ny_, nx_)),
                                 np.full((nz_, ny_, nx_), 2, np.uint8), h, nz_)
        return f, field

    def step(f, field):
        rth.step_thermal(field, 1e-6, rth.DEFAULT_THERMAL, src, beam, losses=False,
                         bottom_dirichlet=353.0)
        rbatch.step_all(f, 1e-6, rkin.DEFAULT_PARAMS, rcfg, n_lanes=8, threads=threads)

    c0 = time.perf_counter()
    step(*domain(4, 8, 8))  # JIT warm-up
    jit = time.perf_counter() - c0
    f, field = domain(nz, ny, nx)
    c0 = time.perf_counter()
    rth.step_thermal(field, 1e-6, rth.DEFAULT_THERMAL, src, beam, losses=False,
                     bottom_dirichlet=353.0)
    t_st = time.perf_counter() - c0
    c0 = time.perf_counter()
    rbatch.step_all(f, 1e-6, rkin.DEFAULT_PARAMS, rcfg, n_lanes=8, threads=threads)
    t_sa = time.perf_counter() - c0
    n = nz * ny * nx
    return {"cell_steps_per_s": n / (t_st + t_sa), "seconds": t_st + t_sa,
            "step_thermal_seconds": t_st, "step_all_seconds": t_sa, "jit_seconds": jit,
            "what": "one full-grid 512x512x256 step: step_thermal (serial numba _stencil_step, "
                    "losses off, Dirichlet 353 K) + step_all (n_lanes=8, threads="
                    f"{threads}) of the unmodified reference"}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def measure_fp64_peak(torch, lib, stream):
    import ctypes as C
    from paper_2402_17580_b200 import _lib
    sc = torch.zeros(1, dtype=torch.float64, device="cuda")
    blocks = 148 * 8
    best = 0.0
    h = C.c_void_p(stream.cuda_stream)
    for it in (2000, 20000, 20000, 20000):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fl = lib.ti64_bench_dfma(_lib.ptr(sc), it, blocks, h)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        if it > 2000:
            best = max(best, fl / (ms * 1e-3))
    return best


class Dist:
    def __init__(self, world, dev):
        self.world, self.dev = world, dev

    def barrier(self):
        import torch
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max(self, v):
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(v)], dtype=torch.float64, device=self.dev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_(self, t):
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t


def measure_ode(torch, pkg, cfg_id, K, W, rank, world, dev, dd, *, counted=True, e2e=True,
                cpu=True, cpu_budget=10.0, clocks=None, log_prefix=""):
    """Timed windows of config `cfg_id` on this rank's shard (see module doc).
    Returns a dict with value / timing / roofline inputs / e2e / cpu leg."""
    from paper_2402_17580_b200.distributed import shard_range
    c = CONFIGS[cfg_id]
    src = pkg.source_for_config(cfg_id)
    lo, hi = shard_range(c["n"], rank, world)
    n = hi - lo
    win = c["window"]
    stream = torch.cuda.current_stream()
    scratch = pkg.batch._scratch(n, dev)
    flush = None
    if c["n"] * 50 <= (256 << 20):
        flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    # restart mode: the window is the whole job (configs 0, 1), so every
    # window re-runs the job from the initial state (restored untimed)
    restart = win == c["job"]
    t_prep = time.perf_counter()
    f = pkg.init_from_source(src, n, point_offset=lo, device=dev)
    pristine = f.copy() if restart else None
    s = 0
    while s < c["start"]:  # untimed preparation, in launches of <= 5000 steps
        k = min(5000, c["start"] - s)
        pkg.advance(f, k, src, step0=s, point_offset=lo, scratch=scratch)
        s += k
    for _ in range(W):  # warm-up windows (untimed)
        if restart:
            _restore(pkg, f, pristine)
            s = 0
        pkg.advance(f, win, src, step0=s, point_offset=lo, snapshot_every=win, scratch=scratch)
        s += win
    if restart:
        _restore(pkg, f, pristine)
        s = 0
    torch.cuda.synchronize()
    prep_s = time.perf_counter() - t_prep
    t_first = s
    start_copy = f.copy() if (counted or cpu or e2e) else None
    hist = torch.zeros((3, 256), dtype=torch.int64, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K)]  # window starts
    ev_w = [torch.cuda.Event(enable_timing=True) for _ in range(K)]  # window ends
    ev_end = torch.cuda.Event(enable_timing=True)
    launches = 0
    sums = None
    dd.barrier()
    if clocks is not None:
        clocks.__enter__()
    for k in range(K):
        if restart and k > 0:
            _restore(pkg, f, pristine)
            s = 0
        if flush is not None:
            flush.fill_(1.0)
        ev[k].record(stream)
        r = pkg.advance(f, win, src, step0=s, point_offset=lo, snapshot_every=win,
                        scratch=scratch)
        ev_w[k].record(stream)
        launches += r.launches
        sums = r.sums
        s += win
    # end of the job's timed part: histogram + cross-rank reduction
    hist.zero_()
    pkg.histogram(f, 256, out=hist)
    launches += 1
    dd.sum_(hist)
    dd.sum_(sums)
    ev_end.record(stream)
    dd.barrier()
    if clocks is not None:
        clocks.__exit__(None, None, None)
    t_windows = [ev[k].elapsed_time(ev_w[k]) * 1e-3 for k in range(K)]
    # the region is the sum of the windows plus the final reduction (restart
    # mode restores the state between windows, untimed; otherwise the
    # windows are back to back)
    t_region = sum(t_windows) + ev_w[K - 1].elapsed_time(ev_end) * 1e-3
    t_max = dd.max(t_region)
    out = {"n_local": n, "lo": lo, "t_region": t_region, "t_max": t_max,
           "t_windows": t_windows, "launches": launches, "prep_s": prep_s,
           "first_step": t_first, "value": c["n"] * win * K / t_max,
           "hist_checksum": int((hist * torch.arange(1, 257, device=dev)).sum().item()),
           "sums_last": [float(x) for x in sums[-1].cpu().numpy()]}
    log(f"{log_prefix}config {cfg_id}: {out['value']:.4e} upd/s, "
        f"{1e3 * sum(t_windows) / K:.2f} ms/window, prep {prep_s:.1f} s")
    final = f
    # flop-model totals of the timed windows: the counted instance from the
    # same starting state; it must reproduce the timed run bit for bit
    stride = c["stride"]
    pts_local = np.arange(0, n, stride, dtype=np.int64)
    sample_after = []
    if counted:
        g = start_copy.copy()
        cnt = pkg.EventCounters(n, dev)
        s2 = t_first
        idx = torch.from_numpy(pts_local).to(dev)
        for k in range(K):
            if restart and k > 0:
                _restore(pkg, g, pristine)
                s2 = 0
            pkg.advance(g, win, src, step0=s2, point_offset=lo, snapshot_every=win,
                        counters=cnt, scratch=scratch)
            s2 += win
            sample_after.append({k2: getattr(g, k2)[idx].cpu().numpy()
                                 for k2 in ("x_alpha_s", "x_alpha_m", "x_beta",
                                            "temperature_old", "seed_active",
                                            "seed_tracked")})
        totals = cnt.totals_dict()
        out["totals"] = totals
        out["flops"] = flops_from_totals(totals)
        out["counted_equals_timed"] = all(
            torch.equal(getattr(g, k2).view(torch.uint8) if getattr(g, k2).dtype != torch.uint8
                        else getattr(g, k2),
                        getattr(final, k2).view(torch.uint8) if getattr(final, k2).dtype !=
                        torch.uint8 else getattr(final, k2))
            for k2 in pkg.batch.NAMES)
        del g, cnt
    # e2e through the public API with the data in pinned host memory
    if e2e:
        host = {k: torch.empty(getattr(final, k).shape, dtype=getattr(final, k).dtype,
                               pin_memory=True) for k in pkg.batch.NAMES}
        ref = start_copy.copy()
        pkg.advance(ref, win, src, step0=t_first, point_offset=lo, snapshot_every=win,
                    scratch=scratch)
        e2e_t = []
        same = None
        for k in range(max(1, min(K, 3))):
            for k2 in pkg.batch.NAMES:  # fresh inputs on the host, outside the timed region
                host[k2].copy_(getattr(start_copy, k2))
            dd.barrier()
            c0 = time.perf_counter()
            fh = pkg.GlobalFields(*[host[k2] for k2 in pkg.batch.NAMES], device="host")
            rh = pkg.advance(fh, win, src, step0=t_first, point_offset=lo, snapshot_every=win,
                             scratch=scratch)
            sums_h = rh.sums.cpu()
            torch.cuda.synchronize()
            e2e_t.append(time.perf_counter() - c0)
            if same is None:
                same = all(torch.equal(host[k2], getattr(ref, k2).cpu())
                           for k2 in pkg.batch.NAMES)
        t_e2e = dd.max(statistics.median(e2e_t))
        h2d = n * (5 * 8 + 2)  # xs, xm, xb, T_old, tracked + 2 flag bytes read
        d2h = n * (6 * 8 + 2) + sums_h.numel() * 8
        out["e2e"] = {"value": c["n"] * win / t_e2e, "unit": UNIT,
                      "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                      "path": "GlobalFields(device='host') + advance() -> ti64_advance_host: "
                              "the state lives in pinned host memory; chunks of 2^22 points are "
                              "staged through four device buffers, the host->device copies of "
                              "the next chunks and the device->host copy of the previous one "
                              "overlapping the chunks' updates; timed from the host arrays to "
                              "the phase sums and the updated host arrays",
                      "bitwise_equal_to_device_run": bool(same),
                      "seconds_per_step": t_e2e}
        del host, ref
    # CPU leg: the oracle port on every stride-th point of this shard from the
    # same starting state; its windows must equal the GPU's bit for bit
    if cpu and rank == 0 and world == 1:
        idx = torch.from_numpy(pts_local).to(dev)
        state = {k2: getattr(start_copy, k2)[idx].cpu().numpy() for k2 in pkg.batch.NAMES}
        leg = oracle_sample_rate(cfg_id, state, pts_local + lo, t_first, K, cpu_budget)
        wins = leg["windows"]
        if sample_after:
            got = sample_after[wins - 1]
            fo = leg["fields"]
            act = got["seed_active"] != 0
            leg["sample_equals_gpu_bitwise"] = bool(
                all(np.array_equal(got[k2].view(np.uint8), getattr(fo, k2).view(np.uint8))
                    for k2 in ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old",
                               "seed_active")) and
                np.array_equal(got["seed_tracked"][act].view(np.uint8),
                               fo.seed_tracked[act].view(np.uint8)))
        del leg["fields"]
        out["cpu"] = leg
    del start_copy, f, final, pristine
    torch.cuda.empty_cache()
    return out


def _restore(pkg, dst, src):
    for k in pkg.batch.NAMES:
        getattr(dst, k).copy_(getattr(src, k))


def roofline_of(m, peak_tf, K):
    """FP64 roofline of the K2 launches of a measure_ode result (per GPU)."""
    if "flops" not in m:
        return None
    t_launch = sum(m["t_windows"]) / K
    achieved = m["flops"] / K / t_launch / 1e12
    return {"bound": "fp64", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
            "frac": achieved / peak_tf,
            "flops_per_update": m["flops"] / m["totals"]["point_updates"],
            "per_launch_s": t_launch}


def measure_extra(torch, pkg, dev, dd, peak_tf, args):
    """Secondary lines (N = 1): config 2 at its full 2^24 points, configs 1
    and 0 as whole jobs, the whole config-4 job on a 2^21-point shard, the
    K4 stencil and the split coupled config-3 step at 512x512x256, K1's HBM
    fraction, and the Crank-Nicolson step_all."""
    from paper_2402_17580_b200 import thermal as th, scanpath
    out = {}
    hbm = 6538.0
    try:
        hbm = float(json.load(open(ROOT / "MEASURED_PEAKS.json"))["hbm_gbs"])
    except Exception:
        pass
    # config 2, all 2^24 points, mid-job windows
    m = measure_ode(torch, pkg, 2, 3, 1, 0, 1, dev, dd, cpu_budget=6.0, log_prefix="extra ")
    out["config2_full_2^24"] = {
        "point_updates_per_s": m["value"], "ms_per_window": 1e3 * sum(m["t_windows"]) / 3,
        "timed_steps": [m["first_step"], m["first_step"] + 3 * CONFIGS[2]["window"]],
        "roofline": roofline_of(m, peak_tf, 3), "e2e": m.get("e2e"),
        "cpu_baseline": {k: m["cpu"][k] for k in ("value", "unit", "cores", "kind", "sample",
                                                   "sample_equals_gpu_bitwise")},
        "counted_equals_timed_bitwise": m.get("counted_equals_timed")}
    # configs 1 and 0: one window = the whole job
    for cid in (1, 0):
        m = measure_ode(torch, pkg, cid, 3, 1, 0, 1, dev, dd, cpu_budget=5.0,
                        log_prefix="extra ")
        rl = roofline_of(m, peak_tf, 3)
        out[f"config{cid}_whole_job"] = {
            "point_updates_per_s": m["value"], "ms_per_job": 1e3 * sum(m["t_windows"]) / 3,
            "algorithmic_flop_rate": rl,
            "note": "the kernel proves most of these updates exact no-ops (cold idle rest, "
                    "steady skip) and skips them, so the algorithmic flop rate is not a "
                    "roofline of executed work" if cid == 1 else
                    "4096 points = 128 warps: latency-bound by size",
            "e2e": m.get("e2e"),
            "cpu_baseline": {k: m["cpu"][k] for k in ("value", "unit", "cores", "kind", "sample",
                                                       "sample_equals_gpu_bitwise")}}
    # whole config-4 job on a 2^21-point shard (per-window rates vs the job)
    src4 = pkg.source_for_config(4)
    nsh = 1 << 21
    f4 = pkg.init_from_source(src4, nsh, device=dev)
    scr = pkg.batch._scratch(nsh, dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pkg.advance(f4, CONFIGS[4]["job"], src4, scratch=scr, snapshot_every=1000)
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    out["config4_whole_job_2^21_shard"] = {"point_updates_per_s": nsh * CONFIGS[4]["job"] / t,
                                           "seconds": t}
    del f4, scr
    # config 3: K4, then the whole 20 000-step coupled job (split step)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    nz, ny, nx = 256, 512, 512
    n = nz * ny * nx
    job3 = 20000
    srcb = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=20e-6)
    segs = scanpath.serpentine((1e-3, 1e-3, 9.24e-3, 9.24e-3), 80e-6, 1.0, 0.35 * 250.0)
    beams = scanpath.beam_schedule(segs, job3, 1e-6)
    dom = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=20e-6, device=dev)
    k = [0]

    def timed(fn, reps):
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        return sorted(ts)[len(ts) // 2]

    def stencil():
        for _ in range(10):
            th.step_thermal(dom.field, 1e-6, th.DEFAULT_THERMAL, srcb, beams[k[0]], losses=False,
                            bottom_dirichlet=353.0, all_built=True)
    t = timed(stencil, 5) / 10
    out["stencil_K4_config3_grid"] = {
        "cells": n, "us": t * 1e6, "GB/s": 16 * n / t / 1e9,
        "frac_of_measured_hbm": 16 * n / t / 1e9 / hbm,
        "bytes_model": "16 B/cell (8 read T_n + 8 write T_n+1)", "pipeline": "TMA + mbarrier ring",
        "timing": "10 consecutive steps per event pair (inputs 1 GiB > L2)"}
    del dom
    dom = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=20e-6, device=dev)
    dom.run(1, 1e-6, beams, srcb)  # idle bits, scratch
    chunk = 5000
    ts = []
    s3 = 1
    while s3 < job3:
        m = min(chunk, job3 - s3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dom.run(m, 1e-6, beams[s3:], srcb)
        b.record()
        b.synchronize()
        ts.append((m, a.elapsed_time(b) * 1e-3))
        s3 += m
    tot = sum(x for _, x in ts)
    # end to end for a job whose fields start and end in host memory: the
    # state is uploaded once and downloaded once around the 20 000 steps
    pin = {k: torch.empty(getattr(dom.fields, k).shape, dtype=getattr(dom.fields, k).dtype,
                          pin_memory=True) for k in pkg.batch.NAMES}
    torch.cuda.synchronize()
    c0 = time.perf_counter()
    for k in pkg.batch.NAMES:
        pin[k].copy_(getattr(dom.fields, k), non_blocking=True)
    torch.cuda.synchronize()
    t_d2h = time.perf_counter() - c0
    up = {k: torch.empty_like(getattr(dom.fields, k)) for k in pkg.batch.NAMES}
    c0 = time.perf_counter()
    for k in pkg.batch.NAMES:
        up[k].copy_(pin[k], non_blocking=True)
    torch.cuda.synchronize()
    t_h2d = time.perf_counter() - c0
    bytes3 = sum(v.numel() * v.element_size() for v in pin.values())
    del up, pin
    h3 = dom.fields.to_host()
    cpu3 = None
    if not args.no_cpu_baseline:  # one full-grid step on the host (port)
        from oracle import oracle as orc
        from paper_2402_17580_b200 import _abi
        hf = orc.HostFields(h3["x_alpha_s"], h3["x_alpha_m"], h3["x_beta"],
                            h3["temperature_old"], h3["temperature_new"], h3["seed_tracked"],
                            h3["seed_active"], h3["seed_direction"])
        ones, built = np.ones((nz, ny, nx)), np.full((nz, ny, nx), 2, np.uint8)
        a3 = _abi.stencil_args(nx, ny, nz, nz, 1e-6, 20e-6, beam=beams[-1], source=srcb,
                               losses=False, bottom=353.0, all_built=True)
        from paper_2402_17580_b200.kinetics import DEFAULT_PARAMS
        from paper_2402_17580_b200.integrator import IntegratorConfig
        c0 = time.perf_counter()
        orc.stencil_step(hf.temperature_old.reshape(nz, ny, nx),
                         hf.temperature_new.reshape(nz, ny, nx), ones, built,
                         th.DEFAULT_THERMAL.kernel_tuple(), a3)
        orc.step_all(hf, 1e-6, DEFAULT_PARAMS.kernel_tuple(), IntegratorConfig().kernel_tuple(),
                     n_lanes=8, threads=cpu_threads())
        t_cpu = time.perf_counter() - c0
        cpu3 = {"value": n / t_cpu, "unit": "cell-steps/s", "cores": cpu_threads(),
                "kind": "port", "sample": "one full-grid 512x512x256 step at the job's end: "
                "oracle stencil_step (OpenMP over planes) + step_all (lanes=8)",
                "seconds": t_cpu}
    out["config3_whole_job"] = {
        "cells": n, "steps": job3, "seconds": tot, "ms_per_step": 1e3 * tot / (job3 - 1),
        "cell_steps_per_s": n * (job3 - 1) / tot,
        "ms_per_step_by_chunk": [1e3 * x / m for m, x in ts],
        "T_max_end": float(h3["temperature_old"].max()),
        "transformed_cells_end": int(np.count_nonzero(h3["x_alpha_s"] != 0.9)),
        "path": "split coupled step: K4 + hot-row bitmap, row scan, kinetics of listed rows",
        "roofline": {"bound": "hbm", "achieved": 16 * n * (job3 - 1) / tot / 1e9, "peak": hbm,
                     "unit": "GB/s", "frac": 16 * n * (job3 - 1) / tot / 1e9 / hbm,
                     "note": "16 B/cell-step (T_n read, T_n+1 written); the kinetics state of "
                             "idle rows is not touched (1/64 B/cell idle map)"},
        "e2e": {"value": n * (job3 - 1) / (tot + t_h2d + t_d2h), "unit": "cell-steps/s",
                "h2d_bytes_per_job": bytes3, "d2h_bytes_per_job": bytes3,
                "h2d_seconds": t_h2d, "d2h_seconds": t_d2h,
                "path": "fields uploaded once from pinned host memory, 20 000 coupled steps "
                        "on the device, fields downloaded once (copies timed on this box)"},
        "cpu_baseline": cpu3}
    del dom, flush, h3
    # K1 (one step_all) at 2^26 cold points: the HBM-bound per-step kernel
    n1 = 1 << 26
    f1 = pkg.GlobalFields.allocate(n1, temperature=300.0, device=dev)
    f1.x_alpha_s.fill_(0.9)
    f1.x_beta.fill_(0.1)
    pkg.step_all(f1, 1e-5)
    t = timed(lambda: pkg.step_all(f1, 1e-5), 5)
    out["K1_step_all_2^26"] = {"ms": t * 1e3, "GB/s": 73 * n1 / t / 1e9,
                               "frac_of_measured_hbm": 73 * n1 / t / 1e9 / hbm,
                               "bytes_model": "73 B/point-update (72 model + 1 seed flag)"}
    del f1
    # Crank-Nicolson step_all on the reference's block-100 benchmark layout
    cfg = pkg.IntegratorConfig(scheme="crank_nicolson", dt_sub_max=0.01)
    n = 1 << 22
    lay = branch_layout(100, n)
    pristine = pkg.GlobalFields(*lay, device=dev)
    it = pkg.step_all(pristine.copy(), 0.01, config=cfg, n_lanes=8, record_iters=True)
    mean_it = it.double().mean().item()
    work = [pristine.copy() for _ in range(5)]
    ts = []
    for w in work:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pkg.step_all(w, 0.01, config=cfg, n_lanes=8)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    t = sorted(ts)[len(ts) // 2]
    fl = reference_flops(lay[0], lay[1], lay[3], lay[4], 8, "crank_nicolson", mean_it)
    out["crank_nicolson_layout_block100_2^22"] = {
        "point_updates_per_s": n / t, "ms": t * 1e3, "mean_fixed_point_iters": mean_it,
        "reference_flops_per_point": fl / n, "TFLOP/s": fl / t / 1e12,
        "frac_of_fp64_peak": fl / t / 1e12 / peak_tf}
    return out


def run_b200(args):
    import torch
    import torch.distributed as dist
    import paper_2402_17580_b200 as pkg
    from paper_2402_17580_b200 import _lib

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.require()
    dd = Dist(world, dev)
    stream = torch.cuda.current_stream()
    peak = measure_fp64_peak(torch, lib, stream) / 1e12
    clk = ClockSampler(local)
    K, W = args.steps, args.warmup
    m = measure_ode(torch, pkg, HEADLINE, K, W, rank, world, dev, dd, clocks=clk,
                    cpu=not args.no_cpu_baseline, cpu_budget=args.cpu_budget)
    extra = None
    if world == 1 and not args.quick:
        extra = measure_extra(torch, pkg, dev, dd, peak, args)
    rl = roofline_of(m, peak, K)
    if rl is not None:
        rl.update({"peak_source": "measured on this box: DFMA stream (ti64_bench_dfma); "
                                  "MEASURED_PEAKS.json has no FP64 entry",
                   "kernel": "advance_kernel<PULSE_SWEEP> (K2), one launch per window",
                   "traffic": K2_PROFILE["dram_bytes_per_launch"],
                   "traffic_source": K2_PROFILE["file"],
                   "traffic_note": "state bytes are 92 B/point per launch (12.3 GB at 2^27); "
                                   "the rest is sector amplification of the 8-byte gathers / "
                                   "scatters in work-class order (each 32-byte sector is "
                                   "touched once per class present in it) and the per-thread "
                                   "pulse tables in local memory; 0.13 TB/s in total, far from "
                                   "the HBM bound (DESIGN.md §5.2)",
                   "executed": {k: K2_PROFILE[k] for k in ("fp64_pipe_active", "issue_active",
                                                            "fp64_inst_per_update")},
                   "ceiling_at_saturated_fp64_pipe": rl["flops_per_update"] /
                   (2.0 * K2_PROFILE["fp64_inst_per_update"]),
                   "ceiling_note": "the bit-exact instruction stream has fp64_inst_per_update "
                                   "FP64-pipe instructions per update, of which only the DFMAs "
                                   "carry two flops: frac cannot exceed flops_per_update / (2 x "
                                   "that) even with the FP64 pipe 100 % busy (DESIGN.md §5.2)",
                   "note": "achieved = the reference's flop model (SURVEY 8d F, from the "
                           "kernel's own branch counters over the timed windows) / mean "
                           "launch time; per GPU"})
    if rank == 0:
        c = CONFIGS[HEADLINE]
        line = {
            "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * m["t_max"] / K,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": config_dict(HEADLINE, world, K, W),
            "roofline": rl,
            "e2e": m.get("e2e"),
            "gpu_launches": m["launches"],
            "clocks": clk.summary(),
            "cpu_baseline": None if "cpu" not in m else
            {k: m["cpu"][k] for k in ("value", "unit", "cores", "kind", "sample")},
            "checks": {"counted_equals_timed_bitwise": m.get("counted_equals_timed"),
                       "cpu_sample_equals_gpu_bitwise":
                           m.get("cpu", {}).get("sample_equals_gpu_bitwise"),
                       "e2e_equals_device_bitwise":
                           (m.get("e2e") or {}).get("bitwise_equal_to_device_run"),
                       "totals": m.get("totals"), "sums_last": m["sums_last"],
                       "hist_checksum": m["hist_checksum"]},
            "timing": {"prep_seconds": m["prep_s"], "window_seconds": m["t_windows"],
                       "points_per_gpu": m["n_local"],
                       "job_estimate_seconds": m["t_max"] / K * c["job"] / c["window"]},
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_plumbing_test(args):
    """CPU (gloo) check of the multi-rank plumbing the GPU arm uses: spawn,
    shard tiling, sum/max all-reduce.  Prints one JSON line on rank 0."""
    import torch
    import torch.distributed as dist
    from paper_2402_17580_b200.distributed import shard_range
    rank, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        dist.init_process_group("gloo")
    n = CONFIGS[HEADLINE]["n"]
    lo, hi = shard_range(n, rank, world)
    t = torch.tensor([float(hi - lo), float(rank + 1)], dtype=torch.float64)
    mx = torch.tensor([float(rank)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    bounds = [shard_range(n, r, world) for r in range(world)]
    if rank == 0:
        print(json.dumps({"plumbing_test": True, "n_gpus": world, "shards": bounds,
                          "points_sum": t[0].item(), "rank_sum": t[1].item(),
                          "max_rank": mx.item()}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ref-check", action="store_true")
    ap.add_argument("--no-config3", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--quick", action="store_true", help="skip the secondary measurements")
    ap.add_argument("--plumbing-test", action="store_true", help=argparse.SUPPRESS)
    argv = sys.argv[1:]
    args = ap.parse_args(argv)
    if args.warmup < 0 or args.steps < 1:
        raise SystemExit("need --steps >= 1 and --warmup >= 0")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus, argv)
    if args.plumbing_test:
        return run_plumbing_test(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
