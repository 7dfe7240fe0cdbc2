"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ti64micro from /root/reference/pkg/src (numba, read-only tree;
NUMBA_CACHE_DIR is pointed at /tmp) and records inputs and outputs of the
reference's own entry points:

  fastmath.npz   fast_exp / fast_ln / fast_pow on sweeps + special values
                 (fastmath.py:246-258)
  steps.npz      step_all cases (batch.py:762): the reference's own test
                 fixtures (conftest.random_states, bench.generate_layout,
                 alternating hot/cold, N=13 tail, identical points),
                 stuck-state seeding sequences, subcycling; every lane width
  advance_cfg*.npz  multi-step runs where temperature_new is filled each step
                 from this project's generator definitions (computed by the
                 oracle's generator) and the kinetics are the
                 reference's step_all; counters per DESIGN.md §3 in numpy
  history.npz    integrate_history (integrator.py:303-325)
  stencil.npz    thermal._stencil_step via step_thermal (thermal.py:321-354)
  cn_steps.npz, cn_history.npz  Crank-Nicolson step_all / integrate_history
  acceptance.npz the reference's acceptance-criterion quantities
                 (test_acceptance.py), incl. the coupled cube builds
  initiation.npz initiate_diffusion sequences (integrator.py:214-265)
  kinetics_api.npz  kinetics.py model functions + fastmath estrin/horner
  report.npz     bench.count_flops / RooflineReport text, output.py VTK
                 snapshots and probe CSV of a micro build
  build.npz      thermal.run_build on the reference's micro build
                 (test_thermal.py:33-43, :192-200): final thermal field, all
                 kinetics arrays, probe rows, for several scan strategies /
                 schemes / powers

The GPU box never runs this script (no /root/reference there); tests read
only the committed .npz files.
"""

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ti64_numba_cache")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(ROOT))

from ti64micro import fastmath as fm  # noqa: E402
from ti64micro.batch import GlobalFields, step_all  # noqa: E402
from ti64micro.bench import generate_layout  # noqa: E402
from ti64micro.integrator import IntegratorConfig, integrate_history  # noqa: E402
from ti64micro.kinetics import DEFAULT_PARAMS  # noqa: E402
from ti64micro import thermal as th  # noqa: E402
from conftest import random_states  # noqa: E402

from oracle import oracle as orc  # noqa: E402  (generator definitions only)
from paper_2402_17580_b200 import sources  # noqa: E402

CFG_E = IntegratorConfig(scheme="explicit")
NAMES = ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old",
         "temperature_new", "seed_tracked", "seed_active", "seed_direction")


def fields_dict(f, prefix):
    return {f"{prefix}{k}": np.array(getattr(f, k)) for k in NAMES}


def make_fastmath():
    rng = np.random.default_rng(101)
    special = np.array([0.0, 1.0, -1.0, -1.36, -750.0, 800.0, np.nan, -708.0,
                        -708.0000001, 709.0, 709.0000001, 1e-300, -1e-300,
                        -707.9, 708.9, np.inf, -np.inf, 0.5, -0.5, 1e-20])
    x_exp = np.concatenate([special, np.linspace(-700.0, 709.0, 20001),
                            rng.uniform(-60, 5, 20000)])
    special_ln = np.array([1.0, np.e, 2.0, 0.0, -1.0, np.nan, 1e-310, 5e-324,
                           2.2250738585072014e-308, 1e-300, 1e300, np.inf,
                           0.9, 1e-14, 0.1, 0.09999999999999998])
    x_ln = np.concatenate([special_ln,
                           np.exp(np.linspace(np.log(1e-300), np.log(1e300), 20001)),
                           1.0 + np.linspace(-1e-3, 1e-3, 2001),
                           rng.uniform(0, 1, 20000)])
    a = np.concatenate([[0.25, 0.9, 1.0, -1.0, 1e-300, 0.0],
                        10.0 ** rng.uniform(-12, 0, 20000)])
    p = np.concatenate([[0.5, 1.0, 1.398, 2.0, 0.6015936254980079, 1.0],
                        rng.uniform(0.0, 2.0, 20000)])
    np.savez_compressed(OUT / "fastmath.npz", x_exp=x_exp, y_exp=fm.fast_exp(x_exp),
                        x_ln=x_ln, y_ln=fm.fast_ln(x_ln), a_pow=a, x_pow=p,
                        y_pow=fm.fast_pow(a, p))


def seeding_fields():
    """Stuck compositions and neighbours at temperatures that trigger and end
    both seeding directions (batch.py:419-464)."""
    temps = [300.0, 600.0, 847.0, 848.0, 900.0, 934.0, 935.001, 1000.0, 1100.0,
             1200.0, 1272.0, 1273.5, 1300.0, 1877.0, 1880.0, 1930.0]
    states = [(0.9, 0.0, 0.1), (0.9, 0.0, 0.09999999999999998), (0.0, 0.0, 1.0),
              (0.0, 0.0, 0.99), (1e-15, 0.0, 1.0), (0.9 - 5e-15, 0.0, 0.1),
              (0.9, 1e-15, 0.1), (0.45, 0.0, 0.55), (0.0, 0.3, 0.7)]
    xs, xm, xb, t0, t1 = [], [], [], [], []
    for (a, b, c) in states:
        for ta in temps:
            for dT in (0.0, 5.0, -5.0):
                xs.append(a), xm.append(b), xb.append(c)
                t0.append(ta), t1.append(ta + dT)
    return GlobalFields(np.array(xs), np.array(xm), np.array(xb), np.array(t0),
                        np.array(t1))


def run_steps(f, dt, lanes, nsteps=1, threads=1, vary=None):
    for s in range(nsteps):
        if vary is not None:
            f.temperature_new[:] = vary(s)
        step_all(f, dt, DEFAULT_PARAMS, CFG_E, n_lanes=lanes, threads=threads)


def make_steps():
    cases = {}

    def add(name, f, dt, lanes, nsteps=1, threads=1, vary=None):
        d = fields_dict(f, "in_")
        g = f.copy()
        run_steps(g, dt, lanes, nsteps, threads, vary)
        d.update(fields_dict(g, "out_"))
        d["dt"] = np.float64(dt)
        d["lanes"] = np.int64(lanes)
        d["nsteps"] = np.int64(nsteps)
        if vary is not None:
            d["t_seq"] = np.stack([vary(s) for s in range(nsteps)])
        for k, v in d.items():
            cases[f"{name}/{k}"] = v

    for lanes in (1, 2, 4, 8):
        add(f"random257_l{lanes}", random_states(257, seed=3), 2e-5, lanes)
    add("random4099_thr2", random_states(4099, seed=9), 2e-5, 8, threads=2)
    add("tail13_l8", random_states(13, seed=6), 2e-5, 8)
    add("tail13_l1", random_states(13, seed=6), 2e-5, 1)
    n = 64
    xs = np.where(np.arange(n) % 2 == 0, 0.2, 0.8)
    t = np.where(np.arange(n) % 2 == 0, 1000.0, 1150.0)
    add("alternating_l8", GlobalFields(xs, np.zeros(n), 1.0 - xs, t, t + 1.0), 2e-5, 8)
    for block in (1, 10, 100):
        add(f"layout_b{block}", generate_layout(block, 4096, seed=block), 0.01, 8)
        add(f"layout_b{block}_dt2e-5", generate_layout(block, 4096, seed=block), 2e-5, 8)
    m = 1000
    add("identical", GlobalFields(np.full(m, 0.3), np.full(m, 0.1), np.full(m, 0.6),
                                  np.full(m, 1000.0), np.full(m, 995.0)), 2e-5, 8)
    add("sub_dt0.05", random_states(32, seed=12, dt_jitter=0.0), 0.05, 8)
    add("sub_dt0.05_jit", random_states(32, seed=11), 0.05, 8)
    add("sub_dt0.01", random_states(32, seed=12, dt_jitter=0.0), 0.01, 8)
    add("sub_dt1.0", random_states(64, seed=15), 1.0, 4)
    add("hot_liquid", random_states(200, seed=16, t_lo=1800.0, t_hi=3000.0), 1e-4, 8)
    add("cold", random_states(200, seed=17, t_lo=293.0, t_hi=900.0), 1e-4, 8)
    for lanes in (1, 8):
        add(f"seed_1step_l{lanes}", seeding_fields(), 1e-4, lanes)
        sf = seeding_fields()
        base_t0 = sf.temperature_old.copy()
        add(f"seed_40step_l{lanes}", sf, 1e-3, lanes, nsteps=40,
            vary=lambda s, b=base_t0: b + 3.0 * np.sin(0.3 * s) * (np.arange(len(b)) % 3))
    np.savez_compressed(OUT / "steps.npz", **cases)


def make_cn():
    """Crank-Nicolson step_all cases (batch.py:357-416, halving :568-674)."""
    from ti64micro.batch import BatchConvergenceError
    CFG_I = IntegratorConfig(scheme="crank_nicolson")
    cases = {}

    def add(name, f, dt, lanes, cfg, nsteps=1, vary=None):
        d = fields_dict(f, "in_")
        g = f.copy()
        fail = np.array([], np.int64)
        iters = None
        for s in range(nsteps):
            if vary is not None:
                g.temperature_new[:] = vary(s)
            try:
                iters = step_all(g, dt, DEFAULT_PARAMS, cfg, n_lanes=lanes, record_iters=True)
            except BatchConvergenceError as e:
                fail = np.array(e.indices, np.int64)
                break
        d.update(fields_dict(g, "out_"))
        d["dt"] = np.float64(dt)
        d["lanes"] = np.int64(lanes)
        d["nsteps"] = np.int64(nsteps)
        d["fail"] = fail
        d["iters"] = np.zeros(0, np.int64) if iters is None else np.asarray(iters, np.int64)
        d["cfg"] = np.array([cfg.dt_sub_max, cfg.eps_abs, cfg.eps_rel,
                             cfg.max_fixed_point_iters, cfg.initiation_threshold,
                             cfg.stuck_tol, cfg.max_halvings], np.float64)
        if vary is not None:
            d["t_seq"] = np.stack([vary(s) for s in range(nsteps)])
        for k, v in d.items():
            cases[f"{name}/{k}"] = v

    for lanes in (1, 2, 4, 8):
        add(f"cn_random257_l{lanes}", random_states(257, seed=4), 0.01, lanes, CFG_I)
    add("cn_tail13_l8", random_states(13, seed=6), 0.01, 8, CFG_I)
    add("cn_sub_dt0.05", random_states(32, seed=12), 0.05, 8, CFG_I)
    add("cn_sub_dt1.0", random_states(64, seed=15), 1.0, 4, CFG_I)
    tight = IntegratorConfig(scheme="crank_nicolson", eps_abs=1e-18, eps_rel=1e-8)
    for lanes in (1, 8):
        add(f"cn_tight_l{lanes}", random_states(257, seed=5), 0.1, lanes, tight)
        add(f"cn_tight_dt2e-5_l{lanes}", random_states(257, seed=7), 2e-5, lanes, tight)
    few = IntegratorConfig(scheme="crank_nicolson", max_fixed_point_iters=3, max_halvings=2,
                           eps_abs=1e-16, eps_rel=1e-9)
    for lanes in (1, 4, 8):
        add(f"cn_halving_l{lanes}", random_states(120, seed=19, t_lo=800.0, t_hi=1300.0),
            0.01, lanes, few)
    halv = IntegratorConfig(scheme="crank_nicolson", eps_abs=1e-18, eps_rel=1e-8,
                            max_fixed_point_iters=6, max_halvings=5, dt_sub_max=1.0)
    for lanes in (1, 2, 8):
        add(f"cn_halving2_l{lanes}", random_states(96, seed=23), 0.3, lanes, halv)
    halv_fail = IntegratorConfig(scheme="crank_nicolson", eps_abs=1e-18, eps_rel=1e-8,
                                 max_fixed_point_iters=6, max_halvings=1, dt_sub_max=1.0)
    for lanes in (1, 8):
        add(f"cn_halving_fail_l{lanes}", random_states(96, seed=23), 0.3, lanes, halv_fail)
    bad = IntegratorConfig(scheme="crank_nicolson", max_fixed_point_iters=1, max_halvings=0,
                           dt_sub_max=1.0)
    add("cn_fail_l8", random_states(40, seed=10, t_lo=950.0, t_hi=1100.0, dt_jitter=0.0),
        1.0, 8, bad)
    for lanes in (1, 8):
        sf = seeding_fields()
        base_t0 = sf.temperature_old.copy()
        add(f"cn_seed_40step_l{lanes}", sf, 1e-3, lanes, CFG_I, nsteps=40,
            vary=lambda s, b=base_t0: b + 3.0 * np.sin(0.3 * s) * (np.arange(len(b)) % 3))
    add("cn_layout_b10", generate_layout(10, 4096, seed=10), 0.01, 8, CFG_I)
    np.savez_compressed(OUT / "cn_steps.npz", **cases)
    hist = {}
    rng = np.random.default_rng(44)
    for h in range(4):
        knots_t = np.concatenate([[0.0], np.sort(rng.uniform(0.1, 6.0, 5))])
        knots_T = rng.uniform(293.0, 2000.0, 6)
        times = np.linspace(0.0, knots_t[-1], 1500 if h % 2 == 0 else 60)
        temps = np.interp(times, knots_t, knots_T)
        hist[f"h{h}/times"] = times
        hist[f"h{h}/temps"] = temps
        hist[f"h{h}/out"] = integrate_history(times, temps, config=CFG_I)
    times = np.arange(0.0, 400.0, 1.0)
    hist["const1000/times"] = times
    hist["const1000/temps"] = np.full_like(times, 1000.0)
    from ti64micro.kinetics import PhaseState
    hist["const1000/out"] = integrate_history(times, hist["const1000/temps"],
                                              state0=PhaseState(0.0, 0.0, 1.0), config=CFG_I)
    np.savez_compressed(OUT / "cn_history.npz", **hist)


def argmax3(xs, xm, xb):
    return np.where((xs >= xm) & (xs >= xb), 0, np.where(xm >= xb, 1, 2))


def make_advance(cfg_id, n, nsteps, snap_every, lanes=8, point_offset=0, src=None,
                 name=None):
    """Reference step_all driven by the project's generator."""
    src = src or sources.source_for_config(cfg_id)
    beam = src.beam_table(nsteps + 1) if cfg_id == 1 else None
    gen = src.tempgen(point_offset=point_offset,
                      beam_ptr=None if beam is None else beam.ctypes.data,
                      beam_steps=0 if beam is None else len(beam))
    init = orc.gen_initial_state(gen, n)
    t0 = orc.gen_temperature(gen, n, 0)
    f = GlobalFields(init.x_alpha_s, init.x_alpha_m, init.x_beta, t0, t0.copy())
    kp = DEFAULT_PARAMS.kernel_tuple()
    mart = np.zeros(n, np.uint32)
    sw = np.zeros(n, np.uint32)
    tot = np.zeros(8, np.uint64)
    sums = []
    for s in range(nsteps):
        f.temperature_new[:] = orc.gen_temperature(gen, n, s + 1)
        xs, xm, xb = f.x_alpha_s.copy(), f.x_alpha_m.copy(), f.x_beta.copy()
        xa = xs + xm
        ramp = 1.0 - fm.fast_exp(-kp.k_alpha_eq * (kp.t_as_start - f.temperature_old))
        xe0 = np.where(f.temperature_old < kp.t_as_end, 0.9,
                       np.where(f.temperature_old > kp.t_as_start, 0.0, ramp))
        grow = (xa < xe0) & (xs > 0.0)
        am = (xm > 0.0) & (xs > 0.0)
        dis = (xa > xe0) & (xa < 0.9)
        tot[0] += n
        tot[1] += int((f.temperature_new < kp.t_am_start).sum())
        tot[2] += int((grow | am).sum())
        tot[3] += int(grow.sum())
        tot[4] += int(am.sum())
        tot[5] += int(dis.sum())
        a0 = argmax3(xs, xm, xb)
        step_all(f, src.dt, DEFAULT_PARAMS, CFG_E, n_lanes=lanes)
        m = f.x_alpha_m > xm
        w = argmax3(f.x_alpha_s, f.x_alpha_m, f.x_beta) != a0
        mart += m.astype(np.uint32)
        sw += w.astype(np.uint32)
        tot[6] += int(m.sum())
        tot[7] += int(w.sum())
        if (snap_every > 0 and (s + 1) % snap_every == 0) or s + 1 == nsteps:
            sums.append([f.x_alpha_s.sum(), f.x_alpha_m.sum(), f.x_beta.sum()])
    out = dict(cfg=np.int64(cfg_id), n=np.int64(n), nsteps=np.int64(nsteps),
               snap_every=np.int64(snap_every), lanes=np.int64(lanes),
               point_offset=np.int64(point_offset), martensite=mart, switches=sw,
               totals=tot, sums=np.array(sums))
    out.update(fields_dict(f, "out_"))
    np.savez_compressed(OUT / (name or f"advance_cfg{cfg_id}.npz"), **out)


def make_history():
    rng = np.random.default_rng(33)
    cases = {}
    for h in range(6):
        knots_t = np.concatenate([[0.0], np.sort(rng.uniform(0.1, 6.0, 5))])
        knots_T = rng.uniform(293.0, 2000.0, 6)
        times = np.linspace(0.0, knots_t[-1], 1500 if h % 2 == 0 else 150)
        temps = np.interp(times, knots_t, knots_T)
        out = integrate_history(times, temps, config=CFG_E)
        cases[f"h{h}/times"] = times
        cases[f"h{h}/temps"] = temps
        cases[f"h{h}/out"] = out
    times = np.arange(0.0, 10.0 + 1e-9, 1e-3)
    temps = 1300.0 + (300.0 - 1300.0) * times / 10.0
    cases["ramp/times"], cases["ramp/temps"] = times, temps
    cases["ramp/out"] = integrate_history(times, temps, config=CFG_E)
    np.savez_compressed(OUT / "history.npz", **cases)


def make_stencil():
    cases = {}
    tp = th.DEFAULT_THERMAL
    # (a) general: plate + powder + inactive, losses on, source on, Dirichlet
    geo = th.BuildGeometry(plate_size=(0.6e-3, 0.6e-3, 0.15e-3),
                           part_size=(0.4e-3, 0.4e-3, 0.1e-3), voxel=0.05e-3)
    sched = th.BuildSchedule()
    field, fields = th.allocate_domain(geo, sched)
    th.activate_layer(field, fields, geo, sched)
    rng = np.random.default_rng(5)
    field.temperature_old[:] = 293.0 + rng.uniform(0, 2500.0, field.temperature_old.shape)
    field.temperature_old[field.state == 0] = 293.0
    src = th.HeatSource(w_eff=180.0, radius=0.06e-3, h_powder=geo.voxel)
    cases["general/src"] = field.temperature_old.copy()
    cases["general/rc_in"] = field.r_c.copy()
    cases["general/state"] = field.state.copy()
    cases["general/z_top"] = np.int64(field.z_top)
    cases["general/h"] = np.float64(field.h)
    dt = 2e-6
    beam = (0.3e-3, 0.28e-3, 180.0, True)
    th.step_thermal(field, dt, tp, src, beam, losses=True, bottom_dirichlet=293.0, nsub=1)
    cases["general/dst"] = field.temperature_new.copy()
    cases["general/rc_out"] = field.r_c.copy()
    cases["general/dt"] = np.float64(dt)
    cases["general/beam"] = np.array(beam[:3])
    cases["general/src_peak"] = np.float64(2.0 * 180.0 / (np.pi * src.radius**2 * src.h_powder))
    cases["general/src_r2inv"] = np.float64(1.0 / src.radius**2)
    # (b) all built (config-3 shape, reduced): chained steps with a moving source
    nz, ny, nx = 8, 16, 16
    h = 20e-6
    t_old = np.full((nz, ny, nx), 353.0)
    t_new = t_old.copy()
    f2 = th.ThermalField(t_old, t_new, np.ones((nz, ny, nx)),
                         np.full((nz, ny, nx), th.STATE_BUILT, np.uint8), h, nz)
    src2 = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=h)
    seq = []
    for k in range(12):
        bx = 40e-6 + 20e-6 * k
        by = 150e-6
        th.step_thermal(f2, 1e-6, tp, src2, (bx, by, 0.35 * 250.0, True), losses=False,
                        bottom_dirichlet=353.0, nsub=1)
        seq.append(f2.temperature_new.copy())
        f2.temperature_old[...] = f2.temperature_new
    cases["built/seq"] = np.stack(seq)
    np.savez_compressed(OUT / "stencil.npz", **cases)


def make_build():
    """run_build (thermal.py:498-589) on the reference tests' micro geometry."""
    from ti64micro.scanpath import ScanPath, serpentine, four_islands
    MM = 1e-3
    geom = th.BuildGeometry(plate_size=(0.6 * MM, 0.6 * MM, 0.15 * MM),
                            part_size=(0.4 * MM, 0.4 * MM, 0.1 * MM), voxel=0.05 * MM)
    cases = {}

    def run(name, power, strategy, cfg=None, **kw):
        base = dict(dt_active=2e-5, interlayer_dwell=0.02, initial_dwell_steps=50,
                    final_cooldown=1.0, preheat=293.0)
        base.update(kw)
        sched = th.BuildSchedule(**base)
        segs = []
        for layer in range(geom.grid[3]):
            segs.extend(strategy(geom.part_extent, 0.08 * MM, 0.96, power, layer))
        scan = ScanPath(segs, dwell=sched.interlayer_dwell)
        field, fields, probes = th.run_build(
            geom, scan, sched, integrator_config=cfg,
            probe_points=[(0.3 * MM, 0.3 * MM, 0.17 * MM), (0.1 * MM, 0.2 * MM, 0.05 * MM)])
        d = {f"{name}/{k}": np.array(getattr(fields, k)) for k in NAMES}
        d[f"{name}/r_c"] = np.array(field.r_c)
        d[f"{name}/state"] = np.array(field.state)
        d[f"{name}/z_top"] = np.int64(field.z_top)
        for i in range(2):
            d[f"{name}/probe{i}"] = np.array(probes[i], dtype=np.float64).reshape(-1, 5)
        d[f"{name}/power"] = np.float64(power)
        d[f"{name}/strategy"] = np.array(strategy.__name__)
        d[f"{name}/scheme"] = np.array("explicit" if cfg is None else cfg.scheme)
        d[f"{name}/sched"] = np.array([sched.dt_active, sched.interlayer_dwell,
                                       sched.initial_dwell_steps, sched.growth_every,
                                       sched.dt_max, sched.final_cooldown, sched.preheat,
                                       sched.room])
        cases.update(d)

    for dur, init, dtmax in ((0.02, 50, 0.1), (1.0, 0, 0.1), (100.0, 2000, 0.1), (0.3, 7, 0.05)):
        sc = th.BuildSchedule(dt_max=dtmax)
        cases[f"cooldown/{dur}_{init}_{dtmax}"] = np.array(th._cooldown_steps(dur, sc, init))
    rng = np.random.default_rng(11)
    t = np.concatenate([rng.uniform(250.0, 5000.0, 200), [1878.0, 1903.0, 1928.0, 3130.0, 4130.0, 4500.0]])
    rc = rng.uniform(0.0, 1.0, t.size)
    cases["helpers/t"] = t
    cases["helpers/rc"] = rc
    cases["helpers/conductivity"] = th.conductivity(t, rc)
    powder = rng.uniform(size=t.size) < 0.5
    cases["helpers/powder"] = powder
    cases["helpers/update_consolidation"] = th.update_consolidation(rc, t, powder)
    cases["helpers/surface_losses"] = th.surface_losses(t)
    x = rng.uniform(0.0, 1e-3, 300)
    y = rng.uniform(0.0, 1e-3, 300)
    zb = rng.uniform(0.0, 1e-4, 300)
    cases["helpers/x"], cases["helpers/y"], cases["helpers/zb"] = x, y, zb
    cases["helpers/source_term"] = th.source_term(x, y, zb, 4e-4, 5e-4)
    g = th.BuildGeometry()
    cases["geometry/default_grid"] = np.array(g.grid)
    cases["geometry/default_part_box"] = np.array(g.part_box)
    cases["geometry/default_part_extent"] = np.array(g.part_extent)
    run("serp180", 180.0, serpentine)
    run("islands150", 150.0, four_islands, preheat=400.0)
    run("zero", 0.0, serpentine)
    run("serp180_cn", 180.0, serpentine, cfg=IntegratorConfig(scheme="crank_nicolson"),
        final_cooldown=0.3)
    np.savez_compressed(OUT / "build.npz", **cases)


def make_report():
    """bench.count_flops / RooflineReport (bench.py:158-257) and the output
    writers (output.py) on reference states."""
    import tempfile
    from ti64micro import bench as rb, output as ro
    from ti64micro.scanpath import ScanPath, serpentine
    cases = {}
    for block in (1, 10, 100):
        lay = generate_layout(block, 1000 + block, seed=block)
        for k in NAMES[:5]:
            cases[f"layout{block}/{k}"] = np.array(getattr(lay, k))
        for lanes in (1, 8):
            cases[f"layout{block}/flops_explicit_l{lanes}"] = np.int64(
                rb.count_flops(lay, "explicit", lanes))
        it = np.arange(lay.n_points) % 5
        cases[f"layout{block}/iters"] = it
        cases[f"layout{block}/flops_cn_l8"] = np.int64(
            rb.count_flops(lay, "crank_nicolson", 8, iters=it))
    runs = [dict(label="explicit_b1", flops=123456789, bytes=72 * 400000, seconds=0.0123),
            dict(label="cn_b100", flops=987654321, bytes=72 * 400000, seconds=0.0456)]
    rep = rb.roofline(runs, measured_bandwidth=6538.0, peak_flops=34120.5,
                      instruction_mix_factor=0.57)
    cases["roofline/csv"] = np.array(rep.to_csv())
    cases["roofline/gnuplot"] = np.array(rep.to_gnuplot())
    cases["roofline/respects"] = np.array(rep.respects_ceilings())
    cases["roofline/mem_dof"] = np.float64(rep.memory_bound_dof_rate)
    MM = 1e-3
    geom = th.BuildGeometry(plate_size=(0.6 * MM, 0.6 * MM, 0.15 * MM),
                            part_size=(0.4 * MM, 0.4 * MM, 0.1 * MM), voxel=0.05 * MM)
    sched = th.BuildSchedule(dt_active=2e-5, interlayer_dwell=0.02, initial_dwell_steps=50,
                             final_cooldown=0.05, preheat=293.0)
    segs = []
    for layer in range(geom.grid[3]):
        segs.extend(serpentine(geom.part_extent, 0.08 * MM, 0.96, 180.0, layer))
    scan = ScanPath(segs, dwell=sched.interlayer_dwell)
    snaps = {}

    def hook(label, t, field, fields):
        with tempfile.NamedTemporaryFile("r", suffix=".vtk") as tf:
            ro.write_vtk_snapshot(tf.name, field, fields, label=label)
            snaps[label] = open(tf.name).read()

    field, fields, probes = th.run_build(geom, scan, sched, snapshot_hook=hook,
                                         probe_points=[(0.3 * MM, 0.3 * MM, 0.17 * MM)])
    for label, text in snaps.items():
        cases[f"vtk/{label}"] = np.array(text)
    with tempfile.NamedTemporaryFile("r", suffix=".csv") as tf:
        ro.write_probe_csv(tf.name, probes[0])
        cases["csv/probe0"] = np.array(open(tf.name).read())
    cases["sched"] = np.array([sched.dt_active, sched.interlayer_dwell,
                               sched.initial_dwell_steps, sched.growth_every, sched.dt_max,
                               sched.final_cooldown, sched.preheat, sched.room])
    np.savez_compressed(OUT / "report.npz", **cases)


def make_kinetics_api():
    """kinetics.py:144-269 model functions and fastmath estrin/horner helpers
    on seeded inputs (scalars and arrays)."""
    from ti64micro import kinetics as rk
    from ti64micro.fastmath import estrin_eval, horner_eval, EXP_CORRECTION, LN_CORRECTION
    rng = np.random.default_rng(5)
    t = np.concatenate([rng.uniform(250.0, 2100.0, 400),
                        [848.0, 935.0, 1273.0, 1373.0, 1878.0, 1928.0, 850.0, 300.0]])
    xs = rng.uniform(-0.05, 0.95, t.size)
    xm = rng.uniform(-0.05, 0.9, t.size)
    xs[:20] = 0.0
    xm[20:40] = 0.0
    c = {"t": t, "xs": xs, "xm": xm}
    c["liquid_fraction"] = rk.liquid_fraction(t)
    c["solid_fraction"] = rk.solid_fraction(t)
    c["x_alpha_eq"] = rk.x_alpha_eq(t)
    c["x_alpha_m_eq"] = rk.x_alpha_m_eq(t, xs)
    c["k_as"], c["k_b"] = rk.diffusion_rate_k(t)
    r = rk.compute_rates((xs, xm), t)
    c["ds"], c["dm"] = r.d_x_alpha_s, r.d_x_alpha_m
    st = rk.apply_corrections((xs, xm), t)
    c["cxs"], c["cxm"], c["cxb"] = st.x_alpha_s, st.x_alpha_m, st.x_beta
    sc = [(0.3, 0.2, 950.0), (0.0, 0.0, 1000.0), (0.9, 0.0, 1200.0), (0.5, 0.4, 700.0)]
    c["scalar_in"] = np.array(sc)
    out = []
    for a, b, tt in sc:
        rr = rk.compute_rates(rk.PhaseState(a, b, 0.0), tt)
        cc = rk.apply_corrections(rk.PhaseState(a, b, 0.0), tt)
        out.append([rr.d_x_alpha_s, rr.d_x_alpha_m, cc.x_alpha_s, cc.x_alpha_m, cc.x_beta,
                    rk.x_alpha_eq(tt), rk.liquid_fraction(tt)])
    c["scalar_out"] = np.array(out)
    y = rng.uniform(0.0, 1.0, 100)
    c["y"] = y
    c["estrin_exp"] = estrin_eval(EXP_CORRECTION, y)
    c["estrin_ln"] = estrin_eval(LN_CORRECTION, y)
    c["estrin_odd"] = estrin_eval((1.0, -0.5, 0.25, 0.125, -1.5), y)
    c["horner_ln"] = horner_eval(LN_CORRECTION, y)
    np.savez_compressed(OUT / "kinetics_api.npz", **c)


def make_acceptance():
    """The reference's acceptance-criterion quantities (test_acceptance.py:51-361)
    computed by the reference itself; the GPU suite reproduces them."""
    import math
    from ti64micro import fastmath as rfm
    from ti64micro.integrator import analytic_beta_growth
    from ti64micro.kinetics import PhaseState, liquid_fraction
    from ti64micro.scanpath import ScanPath, serpentine, four_islands
    CFG_I = IntegratorConfig(scheme="crank_nicolson")
    c = {}
    # 2: lane equivalence of the implicit scheme (max deviation vs 1 lane)
    base = random_states(10_000, seed=21)
    ref = base.copy()
    step_all(ref, 0.01, DEFAULT_PARAMS, CFG_I, n_lanes=1)
    c["c2_ref_states"] = ref.states()
    for lanes in (2, 4, 8):
        f = base.copy()
        step_all(f, 0.01, DEFAULT_PARAMS, CFG_I, n_lanes=lanes)
        c[f"c2_states_l{lanes}"] = f.states()
    c["c2_in"] = np.stack([base.x_alpha_s, base.x_alpha_m, base.x_beta,
                           base.temperature_old, base.temperature_new])
    # 3: continuity over 100 seeded histories, both schemes
    rng = np.random.default_rng(33)
    worst = 0.0
    for _ in range(100):
        knots_t = np.concatenate([[0.0], np.sort(rng.uniform(0.1, 6.0, 5))])
        knots_T = rng.uniform(293.0, 2000.0, 6)
        times = np.linspace(0.0, knots_t[-1], 1500)
        temps = np.interp(times, knots_t, knots_T)
        for cfg in (CFG_E, CFG_I):
            out = integrate_history(times, temps, config=cfg)
            worst = max(worst, float(np.abs(out.sum(axis=1) - (1.0 - liquid_fraction(temps))).max()))
    c["c3_worst"] = np.float64(worst)
    # 4: equilibrium convergence under CN holds
    finals = []
    for t_hold in (1000.0, 1100.0, 1200.0):
        times = np.arange(0.0, 10_000.0 + 0.5, 1.0)
        temps = np.full_like(times, t_hold)
        out = integrate_history(times, temps, state0=PhaseState(0.0, 0.0, 1.0), config=CFG_I)
        finals.append(out[-1])
    c["c4_finals"] = np.array(finals)
    # 5: Appendix-A closed form
    for scheme, dt in (("explicit", 1e-4), ("crank_nicolson", 1e-2)):
        n = int(round(1000.0 / dt))
        times = dt * np.arange(n + 1)
        temps = np.full(n + 1, 1200.0)
        out = integrate_history(times, temps, state0=PhaseState(0.9, 0.0, 0.1),
                                config=IntegratorConfig(scheme=scheme))
        _, exact = analytic_beta_growth(1200.0, dt, n)
        c[f"c5_{scheme}_err"] = np.float64(np.abs(out[1:, 2] - exact).max())
        c[f"c5_{scheme}_xb_tail"] = out[-1000:, 2]
    # 6: explicit (1e-5) vs CN (1e-3) along a 10 s cooling ramp
    t_end = 10.0
    times_e = np.arange(0.0, t_end + 1e-9, 1e-5)
    temps_e = 1300.0 + (300.0 - 1300.0) * times_e / t_end
    out_e = integrate_history(times_e, temps_e, config=CFG_E)
    times_i = np.arange(0.0, t_end + 1e-9, 1e-3)
    temps_i = 1300.0 + (300.0 - 1300.0) * times_i / t_end
    out_i = integrate_history(times_i, temps_i, config=CFG_I)
    checks = np.linspace(0.1, 10.0, 100)
    c["c6_e"] = out_e[np.searchsorted(times_e, checks)]
    c["c6_i"] = out_i[np.searchsorted(times_i, checks)]
    # 7 / 8: the coupled cube builds
    MM = 1e-3

    def cube(geometry, strategy, schedule):
        segs = []
        for layer in range(geometry.grid[3]):
            segs.extend(strategy(geometry.part_extent, 0.08 * MM, 0.96, 180.0, layer))
        scan = ScanPath(segs, dwell=schedule.interlayer_dwell)
        source = th.HeatSource(w_eff=180.0, radius=0.06 * MM, h_powder=geometry.voxel)
        return th.run_build(geometry, scan, schedule, source=source)

    g7 = th.BuildGeometry(plate_size=(1.2 * MM, 1.2 * MM, 0.2 * MM),
                          part_size=(1.0 * MM, 1.0 * MM, 0.25 * MM), voxel=0.05 * MM)
    s7 = th.BuildSchedule(dt_active=2e-5, interlayer_dwell=1.0, initial_dwell_steps=2000,
                          final_cooldown=20.0, preheat=293.0)
    f7, k7, _ = cube(g7, serpentine, s7)
    for k in NAMES:
        c[f"c7_{k}"] = np.array(getattr(k7, k))
    c["c7_r_c"], c["c7_state"] = np.array(f7.r_c), np.array(f7.state)
    g8 = th.BuildGeometry(plate_size=(1.0 * MM, 1.0 * MM, 3.0 * MM),
                          part_size=(1.0 * MM, 1.0 * MM, 1.0 * MM), voxel=0.05 * MM)
    s8 = th.BuildSchedule(dt_active=2e-5, interlayer_dwell=0.35, initial_dwell_steps=500,
                          final_cooldown=10.0, preheat=600.0)
    for name, strat in (("single", serpentine), ("islands", four_islands)):
        f8, k8, _ = cube(g8, strat, s8)
        c[f"c8_{name}_xs"] = np.array(k8.x_alpha_s)
        c[f"c8_{name}_xm"] = np.array(k8.x_alpha_m)
        c[f"c8_{name}_r_c"] = np.array(f8.r_c)
        c[f"c8_{name}_state"] = np.array(f8.state)
        c[f"c8_{name}_T"] = np.array(f8.temperature_old)
    np.savez_compressed(OUT / "acceptance.npz", **c)


def make_initiation():
    """integrator.initiate_diffusion (integrator.py:214-265) sequences."""
    from ti64micro.integrator import initiate_diffusion, SeedingState
    from ti64micro.kinetics import PhaseState
    c = {}
    seqs = {"a2b_1200": (PhaseState(0.9, 0.0, 0.1), 1200.0, 1e-3, 400),
            "a2b_1100_dt01": (PhaseState(0.9, 0.0, 0.1), 1100.0, 0.01, 300),
            "b2a_1000": (PhaseState(0.0, 0.0, 1.0), 1000.0, 0.01, 50),
            "b2a_900": (PhaseState(0.0, 0.0, 1.0), 900.0, 0.05, 80),
            "melt_2000": (PhaseState(0.9, 0.0, 0.1), 2000.0, 1e-3, 3),
            "cold_300": (PhaseState(0.9, 0.0, 0.1), 300.0, 1e-3, 3)}
    for name, (st, t, dt, n) in seqs.items():
        rows = []
        seed = None
        for _ in range(n):
            st, seed = initiate_diffusion(st, t, dt, seed)
            rows.append([st.x_alpha_s, st.x_alpha_m, st.x_beta, float(seed.active),
                         {None: 0.0, "beta_to_alpha_s": 1.0, "alpha_s_to_beta": 2.0}[seed.direction],
                         seed.tracked])
        c[f"{name}/rows"] = np.array(rows)
        c[f"{name}/args"] = np.array([t, dt, n])
    np.savez_compressed(OUT / "initiation.npz", **c)


def _digest(f):
    import hashlib
    out = {}
    act = np.asarray(f.seed_active) != 0
    for k in ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old", "seed_active"):
        out[k] = hashlib.sha256(np.ascontiguousarray(getattr(f, k)).tobytes()).hexdigest()
    out["seed_tracked_active"] = hashlib.sha256(
        np.ascontiguousarray(np.asarray(f.seed_tracked)[act]).tobytes()).hexdigest()
    return out


def make_advance_large():
    """Large reference runs that select the fused kernel's throughput
    instance (> 37 888 points, > 1184 32-point tasks): the final state's
    SHA-256 per array (seed_tracked only where active) and the first 4096
    points in full.  Reference step_all (n_lanes=8) with this project's
    generators (oracle definitions), threads=all."""
    cases = {"cfg4_40960_off3x2^24_0-24000": (4, 40960, 3 << 24, 24000),
             "cfg2_65536_off0_0-6000": (2, 65536, 0, 6000)}
    out = {}
    threads = os.cpu_count() or 1
    for name, (cfg_id, n, off, nsteps) in cases.items():
        src = sources.source_for_config(cfg_id)
        gen = src.tempgen(point_offset=off)
        init = orc.gen_initial_state(gen, n)
        t0 = orc.gen_temperature(gen, n, 0, threads)
        f = GlobalFields(init.x_alpha_s, init.x_alpha_m, init.x_beta, t0, t0.copy())
        for s in range(nsteps):
            f.temperature_new[:] = orc.gen_temperature(gen, n, s + 1, threads)
            step_all(f, src.dt, DEFAULT_PARAMS, CFG_E, n_lanes=8, threads=threads)
        d = _digest(f)
        out[f"{name}/args"] = np.array([cfg_id, n, off, nsteps], np.int64)
        for k, v in d.items():
            out[f"{name}/sha_{k}"] = np.array(v)
        for k in NAMES:
            out[f"{name}/head_{k}"] = np.array(getattr(f, k))[:4096]
        print(name, d["x_alpha_s"][:16], flush=True)
    np.savez_compressed(OUT / "advance_large.npz", **out)


if __name__ == "__main__":
    if "--large-only" in sys.argv:
        make_advance_large()
        print("advance large done")
        sys.exit(0)
    if "--init-only" in sys.argv:
        make_initiation()
        print("initiation done")
        sys.exit(0)
    if "--acceptance-only" in sys.argv:
        make_acceptance()
        print("acceptance done")
        sys.exit(0)
    if "--api-only" in sys.argv:
        make_kinetics_api()
        print("kinetics api done")
        sys.exit(0)
    if "--report-only" in sys.argv:
        make_report()
        print("report done")
        sys.exit(0)
    if "--build-only" in sys.argv:
        make_build()
        print("build done")
        sys.exit(0)
    if "--cn-only" in sys.argv:
        make_cn()
        print("cn done")
        sys.exit(0)
    make_cn()
    print("cn done")
    make_build()
    print("build done")
    make_report()
    print("report done")
    make_kinetics_api()
    print("kinetics api done")
    make_acceptance()
    print("acceptance done")
    make_initiation()
    print("initiation done")
    make_fastmath()
    print("fastmath done")
    make_steps()
    print("steps done")
    make_history()
    print("history done")
    make_stencil()
    print("stencil done")
    make_advance(0, 4096, 20000, 1000)
    print("advance cfg0 done")
    small1 = sources.RosenthalRaster(nx=32, ny=32, nz=4)
    make_advance(1, 4096, 2000, 500, src=small1, name="advance_cfg1_small.npz")
    print("advance cfg1 small done")
    make_advance(2, 512, 50000, 5000, point_offset=12345)
    print("advance cfg2 done")
    make_advance(4, 256, 100000, 10000, point_offset=777)
    print("advance cfg4 done")
