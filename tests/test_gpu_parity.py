"""GPU parity: the sm_100a path (through the C ABI) against the golden
fixtures made from the reference and against the CPU oracle.  Bit-exact for
every state array; phase sums within 1e-12 relative (summation order);
event counts exact."""

import numpy as np
import pytest

from conftest import FIELD_NAMES, assert_bitwise, golden_cases, load_golden, random_states

pytestmark = pytest.mark.gpu

STEPS = golden_cases(load_golden("steps.npz"))


@pytest.fixture(scope="module")
def pkg():
    import paper_2402_17580_b200 as p
    return p


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle as o
    return o


def gpu_fields(pkg, d, prefix=""):
    return pkg.GlobalFields(*[d[prefix + k] for k in FIELD_NAMES[:5]],
                            *[d.get(prefix + k) for k in FIELD_NAMES[5:]])


def assert_fields(f, ref, what):
    h = f.to_host()
    for k in FIELD_NAMES:
        r = ref[k] if isinstance(ref, dict) else getattr(ref, k)
        assert_bitwise(h[k], r, f"{what}:{k}")


def test_fastmath_golden(pkg):
    g = load_golden("fastmath.npz")
    assert_bitwise(pkg.fast_exp(g["x_exp"]), g["y_exp"], "fast_exp")
    assert_bitwise(pkg.fast_ln(g["x_ln"]), g["y_ln"], "fast_ln")
    assert_bitwise(pkg.fast_pow(g["a_pow"], g["x_pow"]), g["y_pow"], "fast_pow")


def test_fastmath_known_answers(pkg):
    # test_fastmath.py:11-61 known answers
    assert pkg.fast_exp(-750.0) == 0.0
    assert pkg.fast_exp(800.0) == np.finfo(np.float64).max
    assert np.isnan(pkg.fast_exp(float("nan")))
    assert abs(pkg.fast_exp(0.0) - 1.0) < 1e-9
    assert np.isnan(pkg.fast_ln(0.0)) and np.isnan(pkg.fast_ln(-1.0))
    assert abs(pkg.fast_ln(1e-310) - np.log(np.finfo(np.float64).tiny)) < 1e-4
    assert abs(pkg.fast_pow(0.25, 0.5) - 0.5) / 0.5 < 1e-5


@pytest.mark.parametrize("name", sorted(STEPS))
def test_step_all_golden(pkg, name):
    case = STEPS[name]
    f = gpu_fields(pkg, case, "in_")
    for s in range(int(case["nsteps"])):
        if "t_seq" in case:
            f.temperature_new.copy_(pkg.batch._torch().from_numpy(case["t_seq"][s]))
        pkg.step_all(f, float(case["dt"]), n_lanes=int(case["lanes"]))
    assert_fields(f, {k: case["out_" + k] for k in FIELD_NAMES}, name)


@pytest.mark.parametrize("lanes", [1, 2, 4, 8])
def test_lane_width_invariance_and_oracle(pkg, orc, lanes):
    # test_batch.py:79-85 at scale, against the oracle at the same lane width
    d = random_states(100_003, seed=42)
    f = pkg.GlobalFields(*[d[k] for k in FIELD_NAMES[:5]])
    h = orc.HostFields(*[d[k] for k in FIELD_NAMES[:5]])
    kp = pkg.DEFAULT_PARAMS.kernel_tuple()
    cfg = pkg.IntegratorConfig().kernel_tuple()
    for s in range(3):
        pkg.step_all(f, 2e-5, n_lanes=lanes)
        orc.step_all(h, 2e-5, kp, cfg, n_lanes=lanes, threads=4)
    assert_fields(f, h, f"lanes={lanes}")


def test_counters_and_traffic(pkg):
    d = random_states(1003, seed=8)
    f = pkg.GlobalFields(*[d[k] for k in FIELD_NAMES[:5]])
    pkg.step_all(f, 2e-5, n_lanes=8)
    assert f.traffic_bytes == 72 * 1003 and f.steps_taken == 1
    t_new = f.host("temperature_new")
    assert np.array_equal(f.host("temperature_old"), t_new)


def test_validation_errors(pkg):
    d = random_states(8, seed=13)
    f = pkg.GlobalFields(*[d[k] for k in FIELD_NAMES[:5]])
    with pytest.raises(ValueError):
        pkg.step_all(f, 2e-5, n_lanes=3)
    with pytest.raises(ValueError):
        pkg.step_all(f, -1.0)
    with pytest.raises(ValueError):
        pkg.step_all(f, 2e-5, n_lanes=16, config=pkg.IntegratorConfig(scheme="crank_nicolson"))


def test_scalar_api_matches_batch(pkg):
    # test_batch.py:97-105
    d = random_states(64, seed=5)
    f = pkg.GlobalFields(*[d[k] for k in FIELD_NAMES[:5]])
    pkg.step_all(f, 2e-5)
    st = f.states()
    for i in (0, 7, 33, 63):
        out = pkg.step_explicit(pkg.PhaseState(d["x_alpha_s"][i], d["x_alpha_m"][i],
                                               d["x_beta"][i]),
                                d["temperature_old"][i], d["temperature_new"][i], 2e-5)
        assert tuple(st[i]) == out.as_tuple()


def test_seeding_scalar_known_answer(pkg):
    # test_integrator.py:356-362 / 426-435: first seeded step at 1200 K
    seed = pkg.SeedingState()
    out = pkg.step_explicit(pkg.PhaseState(0.9, 0.0, 0.1), 1200.0, 1200.0, 1e-4, seeding=seed)
    assert seed.active and seed.direction == "alpha_s_to_beta"
    assert 0.0 < seed.tracked < 1e-30
    assert abs(out.x_beta - 0.1) <= 1e-15


def test_subcycling_equals_chained(pkg):
    # test_integrator.py:449-464
    s0 = pkg.PhaseState(0.45, 0.0, 0.55)
    a = pkg.integrate_interval(s0, 1000.0, 1000.0, 0.1)
    b = s0
    for _ in range(10):
        b = pkg.step_explicit(b, 1000.0, 1000.0, 0.01)
    assert a.as_tuple() == b.as_tuple()


def test_history_golden(pkg):
    for name, case in golden_cases(load_golden("history.npz")).items():
        out = pkg.integrate_history(case["times"], case["temps"])
        assert_bitwise(out, case["out"], name)


def test_history_batched_matches_single(pkg):
    rng = np.random.default_rng(3)
    times = np.linspace(0.0, 2.0, 400)
    temps = 300.0 + 1500.0 * rng.uniform(0, 1, (400, 37))
    batched = pkg.integrate_history(times, temps)
    for j in (0, 11, 36):
        assert_bitwise(batched[:, j, :], pkg.integrate_history(times, temps[:, j]), f"h{j}")


def _advance_vs_golden(pkg, fname, src):
    g = load_golden(fname)
    cfg_id = int(g["cfg"])
    src = src or pkg.source_for_config(cfg_id)
    n, nsteps = int(g["n"]), int(g["nsteps"])
    f = pkg.init_from_source(src, n, point_offset=int(g["point_offset"]))
    cnt = pkg.EventCounters(n, f.device)
    r = pkg.advance(f, nsteps, src, snapshot_every=int(g["snap_every"]), counters=cnt,
                    n_lanes=int(g["lanes"]), point_offset=int(g["point_offset"]))
    assert_fields(f, {k: g["out_" + k] for k in FIELD_NAMES}, fname)
    assert np.array_equal(cnt.martensite.cpu().numpy().astype(np.uint32), g["martensite"])
    assert np.array_equal(cnt.switches.cpu().numpy().astype(np.uint32), g["switches"])
    assert np.array_equal(cnt.totals.cpu().numpy().astype(np.uint64), g["totals"])
    np.testing.assert_allclose(r.sums.cpu().numpy(), g["sums"], rtol=1e-12, atol=1e-12)
    # the uncounted kernel (the timed one: range rest + steady skip) too
    f2 = pkg.init_from_source(src, n, point_offset=int(g["point_offset"]))
    pkg.advance(f2, nsteps, src, snapshot_every=int(g["snap_every"]),
                n_lanes=int(g["lanes"]), point_offset=int(g["point_offset"]))
    assert_fields(f2, {k: g["out_" + k] for k in FIELD_NAMES}, fname + " (uncounted)")


def test_advance_cfg0_golden(pkg):
    _advance_vs_golden(pkg, "advance_cfg0.npz", None)


def test_advance_cfg1_small_golden(pkg):
    _advance_vs_golden(pkg, "advance_cfg1_small.npz",
                       pkg.RosenthalRaster(nx=32, ny=32, nz=4))


def test_advance_cfg2_golden(pkg):
    _advance_vs_golden(pkg, "advance_cfg2.npz", None)


def test_advance_cfg4_golden(pkg):
    _advance_vs_golden(pkg, "advance_cfg4.npz", None)


@pytest.mark.parametrize("cfg_id,nsteps,lanes", [(0, 3000, 8), (1, 400, 8), (2, 2000, 4),
                                                 (4, 2000, 1)])
def test_advance_equals_step_loop(pkg, cfg_id, nsteps, lanes):
    """K2 (fused) == K1 (step_all) driven by the same generator, bitwise."""
    src = pkg.source_for_config(cfg_id)
    if cfg_id == 1:
        src = pkg.RosenthalRaster(nx=64, ny=64, nz=8)
    n = 8192 + 13
    a = pkg.init_from_source(src, n, point_offset=5000)
    b = a.copy()
    step0 = 2000 if cfg_id in (0, 2) else 0
    if step0:
        from paper_2402_17580_b200.batch import gen_temperature
        t = gen_temperature(src, n, step0, point_offset=5000)
        a.temperature_old.copy_(t)
        b.temperature_old.copy_(t)
    pkg.advance(a, nsteps, src, step0=step0, n_lanes=lanes, point_offset=5000,
                snapshot_every=1000)
    from paper_2402_17580_b200.batch import gen_temperature
    for s in range(step0, step0 + nsteps):
        b.temperature_new.copy_(gen_temperature(src, n, s + 1, point_offset=5000))
        pkg.step_all(b, src.dt, n_lanes=lanes)
    ha, hb = a.to_host(), b.to_host()
    for k in FIELD_NAMES:
        if k == "temperature_new":
            continue
        assert_bitwise(ha[k], hb[k], f"cfg{cfg_id}:{k}")


@pytest.mark.parametrize("cfg_id,n", [(0, 8192 + 13), (1, 4096), (2, 1 << 16)])
def test_advance_subcycled_equals_step_loop(pkg, cfg_id, n):
    """nsub > 1 (dt_sub_max = dt / 2.5 -> 3 substeps with interpolated T):
    the general K2 instances (counted and uncounted) == the step_all loop."""
    from paper_2402_17580_b200.batch import gen_temperature
    src = pkg.source_for_config(cfg_id)
    if cfg_id == 1:
        src = pkg.RosenthalRaster(nx=64, ny=64, nz=1)
    config = pkg.IntegratorConfig(dt_sub_max=src.dt / 2.5)
    step0 = 2000 if cfg_id in (0, 2) else 0
    nsteps = 300
    a = pkg.init_from_source(src, n)
    if step0:
        a.temperature_old.copy_(gen_temperature(src, n, step0))
    b, c = a.copy(), a.copy()
    pkg.advance(a, nsteps, src, step0=step0, config=config)
    pkg.advance(c, nsteps, src, step0=step0, config=config, counters=pkg.EventCounters(n, c.device))
    for st in range(step0, step0 + nsteps):
        b.temperature_new.copy_(gen_temperature(src, n, st + 1))
        pkg.step_all(b, src.dt, config=config)
    ha, hb, hc = a.to_host(), b.to_host(), c.to_host()
    for k in FIELD_NAMES:
        if k == "temperature_new":
            continue
        assert_bitwise(ha[k], hb[k], f"cfg{cfg_id} nsub3:{k}")
        assert_bitwise(hc[k], hb[k], f"cfg{cfg_id} nsub3 counted:{k}")


def test_div_rn(pkg):
    """div_rn (the kinetics' inline division) == __ddiv_rn bit for bit: random
    bit patterns over the whole range (subnormal operands and quotients,
    overflow, specials) and quotients straddling the subnormal threshold."""
    import torch
    from paper_2402_17580_b200 import _lib
    lib = _lib.require()
    rng = np.random.default_rng(7)
    n = 1 << 22
    a = rng.integers(0, 2**64, n, dtype=np.uint64).view(np.float64).copy()
    b = rng.integers(0, 2**64, n, dtype=np.uint64).view(np.float64).copy()
    # quotients near and below the smallest normal, and near overflow
    m = n // 4
    b[:m] = rng.uniform(1.0, 2.0, m) * 2.0 ** rng.integers(-60, 60, m)
    a[:m] = b[:m] * rng.uniform(0.5, 2.0, m) * 2.0 ** rng.integers(-1080, -1015, m).astype(float)
    a[m:2 * m] = rng.uniform(1.0, 2.0, m) * 2.0 ** rng.integers(-1074, 1024, m).astype(float)
    b[m:2 * m] = rng.uniform(1.0, 2.0, m) * 2.0 ** rng.integers(-1074, 1024, m).astype(float)
    # exact ties into the subnormal range: odd multiples of 2^-1075 times b
    k = rng.integers(1, 2**20, 4096) * 2 + 1
    bb = rng.integers(1, 2**20, 4096).astype(float)
    a[2 * m:2 * m + 4096] = np.ldexp(k * bb, -1075)
    b[2 * m:2 * m + 4096] = bb
    specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, -1.0, 5e-324, 2.2250738585072014e-308,
                         1.7976931348623157e308, 3.0, 1e-300, 1e300])
    sa, sb = np.meshgrid(specials, specials)
    a[-sa.size:] = sa.ravel()
    b[-sb.size:] = sb.ravel()
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    out, ref = torch.empty_like(da), torch.empty_like(da)
    rc = lib.ti64_div_rn(_lib.ptr(da), _lib.ptr(db), _lib.ptr(out), _lib.ptr(ref), n, None)
    assert rc == 0
    o, r = out.cpu().numpy(), ref.cpu().numpy()
    assert_bitwise(o, r, "div_rn vs __ddiv_rn")
    # and the host's IEEE division (the reference's numba divsd) on non-NaN results
    with np.errstate(all="ignore"):
        h = a / b
    ok = ~np.isnan(h)
    assert_bitwise(o[ok], h[ok], "div_rn vs host IEEE")


def test_k1_subcycled_seed_warp_regression(pkg, orc):
    """One warp of config 2's state at step 2026 (points 96-127 of a 2^16
    run; two lanes with an active seed, the others on the rate path), stepped
    with nsub = 3: with seed_advance as an out-of-line call this warp faulted
    (illegal address) or hung on sm_100a.  The fixture is our own state dump
    (tests/golden/k1_nsub3_seed_warp.npz), checked against the oracle."""
    g = load_golden("k1_nsub3_seed_warp.npz")
    names = ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old", "temperature_new")
    dt = 1e-5
    config = pkg.IntegratorConfig(dt_sub_max=dt / 2.5)
    f = pkg.GlobalFields(*[g[k] for k in names], seed_tracked=g["seed_tracked"],
                         seed_active=g["seed_active"], seed_direction=g["seed_direction"])
    h = orc.HostFields(*[g[k] for k in names], seed_tracked=g["seed_tracked"],
                       seed_active=g["seed_active"], seed_direction=g["seed_direction"])
    pkg.step_all(f, dt, config=config)
    orc.step_all(h, dt, pkg.DEFAULT_PARAMS.kernel_tuple(), config.kernel_tuple(), n_lanes=8)
    got = f.to_host()
    for k in FIELD_NAMES:
        assert_bitwise(got[k], getattr(h, k), f"seed warp nsub3:{k}")


def test_generator_matches_oracle(pkg, orc):
    from paper_2402_17580_b200.batch import gen_temperature
    for cfg_id in (0, 1, 2, 4):
        src = pkg.source_for_config(cfg_id)
        n = 4096
        for step in (0, 1, 3000, 9999):
            tab = src.beam_table(step + 1)
            g = src.tempgen(point_offset=77777, beam_ptr=None if tab is None else tab.ctypes.data,
                            beam_steps=0 if tab is None else len(tab))
            ref = orc.gen_temperature(g, n, step)
            got = gen_temperature(src, n, step, point_offset=77777).cpu().numpy()
            assert_bitwise(got, ref, f"gen cfg{cfg_id} step {step}")


def test_advance_cfg1_full_lattice_block_vs_oracle(pkg, orc):
    """Config 1 at its full 2^20-point lattice, 300 steps; the oracle checks
    two 4096-point blocks (surface and depth) bit for bit."""
    src = pkg.source_for_config(1)
    n = src.n_points
    f = pkg.init_from_source(src, n)
    kp = pkg.DEFAULT_PARAMS.kernel_tuple()
    cfg = pkg.IntegratorConfig().kernel_tuple()
    pkg.advance(f, 300, src, snapshot_every=100)
    h = f.to_host()
    tab = src.beam_table(301)
    for off in (0, 128 * 128 * 5 + 4096):
        g = src.tempgen(point_offset=off, beam_ptr=tab.ctypes.data, beam_steps=len(tab))
        ho = orc.gen_initial_state(g, 4096)
        t0 = orc.gen_temperature(g, 4096, 0)
        ho.temperature_old[:] = t0
        ho.temperature_new[:] = t0
        orc.advance(ho, g, 0, 300, kp, cfg, lanes=8, threads=8)
        for k in FIELD_NAMES:
            assert_bitwise(h[k][off:off + 4096], getattr(ho, k), f"block {off}:{k}")


@pytest.mark.parametrize("cfg_id,step0,nsteps", [(0, 2000, 1500), (2, 2000, 1200), (4, 0, 1200)])
def test_advance_pulse_throughput_instance_vs_oracle(pkg, orc, cfg_id, step0, nsteps):
    """Pulse generators at a launch size that takes the throughput instance
    of K2 (72 registers; small launches take the latency instance, which the
    golden tests cover): two 2048-point blocks checked by the oracle bit for
    bit, and the whole launch equal to the same points run as small
    (latency-instance) launches."""
    from paper_2402_17580_b200.batch import gen_temperature
    src = pkg.source_for_config(cfg_id)
    n = 1 << 16
    f = pkg.init_from_source(src, n)
    if step0:
        f.temperature_old.copy_(gen_temperature(src, n, step0))
    pkg.advance(f, nsteps, src, step0=step0, snapshot_every=500)
    h = f.to_host()
    kp = pkg.DEFAULT_PARAMS.kernel_tuple()
    cfg = pkg.IntegratorConfig().kernel_tuple()
    for off in (0, n - 2048):
        g = src.tempgen(point_offset=off)
        ho = orc.gen_initial_state(g, 2048)
        t0 = orc.gen_temperature(g, 2048, step0)
        ho.temperature_old[:] = t0
        ho.temperature_new[:] = t0
        orc.advance(ho, g, step0, nsteps, kp, cfg, lanes=8, threads=8)
        for k in FIELD_NAMES:
            assert_bitwise(h[k][off:off + 2048], getattr(ho, k), f"cfg{cfg_id} block {off}:{k}")
    small = pkg.init_from_source(src, 4096, point_offset=8192)
    if step0:
        small.temperature_old.copy_(gen_temperature(src, 4096, step0, point_offset=8192))
    pkg.advance(small, nsteps, src, step0=step0, snapshot_every=500, point_offset=8192)
    hs = small.to_host()
    for k in FIELD_NAMES:
        assert_bitwise(h[k][8192:8192 + 4096], hs[k], f"cfg{cfg_id} lat-vs-throughput:{k}")


@pytest.mark.parametrize("over", [dict(k3=0.2), dict(k1=0.5, k2=700.0, k_alpha_m_eq=0.01),
                                  dict(t_alpha_s_end=1300.0)])
@pytest.mark.parametrize("cfg_id,step0", [(4, 20000), (2, 10000)])
def test_advance_cold_loop_other_parameters_vs_oracle(pkg, orc, cfg_id, step0, over):
    """The cold loop of K2 with kinetics parameters other than the defaults:
    k3 = 0.2 puts k_alpha_s's exponential argument outside the host-verified
    range (the loop then keeps fast_exp's and the division's range branches),
    the second set stays inside it with other values, the third has
    T_alpha_s,end above T_alpha_s,start (no range rest, no cold loop).
    Throughput-instance launch, mid-job states; two blocks against the oracle."""
    from paper_2402_17580_b200.batch import gen_temperature
    params = pkg.DEFAULT_PARAMS.with_overrides(**over)
    src = pkg.source_for_config(cfg_id)
    n, pre, nsteps = 1 << 16, 1500, 700
    f = pkg.init_from_source(src, n)
    f.temperature_old.copy_(gen_temperature(src, n, step0))
    pkg.advance(f, pre, src, step0=step0, params=params)
    pkg.advance(f, nsteps, src, step0=step0 + pre, params=params, snapshot_every=300)
    h = f.to_host()
    kp = params.kernel_tuple()
    cfg = pkg.IntegratorConfig().kernel_tuple()
    for off in (4096, n - 2048):
        g = src.tempgen(point_offset=off)
        ho = orc.gen_initial_state(g, 2048)
        t0 = orc.gen_temperature(g, 2048, step0)
        ho.temperature_old[:] = t0
        ho.temperature_new[:] = t0
        orc.advance(ho, g, step0, pre + nsteps, kp, cfg, lanes=8, threads=8)
        for k in FIELD_NAMES:
            assert_bitwise(h[k][off:off + 2048], getattr(ho, k), f"cfg{cfg_id} {over} {off}:{k}")


def test_full_config1_invariants(pkg):
    """Size-independent properties at BASELINE config 1's full size and
    length: continuity sum == 1 - g(T) (acceptance criterion 3, <= 1e-12),
    bounds, and run-to-run determinism of every bit."""
    src = pkg.source_for_config(1)
    n = src.n_points
    runs = []
    for _ in range(2):
        f = pkg.init_from_source(src, n)
        r = pkg.advance(f, 10_000, src, snapshot_every=1000)
        runs.append((f.to_host(), r.sums.cpu().numpy()))
    (h, sums), (h2, sums2) = runs
    for k in FIELD_NAMES:
        assert_bitwise(h[k], h2[k], f"determinism {k}")
    assert np.array_equal(sums, sums2)
    t = h["temperature_old"]
    g = np.clip((t - 1878.0) / 50.0, 0.0, 1.0)
    tot = h["x_alpha_s"] + h["x_alpha_m"] + h["x_beta"]
    assert np.abs(tot - (1.0 - g)).max() <= 1e-12
    assert h["x_alpha_s"].min() >= 0.0 and h["x_alpha_m"].min() >= 0.0
    assert (h["x_alpha_s"] + h["x_alpha_m"]).max() <= 0.9 + 1e-12
    np.testing.assert_allclose(sums[-1], [h["x_alpha_s"].sum(), h["x_alpha_m"].sum(),
                                          h["x_beta"].sum()], rtol=1e-12)


def test_phase_sums_and_histogram(pkg):
    d = random_states(300_001, seed=1)
    f = pkg.GlobalFields(*[d[k] for k in FIELD_NAMES[:5]])
    s = pkg.phase_sums(f).cpu().numpy()
    np.testing.assert_allclose(s, [d["x_alpha_s"].sum(), d["x_alpha_m"].sum(),
                                   d["x_beta"].sum()], rtol=1e-12)
    hist = pkg.histogram(f, 256).cpu().numpy()
    for c, k in enumerate(("x_alpha_s", "x_alpha_m", "x_beta")):
        x = d[k]
        ref = np.bincount(np.clip(np.floor(x * 256).astype(np.int64), 0, 255), minlength=256)
        assert np.array_equal(hist[c], ref)


@pytest.mark.parametrize("cfg_id,n,steps,chunk", [(4, 150_013, 450, 4096), (4, 70_000, 300, 65536),
                                                   (2, 90_001, 400, 8192), (0, 5000, 600, 1024),
                                                   (1, 32768, 300, 5000)])
@pytest.mark.parametrize("lanes", [8, 1])
def test_host_fields_staged_chunks(pkg, cfg_id, n, steps, chunk, lanes):
    """ti64_advance_host: host arrays staged through the device in chunks
    (ragged last chunk, chunk sizes rounded to 1024, a window starting
    mid-job) give the bits of one device-resident advance over all points,
    event counters included; the zero-copy form of the same call agrees too."""
    src = pkg.source_for_config(cfg_id) if cfg_id != 1 else pkg.RosenthalRaster(nx=64, ny=64, nz=8)
    a = pkg.init_from_source(src, n, point_offset=37 * 32)
    pkg.advance(a, 250, src, point_offset=37 * 32, n_lanes=lanes)  # off the initial state
    start = a.to_host()
    ca = pkg.EventCounters(n, a.device)
    ra = pkg.advance(a, steps, src, step0=250, point_offset=37 * 32, n_lanes=lanes,
                     snapshot_every=170, counters=ca)
    want = a.to_host()
    for hc in (chunk, -1):
        h = pkg.GlobalFields(*[start[k] for k in FIELD_NAMES], device="host")
        ch = pkg.EventCounters(n, a.device)
        rh = pkg.advance(h, steps, src, step0=250, point_offset=37 * 32, n_lanes=lanes,
                         snapshot_every=170, counters=ch, host_chunk_points=hc)
        assert_fields(h, want, f"host chunks {hc}")
        np.testing.assert_allclose(rh.sums.cpu().numpy(), ra.sums.cpu().numpy(), rtol=1e-12)
        assert ch.totals_dict() == ca.totals_dict()
        assert np.array_equal(ch.martensite.cpu().numpy(), ca.martensite.cpu().numpy())
        assert np.array_equal(ch.switches.cpu().numpy(), ca.switches.cpu().numpy())


def test_advance_host_c_abi_contract(pkg):
    """ti64_advance_host through ctypes: scratch-size query, argument errors
    (negative return + message, host arrays untouched), empty input, and
    pageable (unpinned) host arrays giving the same bits as pinned ones."""
    import ctypes as C

    import torch
    from paper_2402_17580_b200 import _lib
    from paper_2402_17580_b200.batch import _cfg, _kp
    lib = _lib.require()
    src = pkg.source_for_config(4)
    n = 50_000
    a = pkg.init_from_source(src, n)
    pkg.advance(a, 300, src)
    start = a.to_host()
    pkg.advance(a, 200, src, step0=300)
    want = a.to_host()
    g = src.tempgen(point_offset=0)
    kp, cfg = _kp(pkg.DEFAULT_PARAMS), _cfg(pkg.IntegratorConfig())
    need = lib.ti64_advance_host_scratch_bytes(n, 8192, 200, 0)
    assert need > 3 * 50 * 8192
    assert lib.ti64_advance_host_scratch_bytes(-1, 0, 1, 0) < 0
    scratch = torch.empty(need // 8 + 1, dtype=torch.float64, device="cuda")
    arrs = [np.array(start[k], copy=True) for k in FIELD_NAMES]  # pageable numpy memory
    f = _lib._abi.Fields(*[x.ctypes.data for x in arrs])
    st = _lib.stream_handle()

    def call(nn, staging, nbytes, lanes=8):
        return lib.ti64_advance_host(C.byref(f), nn, C.byref(g), 300, 200, 1, lanes, 0,
                                     C.byref(kp), C.byref(cfg), None, None, staging, nbytes,
                                     8192, st)
    assert call(n, _lib.ptr(scratch), need - 1) == -1      # staging too small
    assert b"staging" in lib.ti64_last_error()
    assert call(n, None, need) == -1                        # no staging
    assert call(n, _lib.ptr(scratch), need, lanes=3) == -1  # bad lane width
    for x, k in zip(arrs, FIELD_NAMES):
        assert_bitwise(x, start[k], f"untouched after errors:{k}")
    assert call(0, _lib.ptr(scratch), need) == 0            # empty input
    assert call(n, _lib.ptr(scratch), need) > 0
    torch.cuda.synchronize()
    for x, k in zip(arrs, FIELD_NAMES):
        assert_bitwise(x, want[k], f"pageable host arrays:{k}")


def test_host_resident_fields_zero_copy(pkg):
    """GlobalFields(device='host'): pinned host state read and written by the
    kernels themselves gives the same bits as device-resident state."""
    src = pkg.RosenthalRaster(nx=64, ny=64, nz=8)
    n = src.n_points
    a = pkg.init_from_source(src, n)
    h = pkg.GlobalFields(*[a.host(k) for k in FIELD_NAMES], device="host")
    assert h.host_resident and h.x_alpha_s.is_pinned()
    ra = pkg.advance(a, 700, src, snapshot_every=300)
    rh = pkg.advance(h, 700, src, snapshot_every=300)
    assert_fields(h, a.to_host(), "advance host vs device")
    assert np.array_equal(rh.sums.cpu().numpy(), ra.sums.cpu().numpy())
    d = random_states(5000, seed=9)
    b = pkg.GlobalFields(*[d[k] for k in FIELD_NAMES[:5]])
    g = pkg.GlobalFields(*[d[k] for k in FIELD_NAMES[:5]], device="host")
    for cfg in (pkg.IntegratorConfig(), pkg.IntegratorConfig(scheme="crank_nicolson")):
        pkg.step_all(b, 1e-3, config=cfg)
        pkg.step_all(g, 1e-3, config=cfg)
        assert_fields(g, b.to_host(), f"step_all host vs device {cfg.scheme}")
