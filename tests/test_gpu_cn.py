"""GPU parity of the Crank-Nicolson path (batch.py:357-416 _cn_substep,
:568-674 halving, :684-695 iteration counts and failure) against the
reference's golden fixtures (tests/golden/cn_*.npz, made by
tests/golden/make_golden.py from the reference) and the CPU oracle.
Bit-exact for every state array and every iteration count."""

import numpy as np
import pytest

from conftest import FIELD_NAMES, assert_bitwise, golden_cases, load_golden, random_states

pytestmark = pytest.mark.gpu

CN = golden_cases(load_golden("cn_steps.npz"))


@pytest.fixture(scope="module")
def pkg():
    import paper_2402_17580_b200 as p
    return p


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle as o
    return o


def _cn_cfg(pkg, c):
    return pkg.IntegratorConfig(scheme="crank_nicolson", dt_sub_max=float(c[0]),
                                eps_abs=float(c[1]), eps_rel=float(c[2]),
                                max_fixed_point_iters=int(c[3]),
                                initiation_threshold=float(c[4]), stuck_tol=float(c[5]),
                                max_halvings=int(c[6]))


def _gpu_fields(pkg, d, prefix=""):
    return pkg.GlobalFields(*[d[prefix + k] for k in FIELD_NAMES[:5]],
                            *[d.get(prefix + k) for k in FIELD_NAMES[5:]])


def _assert_same(f, ref, what):
    h = f.to_host()
    for k in FIELD_NAMES:
        r = ref[k] if isinstance(ref, dict) else getattr(ref, k)
        assert_bitwise(h[k], r, f"{what}:{k}")


@pytest.mark.parametrize("name", sorted(CN))
def test_cn_step_all_golden(pkg, name):
    case = CN[name]
    cfg = _cn_cfg(pkg, case["cfg"])
    f = _gpu_fields(pkg, case, "in_")
    lanes = int(case["lanes"])
    fail, iters = [], None
    for s in range(int(case["nsteps"])):
        if "t_seq" in case:
            f.temperature_new.copy_(pkg.batch._torch().from_numpy(case["t_seq"][s]))
        try:
            iters = pkg.step_all(f, float(case["dt"]), config=cfg, n_lanes=lanes,
                                 record_iters=True)
        except pkg.BatchConvergenceError as e:
            fail = e.indices
            break
    assert fail == list(case["fail"])
    _assert_same(f, {k: case["out_" + k] for k in FIELD_NAMES}, name)
    if case["iters"].size and not fail:
        assert np.array_equal(iters.cpu().numpy(), case["iters"])


def test_cn_history_golden(pkg):
    cfg = pkg.IntegratorConfig(scheme="crank_nicolson")
    for name, case in golden_cases(load_golden("cn_history.npz")).items():
        s0 = pkg.PhaseState(*case["out"][0])
        out = pkg.integrate_history(case["times"], case["temps"], s0, config=cfg)
        assert_bitwise(out, case["out"], name)


@pytest.mark.parametrize("lanes", [1, 2, 4, 8])
@pytest.mark.parametrize("dt,extra", [(2e-5, {}), (0.05, {}),
                                      (0.3, dict(dt_sub_max=1.0, eps_abs=1e-18, eps_rel=1e-8,
                                                 max_fixed_point_iters=6))])
def test_cn_random_vs_oracle(pkg, orc, lanes, dt, extra):
    n = 4099  # ragged tail batch, several warps and blocks
    d = random_states(n, seed=lanes * 31 + int(dt * 1e5) % 97)
    cfg = pkg.IntegratorConfig(scheme="crank_nicolson", **extra)
    h = orc.HostFields(*[d[k] for k in FIELD_NAMES[:5]])
    nsub = orc.num_substeps(dt, cfg.dt_sub_max)
    rc, it = orc.run_range_cn(h, pkg.DEFAULT_PARAMS.kernel_tuple(), cfg.kernel_tuple(),
                              lanes, nsub, dt / nsub)
    f = pkg.GlobalFields(*[d[k] for k in FIELD_NAMES[:5]])
    try:
        iters = pkg.step_all(f, dt, config=cfg, n_lanes=lanes, record_iters=True)
        got = 0
    except pkg.BatchConvergenceError as e:
        got, iters = e.indices[0] + 1, None
    assert got == rc
    _assert_same(f, h, f"cn lanes={lanes} dt={dt}")
    if iters is not None:
        assert np.array_equal(iters.cpu().numpy(), it)


@pytest.mark.parametrize("lanes", [1, 2, 4, 8])
def test_cn_failure_leaves_later_batches(pkg, orc, lanes):
    """Two hard batches inside a cold no-op lattice: the first fails, the
    sweep stops there (batch.py:693-695) and every later point, the second
    hard batch included, is left exactly as it was."""
    n = 200
    d = random_states(n, seed=3)
    a = {k: np.full(n, v) for k, v in zip(FIELD_NAMES[:5], (0.9, 0.0, 0.1, 300.0, 300.0))}
    for sl in (slice(40, 48), slice(120, 128)):
        for k in FIELD_NAMES[:5]:
            a[k][sl] = d[k][sl]
    cfg = pkg.IntegratorConfig(scheme="crank_nicolson", max_fixed_point_iters=2,
                               max_halvings=1, eps_rel=1e-9, eps_abs=1e-14)
    h = orc.HostFields(*[a[k] for k in FIELD_NAMES[:5]])
    rc, _ = orc.run_range_cn(h, pkg.DEFAULT_PARAMS.kernel_tuple(), cfg.kernel_tuple(),
                             lanes, 5, 0.05 / 5)
    assert 41 <= rc <= 48  # (lane-width dependent: 45 for 1, 2, 4 lanes, 41 for 8)
    f = pkg.GlobalFields(*[a[k] for k in FIELD_NAMES[:5]])
    with pytest.raises(pkg.BatchConvergenceError) as ei:
        pkg.step_all(f, 0.05, config=cfg, n_lanes=lanes, record_iters=True)
    assert ei.value.indices == list(range(rc - 1, rc - 1 + lanes))
    _assert_same(f, h, f"cn failure lanes={lanes}")
    assert_bitwise(f.host("x_alpha_s")[120:128], a["x_alpha_s"][120:128], "untouched")


def test_step_crank_nicolson_scalar(pkg):
    d = random_states(32, seed=21)
    cfg = pkg.IntegratorConfig(scheme="crank_nicolson")
    f = pkg.GlobalFields(*[d[k] for k in FIELD_NAMES[:5]])
    it = pkg.step_all(f, 1e-3, config=cfg, n_lanes=1, record_iters=True).cpu().numpy()
    st = f.states()
    for i in (0, 5, 17, 31):
        out, iters = pkg.step_crank_nicolson(
            pkg.PhaseState(d["x_alpha_s"][i], d["x_alpha_m"][i], d["x_beta"][i]),
            d["temperature_old"][i], d["temperature_new"][i], 1e-3, config=cfg)
        assert out.as_tuple() == tuple(st[i])
        assert iters == it[i]


def test_step_crank_nicolson_divergence(pkg):
    # integrator.py:191-211: the iteration cap raises with the last iterate
    cfg = pkg.IntegratorConfig(scheme="crank_nicolson", max_fixed_point_iters=1,
                               eps_abs=1e-18, eps_rel=1e-12)
    s0 = pkg.PhaseState(0.3, 0.2, 0.5)
    with pytest.raises(pkg.FixedPointDivergence) as ei:
        pkg.step_crank_nicolson(s0, 900.0, 1000.0, 0.05, config=cfg)
    e = ei.value
    assert isinstance(e, pkg.BatchConvergenceError)
    assert e.iters == 1 and e.residual_norm > 0.0 and np.isfinite(e.state.x_alpha_s)


def test_integrate_interval_cn_vs_oracle(pkg, orc):
    cfg = pkg.IntegratorConfig(scheme="crank_nicolson", dt_sub_max=0.02)
    d = random_states(16, seed=8)
    for i in range(16):
        s0 = pkg.PhaseState(d["x_alpha_s"][i], d["x_alpha_m"][i], d["x_beta"][i])
        out = pkg.integrate_interval(s0, d["temperature_old"][i], d["temperature_new"][i],
                                     0.1, config=cfg)
        h = orc.HostFields(*[d[k][i:i + 1] for k in FIELD_NAMES[:5]])
        rc, _ = orc.run_range_cn(h, pkg.DEFAULT_PARAMS.kernel_tuple(), cfg.kernel_tuple(),
                                 1, 5, 0.1 / 5)
        assert rc == 0
        assert out.as_tuple() == (h.x_alpha_s[0], h.x_alpha_m[0], h.x_beta[0])


@pytest.mark.parametrize("cfg_id,lanes", [(2, 8), (4, 1), (0, 4)])
def test_advance_cn_equals_oracle_loop(pkg, orc, cfg_id, lanes):
    """advance() with the implicit scheme = the generator + step_all loop."""
    from paper_2402_17580_b200 import sources
    src = sources.source_for_config(cfg_id)
    n, steps = 1000, 12
    cfg = pkg.IntegratorConfig(scheme="crank_nicolson")
    f = pkg.init_from_source(src, n)
    h = orc.HostFields(*[f.host(k) for k in FIELD_NAMES[:5]])
    res = pkg.advance(f, steps, src, config=cfg, n_lanes=lanes, snapshot_every=4)
    ref = orc.advance(h, src.tempgen(point_offset=0), 0, steps,
                      pkg.DEFAULT_PARAMS.kernel_tuple(), cfg.kernel_tuple(), lanes=lanes,
                      snapshot_every=4)
    _assert_same(f, h, f"advance cn lanes={lanes}")
    np.testing.assert_allclose(res.sums.cpu().numpy(), ref["sums"], rtol=1e-12, atol=0)
