"""The reference's thermal property tests (test_thermal.py:46-162) on the
device stencil: stability check, uniform field, insulated conservation,
comparison principle, monotone cooling, source/loss laws."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MM = 1e-3


@pytest.fixture(scope="module")
def th():
    from paper_2402_17580_b200 import thermal
    return thermal


def _micro(th):
    g = th.BuildGeometry(plate_size=(0.6 * MM, 0.6 * MM, 0.15 * MM),
                         part_size=(0.4 * MM, 0.4 * MM, 0.1 * MM), voxel=0.05 * MM)
    s = th.BuildSchedule(dt_active=2e-5, interlayer_dwell=0.02, initial_dwell_steps=50,
                         final_cooldown=1.0, preheat=293.0)
    field, _ = th.allocate_domain(g, s)
    return field


def _set_active(field, rng, lo, hi):
    m = field.active_mask().cpu().numpy()
    t = field.temperature_new.cpu().numpy()
    t[m] = rng.uniform(lo, hi, int(m.sum()))
    field.temperature_new.copy_(field.temperature_new.new_tensor(t))
    field.commit_temperatures()
    return m


def test_stability_bound_checked(th):
    field = _micro(th)
    with pytest.raises(ValueError, match="stability"):
        th.step_thermal(field, 1.0, nsub=1)
    assert th.stable_dt(0.05 * MM) == pytest.approx((0.05 * MM) ** 2 * 4090.0 * 1130.0 / (6.0 * 28.6))


def test_uniform_field_stays_uniform(th):
    field = _micro(th)
    th.step_thermal(field, 2e-5, losses=False)
    m = field.active_mask().cpu().numpy()
    assert np.allclose(field.temperature_new.cpu().numpy()[m], 293.0, atol=1e-12)


def test_insulated_conservation(th):
    field = _micro(th)
    _set_active(field, np.random.default_rng(0), 300.0, 1500.0)
    e0 = field.enthalpy()
    for _ in range(200):
        th.step_thermal(field, 2e-5, losses=False, bottom_dirichlet=None)
        field.commit_temperatures()
    assert abs(field.enthalpy() - e0) / e0 <= 1e-12


def test_comparison_principle(th):
    field = _micro(th)
    m = _set_active(field, np.random.default_rng(1), 293.0, 1500.0)
    hi = field.temperature_old.cpu().numpy()[m].max()
    for _ in range(500):
        th.step_thermal(field, 2e-5, losses=True, bottom_dirichlet=293.0)
        field.commit_temperatures()
        t = field.temperature_old.cpu().numpy()[field.active_mask().cpu().numpy()]
        assert t.min() >= 293.0 - 1e-9 and t.max() <= hi + 1e-9


def test_hot_voxel_cools_monotonically(th):
    field = _micro(th)
    field.temperature_new[1, 6, 6] = 2000.0
    field.commit_temperatures()
    prev = 2000.0
    for _ in range(50):
        th.step_thermal(field, 2e-5, losses=False)
        field.commit_temperatures()
        cur = float(field.temperature_old[1, 6, 6].item())
        assert cur < prev
        prev = cur


def test_source_and_loss_laws(th):
    src = th.HeatSource(w_eff=180.0, radius=0.06 * MM, h_powder=0.05 * MM)
    peak = 2.0 * 180.0 / (math.pi * (0.06 * MM) ** 2 * 0.05 * MM)
    assert th.source_term(0.0, 0.0, 0.0, 0.0, 0.0, src) == pytest.approx(peak, rel=1e-9)
    assert th.source_term(0.06 * MM, 0.0, 0.0, 0.0, 0.0, src) == pytest.approx(
        peak * math.exp(-2.0), rel=1e-6)
    assert th.source_term(0.0, 0.0, 0.06 * MM, 0.0, 0.0, src) == 0.0
    assert th.surface_losses(293.0) == pytest.approx(0.0, abs=1e-12)
    sig = th.DEFAULT_THERMAL.sigma_s
    assert th.surface_losses(2000.0) == pytest.approx(0.7 * sig * (2000.0**4 - 293.0**4), rel=1e-9)
    tc = 4130.0
    evap = (0.82 * 54e3 * math.exp(-5.07e4 * (1.0 / tc - 1.0 / 3130.0))
            * math.sqrt(9.15e-4 / tc) * (8.84e6 + 1130.0 * (tc - 538.0)))
    assert th.surface_losses(5000.0) == pytest.approx(
        0.7 * sig * (5000.0**4 - 293.0**4) + evap, rel=1e-6)
    assert th.conductivity(300.0, 0.5) == pytest.approx(0.5 * 0.286 + 0.5 * 28.6)
