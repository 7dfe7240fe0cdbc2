"""Host-side logic of the drop-in API (no GPU needed)."""

import math

import numpy as np
import pytest

import paper_2402_17580_b200 as pkg
from paper_2402_17580_b200 import sources
from paper_2402_17580_b200.integrator import num_substeps
from oracle import oracle as orc


def test_params_kernel_tuple_matches_reference_values():
    kp = pkg.DEFAULT_PARAMS.kernel_tuple()
    assert kp.exp_as_lo == (2.51 - 1.0) / 2.51
    assert kp.exp_b_hi == (11.0 + 1.0) / 11.0
    assert kp.t_as_start == 1273.0 and kp.t_am_start == 848.0
    p2 = pkg.DEFAULT_PARAMS.with_overrides(c_beta=9.0)
    assert p2.kernel_tuple().exp_b_lo == 8.0 / 9.0


def test_integrator_config_validation():
    with pytest.raises(ValueError):
        pkg.IntegratorConfig(scheme="rk4")
    with pytest.raises(ValueError):
        pkg.IntegratorConfig(dt_sub_max=-1.0)
    c = pkg.IntegratorConfig().kernel_tuple()
    assert c.scheme == 0 and c.stuck_tol == 1e-14 and c.initiation_threshold == 1e-15


def test_num_substeps_matches_oracle():
    for dt in (1e-5, 0.01, 0.0100000001, 0.05, 1.0, 0.1, 5.0, 0.033):
        assert num_substeps(dt, 0.01) == orc.num_substeps(dt, 0.01)
    assert num_substeps(0.05, 0.01) == 5


class _Dummy:
    n_points = 4


def test_step_all_validates_before_touching_the_device():
    with pytest.raises(ValueError):
        pkg.step_all(_Dummy(), 2e-5, n_lanes=3)
    with pytest.raises(ValueError):
        pkg.step_all(_Dummy(), 0.0)
    with pytest.raises(ValueError):
        pkg.step_all(_Dummy(), 1e-5, n_lanes=5,
                     config=pkg.IntegratorConfig(scheme="crank_nicolson"))


def test_convergence_error_types_and_wrms():
    # integrator.py:119-136
    e = pkg.FixedPointDivergence(pkg.PhaseState(0.1, 0.2, 0.7), 3.5, 50)
    assert isinstance(e, pkg.BatchConvergenceError) and e.indices == [0]
    assert e.iters == 50 and e.residual_norm == 3.5
    cfg = pkg.IntegratorConfig()
    r, ref = np.array([1e-6, -2e-6]), np.array([0.3, 0.0])
    w = 1.0 / (cfg.eps_abs + np.abs(ref) * cfg.eps_rel)
    assert pkg.wrms_norm(r, ref, cfg) == float(np.mean((r * w) ** 2))


def test_global_fields_shape_validation():
    with pytest.raises(ValueError):
        pkg.GlobalFields(np.zeros(3), np.zeros(4), np.zeros(3), np.zeros(3), np.zeros(3))


def test_history_validation():
    with pytest.raises(ValueError):
        pkg.integrate_history(np.array([0.0, 1.0, 0.5]), np.array([300.0] * 3))


def test_rosenthal_beam_table():
    src = sources.RosenthalRaster()
    tab = src.beam_table(10001)
    L = src.track_length
    assert src.n_tracks == 26
    assert tab.shape == (10001, 3)
    assert np.all((tab[:, 0] >= 0) & (tab[:, 0] <= L + 1e-15))
    assert set(np.unique(tab[:, 2])) <= {-1.0, 1.0}
    # 1 m/s: 2.56 ms per track
    assert tab[0, 0] == 0.0 and tab[0, 2] == 1.0
    k = int(round(L / src.speed / src.dt))  # steps per track
    assert tab[k + 1, 2] == -1.0 and tab[k + 1, 1] == src.hatch
    assert np.all(tab[:, 1] <= (src.n_tracks - 1) * src.hatch + 1e-15)


def test_generator_definitions_sane():
    """Oracle generator draws follow the BASELINE.json ranges."""
    for cfg_id in (0, 2, 4):
        src = sources.source_for_config(cfg_id)
        g = src.tempgen(point_offset=0)
        t = np.stack([orc.gen_temperature(g, 2000, s) for s in range(0, 100_000, 997)])
        assert np.all(t >= src.base) and np.all(np.isfinite(t))
        assert t.max() > src.base + 500
    src = sources.source_for_config(1)
    tab = src.beam_table(2)
    g = src.tempgen(0, tab.ctypes.data, len(tab))
    t = orc.gen_temperature(g, src.n_points, 1, threads=4)
    assert t.max() == 3000.0 and t.min() >= 353.0


def test_u01_range_and_independence():
    u = np.array([orc.u01(7, p, k) for p in range(200) for k in range(5)])
    assert u.min() >= 0.0 and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.05
