"""GPU parity of the coupled layer build: run_build (thermal.py:498-589) on
the reference tests' micro geometry (test_thermal.py:33-43, :192-200), every
thermal and kinetics step on the device, against the reference's own run
(tests/golden/build.npz, from tests/golden/make_golden.py): final
temperatures, r_c, voxel state, all kinetics arrays and every probe row,
bit for bit; plus the reference tests' physical checks."""

import numpy as np
import pytest

from conftest import FIELD_NAMES, assert_bitwise, load_golden

pytestmark = pytest.mark.gpu

G = load_golden("build.npz")
CASES = sorted({k.split("/")[0] for k in G.files
                if k.split("/")[0] not in ("cooldown", "geometry", "helpers")})
MM = 1e-3


@pytest.fixture(scope="module")
def pkg():
    import paper_2402_17580_b200 as p
    return p


def _run(pkg, name, **kw):
    from paper_2402_17580_b200 import scanpath as sp, thermal as th
    geom = th.BuildGeometry(plate_size=(0.6 * MM, 0.6 * MM, 0.15 * MM),
                            part_size=(0.4 * MM, 0.4 * MM, 0.1 * MM), voxel=0.05 * MM)
    s = G[f"{name}/sched"]
    sched = th.BuildSchedule(dt_active=float(s[0]), interlayer_dwell=float(s[1]),
                             initial_dwell_steps=int(s[2]), growth_every=int(s[3]),
                             dt_max=float(s[4]), final_cooldown=float(s[5]),
                             preheat=float(s[6]), room=float(s[7]))
    strategy = getattr(sp, str(G[f"{name}/strategy"]))
    power = float(G[f"{name}/power"])
    segs = []
    for layer in range(geom.grid[3]):
        segs.extend(strategy(geom.part_extent, 0.08 * MM, 0.96, power, layer))
    scan = sp.ScanPath(segs, dwell=sched.interlayer_dwell)
    cfg = pkg.IntegratorConfig(scheme=str(G[f"{name}/scheme"]))
    return th.run_build(geom, scan, sched, integrator_config=cfg,
                        probe_points=[(0.3 * MM, 0.3 * MM, 0.17 * MM),
                                      (0.1 * MM, 0.2 * MM, 0.05 * MM)], **kw)


@pytest.mark.parametrize("name", CASES)
def test_run_build_matches_reference(pkg, name):
    field, fields, probes = _run(pkg, name)
    h = fields.to_host()
    for k in FIELD_NAMES:
        assert_bitwise(h[k], G[f"{name}/{k}"], f"{name}:{k}")
    assert_bitwise(field.r_c.cpu().numpy(), G[f"{name}/r_c"], f"{name}:r_c")
    assert np.array_equal(field.state.cpu().numpy(), G[f"{name}/state"])
    assert field.z_top == int(G[f"{name}/z_top"])
    for i in range(2):
        got = np.array(probes[i], dtype=np.float64).reshape(-1, 5)
        assert_bitwise(got, G[f"{name}/probe{i}"], f"{name}:probe{i}")


def test_build_physics(pkg):
    """test_thermal.py:206-215 / :218-228 / :244-257 on the GPU build."""
    from paper_2402_17580_b200 import thermal as th
    field, fields, probes = _run(pkg, "serp180")
    state = field.state.cpu().numpy()
    rc = field.r_c.cpu().numpy()
    melted = (state == th.STATE_POWDER) & (rc >= 1.0)
    assert melted.sum() > 0
    flat = melted.ravel()
    assert np.all(fields.host("x_alpha_m")[flat] > 0.88)
    assert np.all(np.abs(fields.host("x_beta")[flat] - 0.1) < 0.02)
    field0, fields0, _ = _run(pkg, "zero")
    m = field0.active_mask().cpu().numpy()
    assert np.allclose(field0.temperature_old.cpu().numpy()[m], 293.0, atol=1e-6)
    snaps = []
    _run(pkg, "serp180", snapshot_hook=lambda label, t, f, kf: snaps.append(
        f.r_c.cpu().numpy().copy()))
    assert all(np.all(b >= a - 1e-15) for a, b in zip(snaps, snaps[1:]))


def test_pointwise_helpers_match_reference(pkg):
    """thermal.py:124-165 (the exponentials through the device fast_exp)."""
    from paper_2402_17580_b200 import thermal as th
    t, rc = G["helpers/t"], G["helpers/rc"]
    assert_bitwise(th.conductivity(t, rc), G["helpers/conductivity"], "conductivity")
    assert_bitwise(th.update_consolidation(rc, t, G["helpers/powder"]),
                   G["helpers/update_consolidation"], "update_consolidation")
    assert_bitwise(th.surface_losses(t), G["helpers/surface_losses"], "surface_losses")
    assert_bitwise(th.source_term(G["helpers/x"], G["helpers/y"], G["helpers/zb"], 4e-4, 5e-4),
                   G["helpers/source_term"], "source_term")
