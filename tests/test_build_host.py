"""Host logic of the layer build (thermal.py:362-495, scanpath.py:58-131)
against values recorded from the reference (tests/golden/build.npz)."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2402_17580_b200 import scanpath as sp
from paper_2402_17580_b200 import thermal as th

G = load_golden("build.npz")


def test_cooldown_steps_match_reference():
    keys = [k for k in G.files if k.startswith("cooldown/")]
    assert keys
    for k in keys:
        dur, init, dtmax = k.split("/")[1].split("_")
        got = th.cooldown_steps(float(dur), th.BuildSchedule(dt_max=float(dtmax)), int(init))
        assert np.array_equal(np.array(got), G[k]), k


def test_geometry_matches_reference():
    g = th.BuildGeometry()
    assert g.grid == tuple(G["geometry/default_grid"])
    assert np.array_equal(np.array(g.part_box), G["geometry/default_part_box"])
    assert np.array_equal(np.array(g.part_extent), G["geometry/default_part_extent"])
    with pytest.raises(ValueError):
        th.BuildGeometry(plate_size=(0.4e-3, 0.4e-3, 0.1e-3), part_size=(1e-3, 1e-3, 1e-4))


def test_scan_path_grouping_and_islands():
    segs = []
    for layer in range(3):
        segs.extend(sp.serpentine((0, 0, 4e-4, 4e-4), 8e-5, 0.96, 180.0, layer))
    path = sp.ScanPath(segs, dwell=0.02)
    assert path.layers() == [0, 1, 2]
    assert all(s.layer == 1 for s in path.layer_segments(1))
    assert path.active_time(0) == pytest.approx((6 * 4e-4 + 5 * 8e-5) / 0.96)
    with pytest.raises(sp.PathError):
        sp.ScanPath(list(reversed(segs)))
    with pytest.raises(sp.PathError):
        sp.ScanPath(segs, dwell=-1.0)
    isl = sp.four_islands((0, 0, 4e-4, 4e-4), 8e-5, 0.96, 180.0)
    # island order (-x,-y), (+x,-y), (-x,+y), (+x,+y); no move crosses a boundary
    assert isl[0].x0 == 0.0 and isl[0].y0 == 0.0
    for s in isl:
        assert (s.x0 <= 2e-4) == (s.x1 <= 2e-4) or min(s.x0, s.x1) == 2e-4
