"""Scan path host logic, mirroring the reference's test_scanpath.py
(beam timeline, segment validation)."""

import pytest

from paper_2402_17580_b200.scanpath import (PathError, ScanSegment, beam_position,
                                            beam_timeline)

def test_beam_position_piecewise_linear():
    segs = [ScanSegment(0, 0, 1e-3, 0, 1.0, 180.0), ScanSegment(1e-3, 0, 1e-3, 2e-3, 1.0, 180.0)]
    spans = beam_timeline(segs)
    assert spans[0] == (0.0, pytest.approx(1e-3)) and spans[1][1] == pytest.approx(3e-3)
    x, y, _, on = beam_position(segs, 0.5e-3)
    assert (x, y, on) == (pytest.approx(0.5e-3), 0.0, True)
    assert not beam_position(segs, 5e-3)[3]


def test_segment_validation():
    for args in ((0, 0, 1, 1, 0.0, 100.0), (0, 0, 1, 1, 1.0, -5.0), (0, 0, 0, 0, 1.0, 100.0)):
        with pytest.raises(PathError):
            ScanSegment(*args)
