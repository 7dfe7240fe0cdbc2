"""Scan path host logic, mirroring the reference's test_scanpath.py
(path-file grammar, error line numbers, round trip, beam timeline)."""

import pytest

from paper_2402_17580_b200.scanpath import (PathError, ScanPath, ScanSegment, beam_position,
                                            beam_timeline, parse_path_file, serialize_path,
                                            serpentine)

MM = 1e-3


def test_parse_minimal_and_comments():
    path = parse_path_file("layer 0\nsegment 0 0 1e-3 0 0.96 180\n")
    assert len(path.segments) == 1 and path.segments[0].speed == 0.96 and path.dwell == 1.0
    path = parse_path_file("# scan program\ndwell 0.5\nlayer 0\nsegment 0 0 1e-3 0 0.96 180 # t\n")
    assert path.dwell == 0.5


def test_parse_errors_carry_line_numbers():
    with pytest.raises(PathError, match="line 2"):
        parse_path_file("layer 0\nsegment 0 0 1 1\n")
    with pytest.raises(PathError, match="line 1"):
        parse_path_file("segment 0 0 1 1 0 100\n")
    with pytest.raises(PathError, match="line 3"):
        parse_path_file("layer 2\nsegment 0 0 1 1 1 0\nlayer 1\n")
    with pytest.raises(PathError, match="line 1"):
        parse_path_file("orbit 1 2 3\n")
    with pytest.raises(PathError, match="line 1"):
        parse_path_file("dwell -1\n")
    with pytest.raises(PathError, match="line 1"):
        parse_path_file("layer x\n")


def test_round_trip():
    segs = serpentine((0.0, 0.0, 1.0 * MM, 1.0 * MM), 0.08 * MM, 0.96, 180.0, layer=0)
    segs += serpentine((0.0, 0.0, 1.0 * MM, 1.0 * MM), 0.08 * MM, 0.96, 180.0, layer=1)
    path = ScanPath(segs, dwell=0.5)
    again = parse_path_file(serialize_path(path))
    assert again.dwell == path.dwell and again.segments == path.segments


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
