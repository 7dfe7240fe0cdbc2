"""Host-side report formats against the reference (tests/golden/report.npz):
RooflineReport text (bench.py:208-257) and the CSV writer (output.py:44-55)."""

import numpy as np

from conftest import load_golden
from paper_2402_17580_b200.bench import RooflineReport
from paper_2402_17580_b200.output import write_probe_csv

G = load_golden("report.npz")


def test_roofline_report_text():
    rep = RooflineReport(6538.0, 34120.5, 0.57)
    rep.add_run("explicit_b1", 123456789, 72 * 400000, 0.0123)
    rep.add_run("cn_b100", 987654321, 72 * 400000, 0.0456)
    assert rep.to_csv() == str(G["roofline/csv"])
    assert rep.to_gnuplot() == str(G["roofline/gnuplot"])
    assert rep.respects_ceilings() == bool(G["roofline/respects"])
    assert rep.memory_bound_dof_rate == float(G["roofline/mem_dof"])


def test_probe_csv_round_trip(tmp_path):
    text = str(G["csv/probe0"])
    lines = text.splitlines()
    rows = [tuple(float(v) for v in ln.split(",")) for ln in lines[1:]]
    p = tmp_path / "probe.csv"
    write_probe_csv(p, rows)
    assert p.read_text() == text
