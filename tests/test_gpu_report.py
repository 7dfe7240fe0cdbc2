"""GPU side of the reporting formats: count_flops on the reference's layouts,
VTK snapshots and probe CSV of a device run_build, byte-identical to the
reference's files (tests/golden/report.npz); device roofline baselines."""

import numpy as np
import pytest

from conftest import FIELD_NAMES, load_golden

pytestmark = pytest.mark.gpu

G = load_golden("report.npz")
MM = 1e-3


@pytest.fixture(scope="module")
def pkg():
    import paper_2402_17580_b200 as p
    return p


@pytest.mark.parametrize("block", [1, 10, 100])
def test_count_flops_matches_reference(pkg, block):
    from paper_2402_17580_b200 import bench as pb
    lay = pkg.GlobalFields(*[G[f"layout{block}/{k}"] for k in FIELD_NAMES[:5]])
    for lanes in (1, 8):
        assert pb.count_flops(lay, "explicit", lanes) == int(
            G[f"layout{block}/flops_explicit_l{lanes}"])
    assert pb.count_flops(lay, "crank_nicolson", 8, iters=G[f"layout{block}/iters"]) == int(
        G[f"layout{block}/flops_cn_l8"])


def test_generate_layout_matches_reference(pkg):
    from paper_2402_17580_b200 import bench as pb
    for block in (1, 10, 100):
        lay = pb.generate_layout(block, 1000 + block, seed=block)
        for k in FIELD_NAMES[:5]:
            assert np.array_equal(lay.host(k), G[f"layout{block}/{k}"])


def test_vtk_and_probe_csv_match_reference(pkg, tmp_path):
    from paper_2402_17580_b200 import output, scanpath as sp, thermal as th
    geom = th.BuildGeometry(plate_size=(0.6 * MM, 0.6 * MM, 0.15 * MM),
                            part_size=(0.4 * MM, 0.4 * MM, 0.1 * MM), voxel=0.05 * MM)
    s = G["sched"]
    sched = th.BuildSchedule(dt_active=float(s[0]), interlayer_dwell=float(s[1]),
                             initial_dwell_steps=int(s[2]), growth_every=int(s[3]),
                             dt_max=float(s[4]), final_cooldown=float(s[5]),
                             preheat=float(s[6]), room=float(s[7]))
    segs = []
    for layer in range(geom.grid[3]):
        segs.extend(sp.serpentine(geom.part_extent, 0.08 * MM, 0.96, 180.0, layer))
    scan = sp.ScanPath(segs, dwell=sched.interlayer_dwell)
    got = {}

    def hook(label, t, field, fields):
        p = tmp_path / f"{label}.vtk"
        output.write_vtk_snapshot(p, field, fields, label=label)
        got[label] = p.read_text()

    field, fields, probes = th.run_build(geom, scan, sched, snapshot_hook=hook,
                                         probe_points=[(0.3 * MM, 0.3 * MM, 0.17 * MM)])
    keys = sorted(k[4:] for k in G.files if k.startswith("vtk/"))
    assert sorted(got) == keys
    for k in keys:
        assert got[k] == str(G[f"vtk/{k}"]), k
    p = tmp_path / "probe.csv"
    output.write_probe_csv(p, probes[0])
    assert p.read_text() == str(G["csv/probe0"])


def test_device_baselines_and_throughput(pkg):
    from paper_2402_17580_b200 import bench as pb
    bw = pb.measure_bandwidth(n=1 << 24, repetitions=3)
    pk = pb.measure_peak_flops(repetitions=2)
    assert 1000.0 < bw < 9000.0      # GB/s, HBM3e
    assert 10000.0 < pk < 60000.0    # GFlop/s FP64
    lay = pb.generate_layout(100, 1 << 16)
    dof, med, iters = pb.measure_throughput(lay, "crank_nicolson", repetitions=3, warmup=1)
    assert dof > 0 and med > 0 and iters.shape == (1 << 16,)
    rep = pb.roofline([dict(label="cn", flops=pb.count_flops(lay, "crank_nicolson", 8,
                                                             iters=iters),
                            bytes=72 * lay.n_points, seconds=med)], bw, pk)
    assert rep.respects_ceilings()
