"""The oracle's strided-subset advance (oracle_advance_points, used by the
full-scale GPU parity tests and the bench's CPU legs) equals the literal
lane-batched reference loop (oracle_advance) on the same points.  CPU only."""

import numpy as np
import pytest

from conftest import assert_bitwise
from oracle import oracle as orc
from paper_2402_17580_b200 import sources
from paper_2402_17580_b200.integrator import IntegratorConfig
from paper_2402_17580_b200.kinetics import DEFAULT_PARAMS

KP = DEFAULT_PARAMS.kernel_tuple()
CFG = IntegratorConfig(scheme="explicit").kernel_tuple()


@pytest.mark.parametrize("cfg_id,n,step0,nsteps", [(0, 256, 1500, 600), (2, 192, 1800, 500),
                                                   (4, 256, 0, 400), (4, 128, 20000, 300)])
def test_subset_equals_full_loop(cfg_id, n, step0, nsteps):
    src = sources.source_for_config(cfg_id)
    g = src.tempgen(point_offset=0)
    full = orc.gen_initial_state(g, n)
    full.temperature_old[:] = orc.gen_temperature(g, n, step0)
    full.temperature_new[:] = full.temperature_old
    pts = np.arange(n, dtype=np.int64)
    sub = orc.gen_initial_points(g, pts)
    sub.temperature_old[:] = full.temperature_old
    sub.temperature_new[:] = full.temperature_old
    rf = orc.advance(full, g, step0, nsteps, KP, CFG, lanes=8)
    rs = orc.advance_points(sub, pts, g, step0, nsteps, KP, CFG, threads=2)
    for k in ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old", "temperature_new"):
        assert_bitwise(getattr(sub, k), getattr(full, k), k)
    act = full.seed_active != 0
    assert np.array_equal(sub.seed_active, full.seed_active)
    assert_bitwise(sub.seed_tracked[act], full.seed_tracked[act], "seed_tracked")
    assert np.array_equal(rs["martensite"], rf["martensite"])
    assert np.array_equal(rs["switches"], rf["switches"])
    assert np.array_equal(rs["totals"], rf["totals"])


def test_subset_is_keyed_by_global_index():
    """A strided subset of a shard at offset 4096 equals those points of the
    contiguous shard."""
    src = sources.source_for_config(4)
    off, n = 4096, 512
    g = src.tempgen(point_offset=off)
    full = orc.gen_initial_state(g, n)
    full.temperature_old[:] = orc.gen_temperature(g, n, 0)
    full.temperature_new[:] = full.temperature_old
    orc.advance(full, g, 0, 300, KP, CFG, lanes=8)
    pts = np.arange(off, off + n, 37, dtype=np.int64)
    sub = orc.gen_initial_points(src.tempgen(point_offset=0), pts)
    orc.advance_points(sub, pts, src.tempgen(point_offset=0), 0, 300, KP, CFG, threads=2)
    for k in ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old"):
        assert_bitwise(getattr(sub, k), getattr(full, k)[pts - off], k)
