"""Pin the CPU oracle to the REAL reference: every golden fixture in
tests/golden/ (made by tests/golden/make_golden.py from ti64micro itself)
must be reproduced bit for bit.  CPU only."""

import numpy as np
import pytest

from conftest import FIELD_NAMES, assert_bitwise, golden_cases, load_golden
from oracle import oracle as orc
from paper_2402_17580_b200 import sources
from paper_2402_17580_b200.kinetics import DEFAULT_PARAMS
from paper_2402_17580_b200.integrator import IntegratorConfig

KP = DEFAULT_PARAMS.kernel_tuple()
CFG = IntegratorConfig(scheme="explicit").kernel_tuple()

STEPS = golden_cases(load_golden("steps.npz"))


def test_fastmath_bitwise():
    g = load_golden("fastmath.npz")
    assert_bitwise(orc.fast_exp(g["x_exp"]), g["y_exp"], "fast_exp")
    assert_bitwise(orc.fast_ln(g["x_ln"]), g["y_ln"], "fast_ln")
    assert_bitwise(orc.fast_pow(g["a_pow"], g["x_pow"]), g["y_pow"], "fast_pow")


def _fields(case, prefix):
    return orc.HostFields(*[case[prefix + k] for k in FIELD_NAMES])


@pytest.mark.parametrize("name", sorted(STEPS))
def test_step_cases_bitwise(name):
    case = STEPS[name]
    f = _fields(case, "in_")
    lanes = int(case["lanes"])
    threads = 2 if "thr2" in name else 1
    for s in range(int(case["nsteps"])):
        if "t_seq" in case:
            f.temperature_new[:] = case["t_seq"][s]
        rc = orc.step_all(f, float(case["dt"]), KP, CFG, n_lanes=lanes, threads=threads)
        assert rc == 0
    for k in FIELD_NAMES:
        assert_bitwise(getattr(f, k), case["out_" + k], f"{name}:{k}")


def test_history_bitwise():
    for name, case in golden_cases(load_golden("history.npz")).items():
        out = orc.history(case["times"], case["temps"], case["out"][0], KP, CFG)
        assert_bitwise(out, case["out"], name)


@pytest.mark.parametrize("fname,src", [
    ("advance_cfg0.npz", None),
    ("advance_cfg1_small.npz", sources.RosenthalRaster(nx=32, ny=32, nz=4)),
    ("advance_cfg2.npz", None),
    ("advance_cfg4.npz", None),
])
def test_advance_bitwise(fname, src):
    g = load_golden(fname)
    cfg_id = int(g["cfg"])
    src = src or sources.source_for_config(cfg_id)
    n, nsteps = int(g["n"]), int(g["nsteps"])
    beam = src.beam_table(nsteps + 1) if cfg_id == 1 else None
    gen = src.tempgen(point_offset=int(g["point_offset"]),
                      beam_ptr=None if beam is None else beam.ctypes.data,
                      beam_steps=0 if beam is None else len(beam))
    f = orc.gen_initial_state(gen, n)
    t0 = orc.gen_temperature(gen, n, 0)
    f.temperature_old[:] = t0
    f.temperature_new[:] = t0
    r = orc.advance(f, gen, 0, nsteps, KP, CFG, lanes=int(g["lanes"]),
                    snapshot_every=int(g["snap_every"]), threads=4)
    for k in FIELD_NAMES:
        assert_bitwise(getattr(f, k), g["out_" + k], f"{fname}:{k}")
    assert np.array_equal(r["martensite"], g["martensite"])
    assert np.array_equal(r["switches"], g["switches"])
    assert np.array_equal(r["totals"], g["totals"])
    # sums: the golden used numpy's pairwise summation; the oracle sums in order
    np.testing.assert_allclose(r["sums"], g["sums"], rtol=1e-12, atol=1e-12)


def test_stencil_general_bitwise():
    c = golden_cases(load_golden("stencil.npz"))["general"]
    from paper_2402_17580_b200.thermal import DEFAULT_THERMAL
    from paper_2402_17580_b200 import _abi
    nz, ny, nx = c["src"].shape
    a = _abi.StencilArgs(nx=nx, ny=ny, nz=nz, z_top=int(c["z_top"]), dt=float(c["dt"]),
                         h=float(c["h"]), beam_x=float(c["beam"][0]),
                         beam_y=float(c["beam"][1]), source_on=1, losses_on=1,
                         bc_bottom_on=1, all_built=0, src_peak=float(c["src_peak"]),
                         src_r2inv=float(c["src_r2inv"]), bc_bottom=293.0,
                         z_base=0, nz_stored=nz, z_begin=0, z_end=int(c["z_top"]))
    dst = c["src"].copy()
    rc = c["rc_in"].copy()
    orc.stencil_step(c["src"].copy(), dst, rc, c["state"].copy(),
                     DEFAULT_THERMAL.kernel_tuple(), a)
    assert_bitwise(dst, c["dst"], "stencil dst")
    assert_bitwise(rc, c["rc_out"], "stencil r_c")


def test_stencil_built_sequence_bitwise():
    c = golden_cases(load_golden("stencil.npz"))["built"]
    from paper_2402_17580_b200.thermal import DEFAULT_THERMAL, HeatSource
    from paper_2402_17580_b200 import _abi
    seq = c["seq"]
    nz, ny, nx = seq.shape[1:]
    h = 20e-6
    src = HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=h)
    t = np.full((nz, ny, nx), 353.0)
    rc = np.ones_like(t)
    state = np.full(t.shape, 2, np.uint8)
    for k in range(seq.shape[0]):
        a = _abi.stencil_args(nx, ny, nz, nz, 1e-6, h,
                              beam=(40e-6 + 20e-6 * k, 150e-6, 0.35 * 250.0, True),
                              source=src, losses=False, bottom=353.0, all_built=True)
        dst = t.copy()
        orc.stencil_step(t, dst, rc, state, DEFAULT_THERMAL.kernel_tuple(), a)
        assert_bitwise(dst, seq[k], f"built step {k}")
        t = dst


CN = golden_cases(load_golden("cn_steps.npz"))


def _cn_cfg(case):
    c = case["cfg"]
    return IntegratorConfig(scheme="crank_nicolson", dt_sub_max=float(c[0]),
                            eps_abs=float(c[1]), eps_rel=float(c[2]),
                            max_fixed_point_iters=int(c[3]), initiation_threshold=float(c[4]),
                            stuck_tol=float(c[5]), max_halvings=int(c[6]))


@pytest.mark.parametrize("name", sorted(CN))
def test_cn_cases_bitwise(name):
    """Crank-Nicolson + halving (batch.py:357-416, :568-674), lane coupling included."""
    case = CN[name]
    cfg = _cn_cfg(case)
    f = _fields(case, "in_")
    lanes = int(case["lanes"])
    dt = float(case["dt"])
    nsub = orc.num_substeps(dt, cfg.dt_sub_max)
    fail = []
    iters = None
    for s in range(int(case["nsteps"])):
        if "t_seq" in case:
            f.temperature_new[:] = case["t_seq"][s]
        rc, iters = orc.run_range_cn(f, KP, cfg.kernel_tuple(), lanes, nsub, dt / nsub)
        if rc != 0:
            fail = list(range(rc - 1, min(rc - 1 + lanes, f.n_points)))
            break
    assert fail == list(case["fail"])
    for k in FIELD_NAMES:
        assert_bitwise(getattr(f, k), case["out_" + k], f"{name}:{k}")
    if case["iters"].size and not fail:
        assert np.array_equal(iters, case["iters"])


def test_cn_history_bitwise():
    for name, case in golden_cases(load_golden("cn_history.npz")).items():
        cfg = IntegratorConfig(scheme="crank_nicolson").kernel_tuple()
        out = orc.history(case["times"], case["temps"], case["out"][0], KP, cfg)
        assert_bitwise(out, case["out"], name)
