"""GPU parity of K4 (7-point heat stencil, thermal.py:205-287) and of the
coupled config-3 step (thermal.py:541-555) against the reference's golden
fixtures and the CPU oracle, bit for bit."""

import numpy as np
import pytest

from conftest import assert_bitwise, golden_cases, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2402_17580_b200 as pkg
    from paper_2402_17580_b200 import _abi, _lib, thermal
    from oracle import oracle as orc
    return dict(torch=torch, pkg=pkg, abi=_abi, lib=_lib, th=thermal, orc=orc)


def gpu_stencil(env, src, dst, rc, state, args, tp=None):
    import ctypes as C
    torch, lib, abi, th = env["torch"], env["lib"], env["abi"], env["th"]
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda()
         for k, v in dict(src=src, dst=dst, rc=rc, state=state).items()}
    tp = tp or th.DEFAULT_THERMAL.kernel_tuple()
    rcode = lib.require().ti64_stencil_step(lib.ptr(t["src"]), lib.ptr(t["dst"]),
                                            lib.ptr(t["rc"]), lib.ptr(t["state"]),
                                            C.byref(abi.thermal_from(tp)), C.byref(args),
                                            lib.stream_handle())
    lib.check(rcode, "ti64_stencil_step")
    return t["dst"].cpu().numpy(), t["rc"].cpu().numpy()


def test_general_golden(env):
    c = golden_cases(load_golden("stencil.npz"))["general"]
    abi = env["abi"]
    nz, ny, nx = c["src"].shape
    a = abi.StencilArgs(nx=nx, ny=ny, nz=nz, z_top=int(c["z_top"]), dt=float(c["dt"]),
                        h=float(c["h"]), beam_x=float(c["beam"][0]), beam_y=float(c["beam"][1]),
                        source_on=1, losses_on=1, bc_bottom_on=1, all_built=0,
                        src_peak=float(c["src_peak"]), src_r2inv=float(c["src_r2inv"]),
                        bc_bottom=293.0, z_base=0, nz_stored=nz, z_begin=0,
                        z_end=int(c["z_top"]))
    dst, rc = gpu_stencil(env, c["src"], c["src"].copy(), c["rc_in"], c["state"], a)
    assert_bitwise(dst, c["dst"], "general dst")
    assert_bitwise(rc, c["rc_out"], "general r_c")


def test_built_golden_sequence(env):
    c = golden_cases(load_golden("stencil.npz"))["built"]
    abi, th = env["abi"], env["th"]
    seq = c["seq"]
    nz, ny, nx = seq.shape[1:]
    src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=20e-6)
    t = np.full((nz, ny, nx), 353.0)
    ones, built = np.ones_like(t), np.full(t.shape, 2, np.uint8)
    for k in range(seq.shape[0]):
        a = abi.stencil_args(nx, ny, nz, nz, 1e-6, 20e-6,
                             beam=(40e-6 + 20e-6 * k, 150e-6, 0.35 * 250.0, True), source=src,
                             losses=False, bottom=353.0, all_built=True)
        t, _ = gpu_stencil(env, t, t.copy(), ones, built, a)
        assert_bitwise(t, seq[k], f"built step {k}")


@pytest.mark.parametrize("shape", [(37, 45, 70), (24, 8, 33)])
def test_built_vs_oracle_and_general(env, shape):
    """Odd tile remainders; the hoisted-conductivity kernel equals both the
    oracle and the general per-face kernel on an all-built grid."""
    abi, th, orc = env["abi"], env["th"], env["orc"]
    nz, ny, nx = shape
    rng = np.random.default_rng(sum(shape))
    t = 353.0 + rng.uniform(0, 2500.0, shape)
    ones, built = np.ones(shape), np.full(shape, 2, np.uint8)
    src = th.HeatSource(w_eff=87.5, radius=50e-6, h_powder=20e-6)
    for k in range(5):
        beam = (nx * 10e-6 + 7e-6 * k, ny * 9e-6, 87.5, True)
        a = abi.stencil_args(nx, ny, nz, nz, 1e-6, 20e-6, beam=beam, source=src, losses=False,
                             bottom=353.0, all_built=True)
        fast, _ = gpu_stencil(env, t, t.copy(), ones, built, a)
        a.all_built = 0
        gen, _ = gpu_stencil(env, t, t.copy(), ones, built, a)
        ref = t.copy()
        orc.stencil_step(t, ref, ones.copy(), built, th.DEFAULT_THERMAL.kernel_tuple(), a)
        assert_bitwise(fast, ref, f"built {shape} step {k}")
        assert_bitwise(gen, ref, f"general {shape} step {k}")
        t = fast


def test_slab_decomposition_equals_whole_grid(env):
    """z-slabs with 1-plane halos (the multi-GPU layout) reproduce the whole
    grid bit for bit, general kernel with powder/inactive cells and losses."""
    abi, th, orc = env["abi"], env["th"], env["orc"]
    nz, ny, nx = 20, 12, 16
    rng = np.random.default_rng(9)
    t = 293.0 + rng.uniform(0, 3500.0, (nz, ny, nx))
    state = np.full((nz, ny, nx), 2, np.uint8)
    state[12:] = 1
    state[17:] = 0
    rc = np.where(state == 2, 1.0, rng.uniform(0, 1, (nz, ny, nx)))
    z_top = 17
    src = th.HeatSource()
    beam = (0.3e-3, 0.2e-3, 180.0, True)
    a = abi.stencil_args(nx, ny, nz, z_top, 1e-7, 50e-6, beam=beam, source=src, losses=True,
                         bottom=293.0)
    whole_dst, whole_rc = gpu_stencil(env, t, t.copy(), rc, state, a)
    ref, rref = t.copy(), rc.copy()
    orc.stencil_step(t, ref, rref, state, th.DEFAULT_THERMAL.kernel_tuple(), a)
    assert_bitwise(whole_dst, ref, "whole")
    assert_bitwise(whole_rc, rref, "whole rc")
    out = t.copy()
    out_rc = rc.copy()
    for z0, z1 in ((0, 5), (5, 11), (11, 17)):
        zb = max(z0 - 1, 0)
        ze = min(z1 + 1, nz)
        sl = slice(zb, ze)
        sa = abi.stencil_args(nx, ny, nz, z_top, 1e-7, 50e-6, beam=beam, source=src,
                              losses=True, bottom=293.0, slab=(zb, ze - zb, z0, z1))
        d, r = gpu_stencil(env, t[sl], t[sl].copy(), rc[sl], state[sl], sa)
        out[z0:z1] = d[z0 - zb:z1 - zb]
        out_rc[z0:z1] = r[z0 - zb:z1 - zb]
    assert_bitwise(out, ref, "slabs")
    assert_bitwise(out_rc, rref, "slabs rc")


def test_coupled_config3_reduced_vs_oracle(env):
    """Config 3 physics on a reduced grid (16 x 48 x 40, 400 steps of 1e-6 s):
    step_thermal + step_all per step, exactly as run_build's couple, against
    the oracle's stencil + step_all."""
    pkg, abi, th, orc = env["pkg"], env["abi"], env["th"], env["orc"]
    from paper_2402_17580_b200 import scanpath
    nz, ny, nx = 16, 48, 40
    h, dt, nsteps = 20e-6, 1e-6, 400
    dom = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h)
    src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=h)
    segs = scanpath.serpentine((0.2e-3, 0.2e-3, 0.6e-3, 0.7e-3), 80e-6, 1.0, 0.35 * 250.0)
    beams = scanpath.beam_schedule(segs, nsteps, dt)
    dom.run(nsteps, dt, beams, src)
    n = nx * ny * nz
    hf = orc.HostFields(np.full(n, 0.9), np.zeros(n), np.full(n, 0.1), np.full(n, 353.0),
                        np.full(n, 353.0))
    kp = pkg.DEFAULT_PARAMS.kernel_tuple()
    cfg = pkg.IntegratorConfig().kernel_tuple()
    ones, built = np.ones((nz, ny, nx)), np.full((nz, ny, nx), 2, np.uint8)
    tp = th.DEFAULT_THERMAL.kernel_tuple()
    for k in range(nsteps):
        a = abi.stencil_args(nx, ny, nz, nz, dt, h, beam=beams[k], source=src, losses=False,
                             bottom=353.0, all_built=True)
        orc.stencil_step(hf.temperature_old.reshape(nz, ny, nx),
                         hf.temperature_new.reshape(nz, ny, nx), ones, built, tp, a)
        orc.step_all(hf, dt, kp, cfg, n_lanes=8, threads=4)
    got = dom.fields.to_host()
    assert float(hf.temperature_old.max()) > 1000.0  # the beam did heat the block
    for k in ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old", "temperature_new",
              "seed_tracked", "seed_active", "seed_direction"):
        assert_bitwise(got[k], getattr(hf, k), f"coupled {k}")


def test_slab_gpu_driver_single_rank_equals_coupled(env):
    """The multi-GPU slab driver at world size 1 is the coupled domain."""
    th = env["th"]
    from paper_2402_17580_b200 import scanpath
    from paper_2402_17580_b200.distributed import SlabCoupledGPU
    nz, ny, nx, h, dt, nsteps = 12, 40, 40, 20e-6, 1e-6, 200
    src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=h)
    segs = scanpath.serpentine((0.2e-3, 0.2e-3, 0.6e-3, 0.6e-3), 80e-6, 1.0, 87.5)
    beams = scanpath.beam_schedule(segs, nsteps, dt)
    a = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h).run(nsteps, dt, beams, src)
    b = SlabCoupledGPU(nz, ny, nx, h).run(nsteps, dt, beams, src)
    ha, hb = a.fields.to_host(), b.fields.to_host()
    for k in ha:
        assert_bitwise(ha[k], hb[k], f"slab driver {k}")


@pytest.mark.parametrize("lanes", [8, 1])
def test_fused_coupled_equals_unfused(env, lanes):
    """The single-pass K4+kinetics kernel (ping-pong T, idle bitmap) equals the
    reference-shaped stencil + step_all sequence bit for bit."""
    th = env["th"]
    from paper_2402_17580_b200 import scanpath
    nz, ny, nx, h, dt, nsteps = 14, 40, 64, 20e-6, 1e-6, 500
    src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=h)
    segs = scanpath.serpentine((0.25e-3, 0.2e-3, 1.0e-3, 0.6e-3), 80e-6, 1.0, 87.5)
    beams = scanpath.beam_schedule(segs, nsteps, dt)
    a = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h)
    a.run(nsteps // 2, dt, beams, src, fused=False, n_lanes=lanes)
    a.run(nsteps - nsteps // 2, dt, beams[nsteps // 2:], src, fused=False, n_lanes=lanes)
    b = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h)
    b.run(nsteps // 2, dt, beams, src, fused=True, n_lanes=lanes)
    b.run(nsteps - nsteps // 2, dt, beams[nsteps // 2:], src, fused=True, n_lanes=lanes)
    ha, hb = a.fields.to_host(), b.fields.to_host()
    assert ha["temperature_old"].max() > 1500.0
    for k in ha:
        assert_bitwise(ha[k], hb[k], f"fused {k}")


def test_cp_async_pipeline_equals_tma(env, tmp_path):
    """Both K4 pipelines (TMA default; cp.async with TI64_NO_TMA=1) give the
    same bits, for the stencil and the fused coupled step."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    outs = []
    for flag in ("0", "1"):
        out = tmp_path / f"ab_{flag}.npz"
        e = dict(os.environ, TI64_NO_TMA=flag)
        subprocess.run([sys.executable, str(root / "tools" / "stencil_ab.py"), str(out)],
                       env=e, check=True, cwd=root)
        outs.append(np.load(out))
    for k in outs[0].files:
        assert_bitwise(outs[0][k], outs[1][k], f"tma vs cp.async {k}")


def test_split_coupled_step_equals_fused(env, tmp_path):
    """The split coupled step (default: stencil + hot-row bitmap, row scan,
    one warp per listed row) and the fused kernel (split=False) give
    the same bits: temperatures, phase fractions, seed arrays and counters
    after 300 steps of a moving source (hot rows, a transformed trail)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    outs = []
    for mode in ("split", "fused"):
        out = tmp_path / f"mode_{mode}.npz"
        subprocess.run([sys.executable, str(root / "tools" / "stencil_ab.py"), str(out), mode],
                       env=dict(os.environ), check=True, cwd=root)
        outs.append(np.load(out))
    xs = outs[0]["x_alpha_s"]
    assert np.count_nonzero(xs != 0.9) > 0  # the trail exists: split rows were run
    for k in outs[0].files:
        assert_bitwise(outs[0][k], outs[1][k], f"split vs fused {k}")


def _config3_like(th, nz, ny, nx, h, dt, nsteps):
    from paper_2402_17580_b200 import scanpath
    src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=h)
    segs = scanpath.serpentine((0.2e-3, 0.2e-3, 1.0e-3, 0.6e-3), 80e-6, 1.0, 87.5)
    return src, scanpath.beam_schedule(segs, nsteps, dt)


def test_slab_split_single_rank_equals_coupled(env):
    """The slab-form split coupled step at world size 1 (one call per step)
    equals the whole-grid coupled domain, every array bit for bit."""
    th = env["th"]
    from paper_2402_17580_b200.distributed import SlabCoupledGPU
    nz, ny, nx, h, dt, nsteps = 16, 40, 64, 20e-6, 1e-6, 300
    src, beams = _config3_like(th, nz, ny, nx, h, dt, nsteps)
    a = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h).run(nsteps, dt, beams, src)
    b = SlabCoupledGPU(nz, ny, nx, h)
    assert b.split
    b.run(nsteps // 3, dt, beams, src)
    b.run(nsteps - nsteps // 3, dt, beams[nsteps // 3:], src)
    ha, hb = a.fields.to_host(), b.fields.to_host()
    assert ha["temperature_old"].max() > 1500.0
    assert np.count_nonzero(ha["x_alpha_s"] != 0.9) > 0
    for k in ha:
        assert_bitwise(ha[k], hb[k], f"slab split {k}")


@pytest.mark.parametrize("world", [2, 3, 5])
def test_slab_split_emulated_ranks_equal_whole_grid(env, world):
    """The multi-GPU schedule of SlabCoupledGPU (edge planes, halo exchange
    of the new edge planes into the neighbours' next buffers, interior
    planes, swap) with `world` slabs interleaved on one device and the
    exchange done by copies, against the whole grid: every owned cell's
    temperature and kinetics state bit for bit."""
    import torch
    th = env["th"]
    from paper_2402_17580_b200.distributed import SlabCoupledGPU
    nz, ny, nx, h, dt, nsteps = 15, 40, 64, 20e-6, 1e-6, 240
    src, beams = _config3_like(th, nz, ny, nx, h, dt, nsteps)
    a = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h).run(nsteps, dt, beams, src)
    ranks = [SlabCoupledGPU(nz, ny, nx, h, rank=r, world=world) for r in range(world)]

    def exchange():
        for r, s in enumerate(ranks):  # edge planes -> neighbours' halo planes
            lo, hi = s.z0 - s.zb, s.z1 - s.zb
            if r > 0:
                nb = ranks[r - 1]
                nb._nxt[nb.z1 - nb.zb].copy_(s._nxt[lo])
            if r < world - 1:
                nb = ranks[r + 1]
                nb._nxt[nb.z0 - 1 - nb.zb].copy_(s._nxt[hi - 1])

    for s in ranks:
        s.begin(dt, src)
    for k in range(nsteps):
        for s in ranks:
            s.phase_edges(beams[k])
        exchange()
        for s in ranks:
            s.phase_interior(beams[k])
        for s in ranks:
            s.finish_step()
    for s in ranks:
        s.end(nsteps)
    T = torch.cat([s.temperature() for s in ranks], 0).cpu().numpy().ravel()
    ha = a.fields.to_host()
    assert_bitwise(T, ha["temperature_old"], f"world {world} T")
    for k in ("x_alpha_s", "x_alpha_m", "x_beta", "seed_active", "seed_tracked",
              "seed_direction"):
        got = np.concatenate([s.fields.host(k) for s in ranks])
        assert_bitwise(got, ha[k], f"world {world} {k}")


def test_coupled_graph_replay_equals_direct(env):
    """The step loop as a replayed CUDA graph (beam rows from a device table,
    a device step counter) equals the directly launched loop bit for bit."""
    th = env["th"]
    nz, ny, nx, h, dt, nsteps = 16, 40, 64, 20e-6, 1e-6, 301
    src, beams = _config3_like(th, nz, ny, nx, h, dt, nsteps)
    a = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h).run(nsteps, dt, beams, src)
    b = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h).run(nsteps, dt, beams, src, graph=True)
    ha, hb = a.fields.to_host(), b.fields.to_host()
    assert ha["temperature_old"].max() > 1500.0
    for k in ha:
        assert_bitwise(ha[k], hb[k], f"graph {k}")


@pytest.mark.parametrize("nsteps,parts", [(301, (301,)), (400, (3, 100, 297)), (2, (2,))])
def test_coupled_overlapped_kinetics_equals_serial(env, nsteps, parts):
    """Three rotating temperature buffers with the row kinetics of step k on
    a second stream beside the stencil of step k+1 (the default of
    CoupledDomain.run) equal the one-stream ping-pong loop bit for bit, also
    when the run is issued in several calls (buffer roles restart per call)
    and when it is too short to overlap."""
    th = env["th"]
    nz, ny, nx, h, dt = 16, 40, 64, 20e-6, 1e-6
    src, beams = _config3_like(th, nz, ny, nx, h, dt, nsteps)
    a = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h).run(nsteps, dt, beams, src, overlap=False)
    b = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h)
    k = 0
    for p in parts:
        b.run(p, dt, beams[k:k + p], src)
        k += p
    ha, hb = a.fields.to_host(), b.fields.to_host()
    if nsteps > 100:
        assert ha["temperature_old"].max() > 1500.0
        assert np.count_nonzero(ha["x_alpha_s"] != 0.9) > 0
    for key in ha:
        assert_bitwise(ha[key], hb[key], f"overlap {key}")
    assert_bitwise(hb["temperature_old"], hb["temperature_new"], "T_old == T_new at the end")
