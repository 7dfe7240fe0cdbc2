"""Full-scale, full-length parity of the kernels the bench times.

The fused advance kernel (K2) picks a latency instance for small launches
(<= 1184 32-point tasks) and a throughput instance for everything the bench
measures; the per-config goldens are small, so this file pins the
throughput instance at the BASELINE sizes and lengths:

  * config 1, the whole job (2^20 points x 10 000 steps), every point;
  * config 2, the whole job (2^24 x 50 000), every 1024th point, with the
    event counters of the counted instance;
  * config 4, the 2^24-point shard of rank 0 of 8 x 100 000 steps, every
    4096th point;
  * config 3, the first 10 steps of the split coupled step on the full
    512 x 512 x 256 grid, every cell;
  * reference-made goldens of > 37 888 points (tests/golden/advance_large.npz,
    made by tests/golden/make_golden.py --large-only from ti64micro itself).

The oracle (oracle/ti64_oracle.c, pinned to the reference by
test_oracle_golden.py) runs the reference loop on the selected points
(oracle_advance_points: points are independent; generators are keyed by the
global point index).  States are compared bit for bit; seed_tracked where the
seed is active (elsewhere it is lane-width-dependent residue, batch.py:687-692).
Reference: batch.py:762-813 (step_all), test_batch.py:79-85 / :145-150
(lane / thread invariance that makes subsets exact).
"""

import hashlib

import numpy as np
import pytest

from conftest import assert_bitwise, golden_cases, load_golden

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

STATE = ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old")


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2402_17580_b200 as pkg
    from oracle import oracle as orc
    return {"pkg": pkg, "orc": orc, "torch": torch, "dev": torch.device("cuda", 0),
            "kp": pkg.DEFAULT_PARAMS.kernel_tuple(),
            "cfg": pkg.IntegratorConfig().kernel_tuple()}


def _compare_sample(env, f, idx, host, what):
    torch = env["torch"]
    ti = torch.from_numpy(idx).to(env["dev"])
    got = {k: getattr(f, k)[ti].cpu().numpy() for k in STATE + ("seed_active", "seed_tracked",
                                                                "seed_direction")}
    for k in STATE:
        assert_bitwise(got[k], getattr(host, k), f"{what}:{k}")
    assert np.array_equal(got["seed_active"], host.seed_active), f"{what}: seed_active"
    act = host.seed_active != 0
    assert_bitwise(got["seed_tracked"][act], host.seed_tracked[act], f"{what}: seed_tracked")
    assert np.array_equal(got["seed_direction"][act], host.seed_direction[act])


def _oracle_run(env, src, pts, nsteps, beam=None):
    orc = env["orc"]
    kw = {} if beam is None else {"beam_ptr": beam.ctypes.data, "beam_steps": len(beam)}
    gen = src.tempgen(point_offset=0, **kw)
    h = orc.gen_initial_points(gen, pts)
    r = orc.advance_points(h, pts, gen, 0, nsteps, env["kp"], env["cfg"])
    return h, r


def test_config1_whole_job_every_point(env):
    pkg = env["pkg"]
    src = pkg.source_for_config(1)
    n = src.n_points
    f = pkg.init_from_source(src, n)
    pkg.advance(f, 10_000, src, snapshot_every=1000)  # the bench's instance (uncounted)
    beam = np.ascontiguousarray(src.beam_table(10_001))
    pts = np.arange(n, dtype=np.int64)
    h, _ = _oracle_run(env, src, pts, 10_000, beam)
    assert float(h.x_alpha_m.max()) > 0.0  # martensite formed under the raster
    _compare_sample(env, f, pts, h, "config1 job")


def test_config2_whole_job_every_1024th_point_with_counters(env):
    pkg, torch = env["pkg"], env["torch"]
    src = pkg.source_for_config(2)
    n = 1 << 24
    f = pkg.init_from_source(src, n)
    timed = f.copy()
    cnt = pkg.EventCounters(n, env["dev"])
    pkg.advance(f, 50_000, src, snapshot_every=5000, counters=cnt)
    pkg.advance(timed, 50_000, src, snapshot_every=5000)
    for k in pkg.batch.NAMES:  # counted instance == timed instance, every point
        a, b = getattr(f, k), getattr(timed, k)
        if a.dtype == torch.float64:
            a, b = a.view(torch.int64), b.view(torch.int64)
        assert torch.equal(a, b), f"counted != timed in {k}"
    del timed
    pts = np.arange(0, n, 1024, dtype=np.int64)
    h, r = _oracle_run(env, src, pts, 50_000)
    _compare_sample(env, f, pts, h, "config2 job")
    ti = torch.from_numpy(pts).to(env["dev"])
    assert np.array_equal(cnt.martensite[ti].cpu().numpy().astype(np.uint32), r["martensite"])
    assert np.array_equal(cnt.switches[ti].cpu().numpy().astype(np.uint32), r["switches"])
    assert int(r["totals"][6]) > 0 and int(r["totals"][7]) > 0  # events did happen


def test_config4_rank0_of_8_shard_every_4096th_point(env):
    pkg = env["pkg"]
    from paper_2402_17580_b200.distributed import shard_range
    src = pkg.source_for_config(4)
    lo, hi = shard_range(1 << 27, 0, 8)
    f = pkg.init_from_source(src, hi - lo, point_offset=lo)
    for s0 in range(0, 100_000, 20_000):
        pkg.advance(f, 20_000, src, step0=s0, point_offset=lo)
    pts = np.arange(0, hi - lo, 4096, dtype=np.int64)
    h, _ = _oracle_run(env, src, pts + lo, 100_000)
    _compare_sample(env, f, pts, h, "config4 shard")


def test_config4_last_shard_window_every_4096th_point(env):
    """Rank 7 of 8 (global offset 7 * 2^24) over the bench's start region."""
    pkg = env["pkg"]
    from paper_2402_17580_b200.distributed import shard_range
    src = pkg.source_for_config(4)
    lo, hi = shard_range(1 << 27, 7, 8)
    f = pkg.init_from_source(src, hi - lo, point_offset=lo)
    pkg.advance(f, 21_000, src, point_offset=lo)
    pts = np.arange(0, hi - lo, 4096, dtype=np.int64)
    h, _ = _oracle_run(env, src, pts + lo, 21_000)
    _compare_sample(env, f, pts, h, "config4 rank 7")


def test_config3_first_10_full_grid_steps(env):
    pkg, orc = env["pkg"], env["orc"]
    from paper_2402_17580_b200 import _abi, scanpath, thermal as th
    nz, ny, nx = 256, 512, 512
    h, dt, nsteps = 20e-6, 1e-6, 10
    dom = th.CoupledDomain(nx=nx, ny=ny, nz=nz, h=h)
    src = th.HeatSource(w_eff=0.35 * 250.0, radius=50e-6, h_powder=h)
    segs = scanpath.serpentine((1e-3, 1e-3, 9.24e-3, 9.24e-3), 80e-6, 1.0, 0.35 * 250.0)
    beams = scanpath.beam_schedule(segs, nsteps, dt)
    dom.run(nsteps, dt, beams, src)  # the bench's path: the split coupled step
    n = nx * ny * nz
    hf = orc.HostFields(np.full(n, 0.9), np.zeros(n), np.full(n, 0.1), np.full(n, 353.0),
                        np.full(n, 353.0))
    ones, built = np.ones((nz, ny, nx)), np.full((nz, ny, nx), 2, np.uint8)
    tp = th.DEFAULT_THERMAL.kernel_tuple()
    for k in range(nsteps):
        a = _abi.stencil_args(nx, ny, nz, nz, dt, h, beam=beams[k], source=src, losses=False,
                              bottom=353.0, all_built=True)
        orc.stencil_step(hf.temperature_old.reshape(nz, ny, nx),
                         hf.temperature_new.reshape(nz, ny, nx), ones, built, tp, a)
        orc.step_all(hf, dt, env["kp"], env["cfg"], n_lanes=8, threads=orc.max_threads())
    assert float(hf.temperature_old.max()) > 400.0  # the beam heated the top plane
    got = dom.fields.to_host()
    for k in ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old"):
        assert_bitwise(got[k], getattr(hf, k), f"config3 {k}")


LARGE = golden_cases(load_golden("advance_large.npz"))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(LARGE))
def test_reference_large_golden(env, name):
    """Pinned to the reference directly (no oracle in between), at sizes that
    select K2's throughput instance."""
    pkg = env["pkg"]
    case = LARGE[name]
    cfg_id, n, off, nsteps = (int(x) for x in case["args"])
    assert (n + 31) // 32 > 1184  # the throughput instance
    src = pkg.source_for_config(cfg_id)
    f = pkg.init_from_source(src, n, point_offset=off)
    pkg.advance(f, nsteps, src, point_offset=off)
    got = f.to_host()
    for k in ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old", "seed_active"):
        assert_bitwise(got[k][:4096], case["head_" + k], f"{name}:{k} head")
        assert _sha(got[k]) == str(case["sha_" + k]), f"{name}: {k} digest"
    act = got["seed_active"] != 0
    assert _sha(got["seed_tracked"][act]) == str(case["sha_seed_tracked_active"])
