"""Multi-rank logic of the multi-GPU driver on CPU: torch.distributed with
the gloo backend, world_size 2 and 3, the oracle standing in for the GPU
kernels.  The decomposition must reproduce the single-process result bit
for bit (point shards: generators keyed by global index; z-slabs: halo
exchange + slab-form stencil)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_17580_b200 import distributed as D
from paper_2402_17580_b200 import sources
from paper_2402_17580_b200.integrator import IntegratorConfig
from paper_2402_17580_b200.kinetics import DEFAULT_PARAMS

KP = DEFAULT_PARAMS.kernel_tuple()
CFG = IntegratorConfig().kernel_tuple()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def test_shard_and_slab_ranges():
    for n in (0, 31, 4096, 1 << 20, 1000003):
        for w in (1, 2, 3, 8):
            edges = [D.shard_range(n, r, w) for r in range(w)]
            assert edges[0][0] == 0 and edges[-1][1] == n
            for (a, b), (c, d) in zip(edges, edges[1:]):
                assert b == c and a <= b
                assert b % 32 == 0 or b == n
    for w in (1, 2, 4, 8):
        sl = [D.slab_range(256, r, w) for r in range(w)]
        assert sl[0][0] == 0 and sl[-1][1] == 256
        assert all(b - a == 256 // w for a, b in sl)


def _sharded_worker(rank, world, port, q):
    from oracle import oracle as orc
    _init(rank, world, port)
    src = sources.source_for_config(0)
    n_total, nsteps = 1000, 1500
    lo, hi = D.shard_range(n_total, rank, world)
    g = src.tempgen(point_offset=lo)
    f = orc.gen_initial_state(g, hi - lo)
    t0 = orc.gen_temperature(g, hi - lo, 0)
    f.temperature_old[:] = t0
    f.temperature_new[:] = t0
    r = orc.advance(f, g, 0, nsteps, KP, CFG, lanes=8, snapshot_every=500)
    sums = torch.from_numpy(r["sums"].copy())
    D.allreduce_sum(sums)
    tot = torch.from_numpy(r["totals"].astype(np.int64))
    D.allreduce_sum(tot)
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, f.states()))
    if rank == 0:
        q.put((sums.numpy(), tot.numpy(), gathered))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_point_shards_equal_single_run(world):
    from oracle import oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_sharded_worker, args=(world, _free_port(), q), nprocs=world,
                       start_method="spawn")
    sums, tot, gathered = q.get()
    src = sources.source_for_config(0)
    g = src.tempgen(point_offset=0)
    f = orc.gen_initial_state(g, 1000)
    t0 = orc.gen_temperature(g, 1000, 0)
    f.temperature_old[:] = t0
    f.temperature_new[:] = t0
    r = orc.advance(f, g, 0, 1500, KP, CFG, lanes=8, snapshot_every=500)
    st = np.concatenate([s for _, s in sorted(gathered, key=lambda x: x[0])])
    assert np.array_equal(st.view(np.int64), f.states().view(np.int64))
    np.testing.assert_allclose(sums, r["sums"], rtol=1e-12)
    assert np.array_equal(tot, r["totals"].astype(np.int64))


NZ, NY, NX = 12, 10, 14
H, DT, NSTEPS = 20e-6, 1e-6, 60


def _coupled_reference():
    from oracle import oracle as orc
    from paper_2402_17580_b200 import _abi
    from paper_2402_17580_b200.thermal import DEFAULT_THERMAL, HeatSource
    n = NZ * NY * NX
    f = orc.HostFields(np.full(n, 0.9), np.zeros(n), np.full(n, 0.1), np.full(n, 353.0),
                       np.full(n, 353.0))
    ones, built = np.ones((NZ, NY, NX)), np.full((NZ, NY, NX), 2, np.uint8)
    src = HeatSource(w_eff=87.5, radius=50e-6, h_powder=H)
    for k in range(NSTEPS):
        beam = (60e-6 + 2e-6 * k, 100e-6, 87.5, True)
        a = _abi.stencil_args(NX, NY, NZ, NZ, DT, H, beam=beam, source=src, losses=False,
                              bottom=353.0, all_built=True)
        orc.stencil_step(f.temperature_old.reshape(NZ, NY, NX),
                         f.temperature_new.reshape(NZ, NY, NX), ones, built,
                         DEFAULT_THERMAL.kernel_tuple(), a)
        orc.step_all(f, DT, KP, CFG, n_lanes=8)
    return f


def _slab_worker(rank, world, port, q, overlap=True):
    from oracle import oracle as orc
    from paper_2402_17580_b200 import _abi
    from paper_2402_17580_b200.thermal import DEFAULT_THERMAL, HeatSource
    _init(rank, world, port)
    z0, z1 = D.slab_range(NZ, rank, world)
    zb, ze = max(z0 - 1, 0), min(z1 + 1, NZ)
    ns = ze - zb
    t_old = torch.full((ns, NY, NX), 353.0, dtype=torch.float64)
    t_new = t_old.clone()
    plane = NY * NX
    own = (z1 - z0) * plane
    state = {k: np.zeros(own) for k in ("xs", "xm", "xb")}
    state["xs"][:] = 0.9
    state["xb"][:] = 0.1
    seeds = (np.zeros(own), np.zeros(own, np.uint8), np.zeros(own, np.uint8))
    ones, built = np.ones((ns, NY, NX)), np.full((ns, NY, NX), 2, np.uint8)
    src = HeatSource(w_eff=87.5, radius=50e-6, h_powder=H)
    tp = DEFAULT_THERMAL.kernel_tuple()
    beam_k = [0]

    def stencil(src_t, dst_t, args):
        orc.stencil_step(src_t.numpy(), dst_t.numpy(), ones, built, tp, args)

    def step(lo, hi, dt):
        to = t_old.view(-1).numpy()[lo:hi]
        tn = t_new.view(-1).numpy()[lo:hi]
        hf = orc.HostFields(state["xs"], state["xm"], state["xb"], to, tn, *seeds)
        orc.step_all(hf, dt, KP, CFG, n_lanes=8)
        state["xs"][:], state["xm"][:], state["xb"][:] = hf.x_alpha_s, hf.x_alpha_m, hf.x_beta
        seeds[0][:], seeds[1][:], seeds[2][:] = hf.seed_tracked, hf.seed_active, hf.seed_direction
        to[:] = hf.temperature_old

    drv = D.SlabCoupledDriver(NZ, NY, NX, rank, world, t_old, t_new, stencil, step,
                              D.torch_exchange, overlap=overlap)

    def args_for(slab):
        k = beam_k[0]
        beam = (60e-6 + 2e-6 * k, 100e-6, 87.5, True)
        return _abi.stencil_args(NX, NY, NZ, NZ, DT, H, beam=beam, source=src, losses=False,
                                 bottom=353.0, all_built=True, slab=slab)

    for k in range(NSTEPS):
        beam_k[0] = k
        drv.run_step(DT, args_for)
    t_all = D.gather_planes(t_old, z0, z1, zb, NZ, world, rank)
    xs_all = [None] * world
    dist.all_gather_object(xs_all, (z0, state["xs"].copy(), state["xm"].copy(),
                                    state["xb"].copy()))
    if rank == 0:
        q.put((t_all.numpy(), xs_all))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,overlap", [(2, False), (2, True), (3, True), (7, True)])
def test_zslab_halo_exchange_equals_whole_grid(world, overlap):
    """Blocking swap and the overlapped schedule (edge planes, async halo
    send of T_{n+1}, interior + kinetics) both equal the whole-grid run
    bitwise; world 7 puts 1- and 2-plane slabs (no interior) in play."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_slab_worker, args=(world, _free_port(), q, overlap), nprocs=world,
                       start_method="spawn")
    t_all, parts = q.get()
    ref = _coupled_reference()
    assert np.array_equal(t_all.reshape(-1).view(np.int64), ref.temperature_old.view(np.int64))
    parts = sorted(parts, key=lambda p: p[0])
    for i, name in ((1, "x_alpha_s"), (2, "x_alpha_m"), (3, "x_beta")):
        got = np.concatenate([p[i] for p in parts])
        assert np.array_equal(got.view(np.int64), getattr(ref, name).view(np.int64)), name
    assert ref.temperature_old.max() > 600.0
