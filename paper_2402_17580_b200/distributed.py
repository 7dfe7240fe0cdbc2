"""Multi-GPU driver: one process per GPU (torch.distributed, NCCL on B200).

Two decompositions:

* Pure-ODE configs (0, 1, 2, 4): points are independent, so each rank owns a
  contiguous block of global point indices (aligned to 32 so the reference's
  lane groups, batch.py:531, never straddle ranks) and advances it with the
  fused kernel; the generators are keyed by the GLOBAL point index, so the
  union of the shards is bit-identical to a single-GPU run.  The only
  collective is the final (and per-snapshot) all-reduce of the phase sums,
  histograms and event totals.
* Coupled config 3: z-slabs of the (nz, ny, nx) grid with one halo plane on
  each side.  Every step the ranks swap boundary planes of T_n with their z
  neighbours (point-to-point send/recv), run K4 on their own planes in slab
  form (global boundary conditions by global z index: the Dirichlet plate on
  rank 0, the beam on the rank owning z_top - 1) and then the kinetics step
  on their own cells.

The decomposition logic is backend-agnostic (`SlabCoupledDriver` takes the
stencil and step callables), so it is tested on CPU with the gloo backend and
the oracle, and runs on GPUs with NCCL and the CUDA kernels.
"""

import numpy as np

__all__ = ["shard_range", "slab_range", "ShardedAdvance", "SlabCoupledDriver",
           "allreduce_sum"]


def shard_range(n, rank, world, align=32):
    """Contiguous block [lo, hi) of n points for `rank`, boundaries aligned."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    def edge(r):
        if r >= world:
            return n
        return min(n, (n * r // world) // align * align)
    return edge(rank), edge(rank + 1)


def slab_range(nz, rank, world):
    """Owned z-planes [z0, z1) of `rank` (balanced contiguous slabs)."""
    if world > nz:
        raise ValueError("more ranks than planes")
    return nz * rank // world, nz * (rank + 1) // world


def allreduce_sum(t, group=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class ShardedAdvance:
    """One rank's share of a pure-ODE config (no communication while stepping)."""

    def __init__(self, source, n_total, rank=0, world=1, device=None):
        from .batch import init_from_source
        self.source = source
        self.n_total = n_total
        self.lo, self.hi = shard_range(n_total, rank, world)
        self.fields = init_from_source(source, self.hi - self.lo, point_offset=self.lo,
                                       device=device)
        self.step = 0

    def run(self, n_steps, snapshot_every=0, counters=None, reduce=True, scratch=None):
        from .batch import advance
        r = advance(self.fields, n_steps, self.source, step0=self.step,
                    snapshot_every=snapshot_every, counters=counters,
                    point_offset=self.lo, scratch=scratch)
        self.step += n_steps
        sums = r.sums
        if reduce:
            allreduce_sum(sums)
        return sums

    def histogram(self, nbins=256, reduce=True):
        from .batch import histogram
        h = histogram(self.fields, nbins)
        if reduce:
            allreduce_sum(h)
        return h


class SlabCoupledDriver:
    """Config-3 z-slab driver.

    Arrays (any backend) hold the rank's planes plus halos: stored planes
    [zb, ze) = [max(z0-1, 0), min(z1+1, nz)).  `stencil(src, dst, args)` runs
    K4 on the stored arrays in slab form; `step(lo, hi, dt)` runs the
    kinetics step on the owned cells, stored flat indices [lo, hi) of the
    temperature buffers; `send/recv` move one plane.
    """

    def __init__(self, nz, ny, nx, rank, world, t_old, t_new, stencil, step, exchange,
                 overlap=True):
        self.nz, self.ny, self.nx = nz, ny, nx
        self.rank, self.world = rank, world
        self.z0, self.z1 = slab_range(nz, rank, world)
        self.zb = max(self.z0 - 1, 0)
        self.ze = min(self.z1 + 1, nz)
        self.t_old, self.t_new = t_old, t_new  # (ze - zb, ny, nx)
        self.stencil, self.step_fn, self.exchange = stencil, step, exchange
        self.overlap = overlap
        self._halos_current = False

    @property
    def slab(self):
        return (self.zb, self.ze - self.zb, self.z0, self.z1)

    def owned_flat_range(self):
        plane = self.ny * self.nx
        return (self.z0 - self.zb) * plane, (self.z1 - self.zb) * plane

    def halo_exchange(self):
        """Send my edge planes of T_n, receive the neighbours' into the halos."""
        lo, hi = self.z0 - self.zb, self.z1 - self.zb
        ops = []
        if self.rank > 0:
            ops.append(("send", self.t_old[lo], self.rank - 1))
            ops.append(("recv", self.t_old[lo - 1], self.rank - 1))
        if self.rank < self.world - 1:
            ops.append(("send", self.t_old[hi - 1], self.rank + 1))
            ops.append(("recv", self.t_old[hi], self.rank + 1))
        self.exchange(ops)

    def _edge_ops(self):
        """T_{n+1} of my edge planes straight into the neighbours' T_old halo
        planes (their next step's T_n), their edges into mine."""
        lo, hi = self.z0 - self.zb, self.z1 - self.zb
        ops = []
        if self.rank > 0:
            ops.append(("send", self.t_new[lo], self.rank - 1))
            ops.append(("recv", self.t_old[lo - 1], self.rank - 1))
        if self.rank < self.world - 1:
            ops.append(("send", self.t_new[hi - 1], self.rank + 1))
            ops.append(("recv", self.t_old[hi], self.rank + 1))
        return ops

    def run_step(self, dt, args_for):
        """One coupled step: K4 on own planes, kinetics on own cells.

        overlap=False: blocking halo swap of T_n, then the whole slab.
        overlap=True (default): the two edge planes first, then their new
        values go out to the neighbours' halos asynchronously while the
        interior planes and the kinetics run; the transfer only has to land
        before the next step's edge planes.  Ordering makes it race-free: a
        halo is overwritten only after this rank's edge planes consumed it,
        the sends read T_{n+1} (the kinetics roll touches T_old of owned
        cells only), and the interior planes never read a halo.
        """
        lo, hi = self.owned_flat_range()
        if not self.overlap:
            self.halo_exchange()
            self.stencil(self.t_old, self.t_new, args_for(self.slab))
            self.step_fn(lo, hi, dt)
            return
        if not self._halos_current:
            self.halo_exchange()  # first step: halos of the initial T_old
            self._halos_current = True
        zb, nzs = self.zb, self.ze - self.zb
        for z in sorted({self.z0, self.z1 - 1}):
            self.stencil(self.t_old, self.t_new, args_for((zb, nzs, z, z + 1)))
        pending = self.exchange(self._edge_ops(), wait=False)
        if self.z1 - self.z0 > 2:
            self.stencil(self.t_old, self.t_new, args_for((zb, nzs, self.z0 + 1, self.z1 - 1)))
        self.step_fn(lo, hi, dt)
        pending.wait()


class _Pending:
    def __init__(self, reqs):
        self.reqs = reqs

    def wait(self):
        # NCCL: the current stream waits for the transfer (the host does not);
        # gloo: the host waits
        for r in self.reqs:
            r.wait()
        self.reqs = []


def torch_exchange(ops, wait=True):
    """Point-to-point plane exchange with torch.distributed (NCCL or gloo).
    wait=False returns a handle whose wait() completes the exchange; NCCL
    orders the sends after the work already queued on the current stream,
    so later kernels overlap the transfer."""
    import torch.distributed as dist
    p2p = [dist.P2POp(dist.isend if kind == "send" else dist.irecv, tensor, peer)
           for kind, tensor, peer in ops]
    pending = _Pending(dist.batch_isend_irecv(p2p) if p2p else [])
    if wait:
        pending.wait()
    return pending


def gather_planes(local, z0, z1, zb, nz, world, rank):
    """Assemble the owned planes of every rank on all ranks (test helper)."""
    import torch
    import torch.distributed as dist
    own = local[z0 - zb:z1 - zb].contiguous()
    sizes = [slab_range(nz, r, world) for r in range(world)]
    bufs = [torch.empty((b - a,) + tuple(own.shape[1:]), dtype=own.dtype, device=own.device)
            for a, b in sizes]
    if world == 1:
        return own
    # all_gather needs equal sizes: pad to the largest slab
    mx = max(b - a for a, b in sizes)
    pad = torch.zeros((mx,) + tuple(own.shape[1:]), dtype=own.dtype, device=own.device)
    pad[:own.shape[0]] = own
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad)
    for i, (a, b) in enumerate(sizes):
        bufs[i] = outs[i][:b - a]
    return torch.cat(bufs, 0)


class SlabCoupledGPU:
    """Config 3 on this rank's GPU: the z-slab (+ 1-plane halos) of the grid
    and the kinetics state of the owned cells.

    Grids with nx % 32 == 0 run the split coupled step (ti64_coupled_step in
    slab form: K4 + hot-row bitmap, row scan, kinetics of listed rows) on
    ping-pong temperature buffers, with the same edge-planes-first halo
    schedule as SlabCoupledDriver: each step computes the two edge planes,
    posts their T_{n+1} to the neighbours' halo planes of the next buffer
    (NCCL point-to-point, ordered after the edge kernels on the stream),
    computes the interior planes while the transfer runs, and waits only
    before the buffers swap.  At world size 1 a step is one call.  Other
    grids take the reference-shaped path (K4 then step_all per step)."""

    def __init__(self, nz, ny, nx, h, rank=0, world=1, device=None, t0=353.0,
                 state0=(0.9, 0.0, 0.1)):
        import torch
        from . import _lib
        from .batch import GlobalFields, _default_device
        dev = device or _default_device()
        self.nz, self.ny, self.nx, self.h = nz, ny, nx, h
        self.rank, self.world = rank, world
        z0, z1 = slab_range(nz, rank, world)
        zb, ze = max(z0 - 1, 0), min(z1 + 1, nz)
        self.z0, self.z1, self.zb, self.ze = z0, z1, zb, ze
        self.split = nx % 32 == 0
        self.t_old = torch.full((ze - zb, ny, nx), float(t0), dtype=torch.float64, device=dev)
        self.t_new = self.t_old.clone()
        plane = ny * nx
        lo, hi = (z0 - zb) * plane, (z1 - zb) * plane
        n = hi - lo
        full = lambda v: torch.full((n,), float(v), dtype=torch.float64, device=dev)
        self.fields = GlobalFields(full(state0[0]), full(state0[1]), full(state0[2]),
                                   self.t_old.view(-1)[lo:hi], self.t_new.view(-1)[lo:hi],
                                   device=dev)
        self.step = 0
        self.device = dev
        if self.split:
            self._idle_bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
            words = _lib.check(_lib.require().ti64_coupled_scratch_words(n),
                               "ti64_coupled_scratch_words")
            self._scratch = torch.zeros(words, dtype=torch.int32, device=dev)
            self._bits_valid = False
            self._cur, self._nxt = self.t_old, self.t_new
        else:
            self.driver = SlabCoupledDriver(nz, ny, nx, rank, world, self.t_old, self.t_new,
                                            self._stencil, self._step, torch_exchange)

    # --- reference-shaped path (any nx) ---------------------------------
    def _stencil(self, src, dst, args):
        import ctypes as C
        from . import _abi, _lib
        from .thermal import DEFAULT_THERMAL
        tp = _abi.thermal_from(DEFAULT_THERMAL.kernel_tuple())
        rc = _lib.require().ti64_stencil_step(_lib.ptr(src), _lib.ptr(dst), None, None,
                                              C.byref(tp), C.byref(args), _lib.stream_handle())
        _lib.check(rc, "ti64_stencil_step")

    def _step(self, lo, hi, dt):
        from .batch import step_all
        step_all(self.fields, dt, n_lanes=8)

    # --- split coupled step in slab form ----------------------------------
    def _coupled(self, cur, nxt, z_begin, z_end, dt, beam, source, bottom, consts):
        import ctypes as C
        from . import _abi, _lib
        tp, kpc, cfgc, fs, lanes = consts
        a = _abi.stencil_args(self.nx, self.ny, self.nz, self.nz, dt, self.h, beam=beam,
                              source=source, losses=False, bottom=bottom, all_built=True,
                              slab=(self.zb, self.ze - self.zb, z_begin, z_end))
        rc = _lib.require().ti64_coupled_step(
            _lib.ptr(cur), _lib.ptr(nxt), C.byref(fs), self.z0, _lib.ptr(self._idle_bits),
            _lib.ptr(self._scratch), C.byref(tp), C.byref(a), C.byref(kpc), C.byref(cfgc),
            int(lanes), 0 if self._bits_valid else 1, _lib.stream_handle())
        _lib.check(rc, "ti64_coupled_step")

    def _halo_ops(self, buf):
        """Edge planes of `buf` to the neighbours' halo planes of their `buf`."""
        lo, hi = self.z0 - self.zb, self.z1 - self.zb
        ops = []
        if self.rank > 0:
            ops.append(("send", buf[lo], self.rank - 1))
            ops.append(("recv", buf[lo - 1], self.rank - 1))
        if self.rank < self.world - 1:
            ops.append(("send", buf[hi - 1], self.rank + 1))
            ops.append(("recv", buf[hi], self.rank + 1))
        return ops

    def run(self, n_steps, dt, beams, source, bottom=353.0, kinetics_params=None,
            integrator_config=None, n_lanes=8):
        from . import _abi
        if not self.split:
            def args_for(slab):
                return _abi.stencil_args(self.nx, self.ny, self.nz, self.nz, dt, self.h,
                                         beam=beams[self._k], source=source, losses=False,
                                         bottom=bottom, all_built=True, slab=slab)
            for k in range(n_steps):
                self._k = k
                self.driver.run_step(dt, args_for)
                self.step += 1
            return self
        self.begin(dt, source, bottom, kinetics_params, integrator_config, n_lanes)
        if self.world > 1 and self.step == 0:
            torch_exchange(self._halo_ops(self._cur))  # halos of the initial T
        for k in range(n_steps):
            if self.world == 1:
                self.phase_all(beams[k])
            else:
                self.phase_edges(beams[k])
                pending = torch_exchange(self._halo_ops(self._nxt), wait=False)
                self.phase_interior(beams[k])
                pending.wait()
            self.finish_step()
        return self.end(n_steps)

    # phases of one split step (exposed so a test can interleave several
    # slabs on one device, exchanging halos with plain copies)
    def begin(self, dt, source, bottom=353.0, kinetics_params=None, integrator_config=None,
              n_lanes=8):
        from . import _abi
        from .integrator import IntegratorConfig
        from .kinetics import DEFAULT_PARAMS
        from .thermal import DEFAULT_THERMAL
        kp = kinetics_params or DEFAULT_PARAMS
        cfg = integrator_config or IntegratorConfig(scheme="explicit")
        self._run = (dt, source, bottom,
                     (_abi.thermal_from(DEFAULT_THERMAL.kernel_tuple()),
                      _abi.kparams_from(kp.kernel_tuple()), _abi.icfg_from(cfg.kernel_tuple()),
                      self.fields.cstruct(), n_lanes))

    def _do(self, z_begin, z_end, beam):
        dt, source, bottom, consts = self._run
        self._coupled(self._cur, self._nxt, z_begin, z_end, dt, beam, source, bottom, consts)

    def phase_all(self, beam):
        self._do(self.z0, self.z1, beam)

    def phase_edges(self, beam):
        for z in sorted({self.z0, self.z1 - 1}):
            self._do(z, z + 1, beam)

    def phase_interior(self, beam):
        if self.z1 - self.z0 > 2:
            self._do(self.z0 + 1, self.z1 - 1, beam)

    def finish_step(self):
        self._bits_valid = True
        self._cur, self._nxt = self._nxt, self._cur
        self.step += 1

    def end(self, n_steps):
        # the reference ends a step with temperature_old == temperature_new
        other = self.t_new if self._cur is self.t_old else self.t_old
        other.copy_(self._cur)
        self.fields.traffic_bytes += 72 * self.fields.n_points * n_steps
        self.fields.steps_taken += n_steps
        return self

    def temperature(self):
        """The owned planes of the current T (a view)."""
        return self._cur[self.z0 - self.zb:self.z1 - self.zb]
