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
    """Config 3 on this rank's GPU: z-slab (+ halos) of the grid with the
    kinetics state of the owned cells; K4 and K1 from libti64b200.so, halo
    planes over NCCL (torch.distributed point-to-point)."""

    def __init__(self, nz, ny, nx, h, rank=0, world=1, device=None, t0=353.0,
                 state0=(0.9, 0.0, 0.1)):
        import torch
        from .batch import GlobalFields, _default_device
        dev = device or _default_device()
        self.nz, self.ny, self.nx, self.h = nz, ny, nx, h
        z0, z1 = slab_range(nz, rank, world)
        zb, ze = max(z0 - 1, 0), min(z1 + 1, nz)
        self.t_old = torch.full((ze - zb, ny, nx), float(t0), dtype=torch.float64, device=dev)
        self.t_new = self.t_old.clone()
        plane = ny * nx
        lo, hi = (z0 - zb) * plane, (z1 - zb) * plane
        n = hi - lo
        full = lambda v: torch.full((n,), float(v), dtype=torch.float64, device=dev)
        self.fields = GlobalFields(full(state0[0]), full(state0[1]), full(state0[2]),
                                   self.t_old.view(-1)[lo:hi], self.t_new.view(-1)[lo:hi],
                                   device=dev)
        assert self.fields.temperature_old.data_ptr() == self.t_old.view(-1)[lo:].data_ptr()
        self.driver = SlabCoupledDriver(nz, ny, nx, rank, world, self.t_old, self.t_new,
                                        self._stencil, self._step, torch_exchange)
        self.step = 0

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

    def run(self, n_steps, dt, beams, source, bottom=353.0):
        from . import _abi
        k0 = self.step

        def args_for(slab, k=None):
            return _abi.stencil_args(self.nx, self.ny, self.nz, self.nz, dt, self.h,
                                     beam=beams[self._k], source=source, losses=False,
                                     bottom=bottom, all_built=True, slab=slab)
        for k in range(n_steps):
            self._k = k
            self.driver.run_step(dt, args_for)
            self.step += 1
        del k0
        return self
