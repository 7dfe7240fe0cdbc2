"""Device-resident SoA state and the drop-in ``step_all`` (B200 path).

Mirrors ti64micro/batch.py's public surface: ``GlobalFields``
(batch.py:99-146), ``step_all`` (batch.py:762-813), ``BatchConvergenceError``
(batch.py:74-79), ``SUPPORTED_LANES``, ``BYTES_PER_POINT``.  The five
global vectors and the seed arrays live in HBM as torch tensors (torch is
only the allocator / stream provider); every update runs in
libti64b200.so through the C ABI of include/ti64_b200.h.

Deviations from the reference API, all deliberate:
  * field attributes are CUDA tensors; ``states()``, ``to_host()`` and
    ``host(name)`` return numpy copies;
  * ``threads`` is accepted and ignored (the device decides parallelism);
    results are thread-count invariant exactly as in the reference;
  * on an implicit-scheme failure the points of later batches are left
    untouched, as in the reference's single sweep (threads=1).
Additions: ``advance`` (fused multi-step update with on-device temperature
generators), ``phase_sums``, ``histogram``, ``run_history``.
"""

import ctypes as C
import functools
from dataclasses import dataclass, field

import numpy as np

from . import _abi, _lib
from .errors import BatchConvergenceError
from .integrator import IntegratorConfig, num_substeps
from .kinetics import DEFAULT_PARAMS

__all__ = ["SUPPORTED_LANES", "BYTES_PER_POINT", "DOF_PER_POINT", "GlobalFields",
           "BatchConvergenceError", "step_all", "run_range", "advance",
           "AdvanceResult", "EventCounters", "phase_sums", "histogram",
           "fast_exp", "fast_ln", "fast_pow", "init_from_source", "blend",
           "branch_dispatch"]

SUPPORTED_LANES = (1, 2, 4, 8)
BYTES_PER_POINT = 72  # 5 loads + 4 stores of 8 B (batch.py:46)
DOF_PER_POINT = 3

_F64 = ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old", "temperature_new",
        "seed_tracked")
_U8 = ("seed_active", "seed_direction")
NAMES = _F64[:5] + ("seed_tracked", "seed_active", "seed_direction")


def _torch():
    import torch
    return torch


def _default_device():
    torch = _torch()
    _lib.require()
    return torch.device("cuda", torch.cuda.current_device())


def _to_device(a, dtype, n, name, device):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        t = a.detach()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.dtype(dtype))))
    if device.type == "cpu":  # host-resident fields: pinned, mapped into the GPU (UVA)
        t = t.to(device="cpu", dtype=getattr(torch, dtype)).contiguous()
        if not t.is_pinned():
            t = t.pin_memory()
    else:
        t = t.to(device=device, dtype=getattr(torch, dtype)).contiguous()
    if tuple(t.shape) != (n,):
        raise ValueError(f"field {name} must have shape ({n},)")
    return t


@dataclass
class GlobalFields:
    """The five global state vectors plus per-point seeding bookkeeping,
    resident on the GPU (batch.py:99-146).

    device="host" keeps them in pinned host memory instead, mapped into the
    GPU's address space.  step_all then reads its inputs from and writes its
    results to host memory itself (zero-copy, coalesced); the fused advance
    stages chunks of points through device buffers with the copies of the
    neighbouring chunks overlapping each chunk's update (ti64_advance_host) —
    the end-to-end path for data that lives on the host.
    Host reads (states/host/to_host) synchronise the device first."""

    x_alpha_s: object
    x_alpha_m: object
    x_beta: object
    temperature_old: object
    temperature_new: object
    seed_tracked: object = None
    seed_active: object = None
    seed_direction: object = None
    traffic_bytes: int = 0
    steps_taken: int = 0
    device: object = field(default=None, repr=False)

    def __post_init__(self):
        n = int(np.shape(self.x_alpha_s)[0]) if np.ndim(self.x_alpha_s) == 1 else -1
        for name in _F64[:5]:
            if tuple(np.shape(getattr(self, name))) != (n,) or n < 0:
                raise ValueError(f"field {name} must have shape ({max(n, 0)},)")
        torch = _torch()
        if self.device == "host" or (isinstance(self.device, torch.device) and
                                     self.device.type == "cpu"):
            _lib.require()
            self.device = torch.device("cpu")
        dev = self.device if self.device is not None else _default_device()
        self.device = dev
        for name in _F64[:5]:
            setattr(self, name, _to_device(getattr(self, name), "float64", n, name, dev))
        torch = _torch()
        if self.seed_tracked is None:
            self.seed_tracked = torch.zeros(n, dtype=torch.float64, device=dev)
        self.seed_tracked = _to_device(self.seed_tracked, "float64", n, "seed_tracked", dev)
        for name in _U8:
            v = getattr(self, name)
            if v is None:
                v = torch.zeros(n, dtype=torch.uint8, device=dev)
            setattr(self, name, _to_device(v, "uint8", n, name, dev))  # (pins host arrays)

    @property
    def n_points(self):
        return int(self.x_alpha_s.shape[0])

    @property
    def host_resident(self):
        return self.device.type == "cpu"

    @property
    def compute_device(self):
        """The CUDA device the kernels run on (scratch, sums, iteration counts)."""
        return _default_device() if self.host_resident else self.device

    def _sync_host(self):
        if self.host_resident:
            _torch().cuda.synchronize()

    @classmethod
    def allocate(cls, n, temperature=293.0, device=None):
        t = np.full(n, float(temperature))
        return cls(np.zeros(n), np.zeros(n), np.zeros(n), t, t.copy(), device=device)

    def states(self, out=None):
        """(n, 3) numpy array of phase fractions (copied from the device).

        `out`: optional (n, 3) float64 host tensor (pin it for full D2H
        bandwidth) that receives the copy; its numpy view is returned."""
        torch = _torch()
        self._sync_host()
        st = torch.stack([self.x_alpha_s, self.x_alpha_m, self.x_beta], 1)
        if out is None:
            return st.cpu().numpy()
        out.copy_(st)
        return out.numpy()

    def host(self, name):
        self._sync_host()
        return getattr(self, name).cpu().numpy()

    def to_host(self):
        return {k: self.host(k) for k in NAMES}

    def copy(self):
        return GlobalFields(*[getattr(self, k).clone() for k in NAMES],
                            traffic_bytes=self.traffic_bytes, steps_taken=self.steps_taken,
                            device=self.device)

    def cstruct(self):
        return _abi.Fields(*[getattr(self, k).data_ptr() for k in NAMES])


def blend(mask, a, b):
    """Lane-wise select (batch.py:196-198)."""
    return np.where(mask, a, b)


def branch_dispatch(mask):
    """'all' / 'none' / 'some' scenario of a condition mask (batch.py:201-208);
    on the device the same decision is a warp vote over the lane group."""
    mask = np.asarray(mask, dtype=bool)
    if mask.all():
        return "all"
    if not mask.any():
        return "none"
    return "some"


def _keep_for_stream(stream, *tensors):
    """Temporaries allocated on the current stream but used by kernels queued
    on a caller-supplied `stream`: tell torch's caching allocator, so their
    memory is not handed out again before that stream's queued work is done
    (record_stream)."""
    if stream is None:
        return
    torch = _torch()
    if stream == torch.cuda.current_stream():
        return
    for t in tensors:
        if t is not None and t.is_cuda:
            t.record_stream(stream)


def _kp(params):
    return _abi.kparams_from(params.kernel_tuple())


def _cfg(config):
    return _abi.icfg_from(config.kernel_tuple())


@functools.lru_cache(maxsize=64)
def _kp_struct(kp_tuple):
    return _abi.kparams_from(kp_tuple)


@functools.lru_cache(maxsize=64)
def _cfg_struct(cfg_tuple):
    return _abi.icfg_from(cfg_tuple)


def run_range(fields, start, stop, lanes, nsub, dt_sub, kp_tuple, cfg_tuple,
              record_iters=False, iters_out=None, stream=None):
    """Kernel entry (batch.py:716-727): one macro step of points [start, stop)."""
    lib = _lib.require()
    fs = fields.cstruct()
    kp = _kp_struct(kp_tuple)
    cfg = _cfg_struct(cfg_tuple)
    rc = lib.ti64_run_range(C.byref(fs), int(start), int(stop), int(lanes), int(nsub),
                            float(dt_sub), C.byref(kp), C.byref(cfg), int(bool(record_iters)),
                            _lib.ptr(iters_out), _lib.stream_handle(stream))
    _lib.check(rc, "ti64_run_range")
    return rc


def step_all(fields, dt, params=DEFAULT_PARAMS, config=IntegratorConfig(), n_lanes=8,
             threads=1, record_iters=False, stream=None):
    """Advance every point by the macro step dt (batch.py:762-813).

    Bit-identical to the reference's step_all for the same n_lanes, for both
    schemes (all eight arrays, including the lane-batch seed write-back and,
    for Crank-Nicolson, the lane coupling of the batch fixed-point loop and
    its halving retries).  temperature_old takes temperature_new's value in
    the same pass.  The explicit scheme is stream-ordered (returns once
    queued); the implicit scheme synchronises to learn the failing batch.

    Returns the per-point fixed-point iteration counts (int64 CUDA tensor,
    zero for the explicit scheme) when record_iters is set, else None.
    Raises BatchConvergenceError naming the first failing batch's points.
    """
    if n_lanes not in SUPPORTED_LANES:
        raise ValueError(f"n_lanes must be one of {SUPPORTED_LANES}")
    if dt <= 0:
        raise ValueError("dt must be positive")
    n = fields.n_points
    nsub = num_substeps(float(dt), config.dt_sub_max)
    iters = None
    if record_iters:
        iters = _torch().zeros(n, dtype=_torch().int64, device=fields.compute_device)
    rc = run_range(fields, 0, n, n_lanes, nsub, float(dt) / nsub, params.kernel_tuple(),
                   config.kernel_tuple(), record_iters, iters, stream)
    _keep_for_stream(stream, iters)
    fields.traffic_bytes += BYTES_PER_POINT * n
    fields.steps_taken += 1
    if rc > 0:
        b = rc - 1
        raise BatchConvergenceError(list(range(b, min(b + n_lanes, n))))
    return iters


# --------------------------------------------------------------------------
# fused advance with on-device temperature generators
# --------------------------------------------------------------------------

class EventCounters:
    """Per-point martensite-event / phase-switch counters (u32) and the
    8 totals of include/ti64_b200.h (ti64_counters.totals_d)."""

    def __init__(self, n, device):
        torch = _torch()
        self.martensite = torch.zeros(n, dtype=torch.int32, device=device)
        self.switches = torch.zeros(n, dtype=torch.int32, device=device)
        self.totals = torch.zeros(8, dtype=torch.int64, device=device)

    def cstruct(self):
        return _abi.Counters(self.martensite.data_ptr(), self.switches.data_ptr(),
                             self.totals.data_ptr())

    def totals_dict(self):
        v = self.totals.cpu().numpy().astype(np.uint64)
        return dict(zip(_abi.TOTALS_FIELDS, (int(x) for x in v)))


@dataclass
class AdvanceResult:
    sums: object          # (n_snapshots, 3) float64 device tensor
    counters: object      # EventCounters or None
    steps: int
    launches: int


_beam_cache = {}  # insertion-ordered: LRU eviction of the oldest entry
_BEAM_CACHE_MAX = 8


def beam_table(source, rows, device):
    """Device beam table of `source` (None for pulse sources), cached.  An
    evicted table is only released through torch's caching allocator, which
    is stream-ordered; callers launching on another stream record it there
    (_keep_for_stream), so a queued kernel never reads reused memory."""
    key = (source, rows, str(device))
    t = _beam_cache.pop(key, None) if key in _beam_cache else None
    if t is None:
        packed = getattr(source, "packed_beam", None)
        tab = packed(rows) if packed is not None else source.beam_table(rows)
        t = None if tab is None else _torch().from_numpy(tab).to(device)
        while len(_beam_cache) >= _BEAM_CACHE_MAX:
            _beam_cache.pop(next(iter(_beam_cache)))
    _beam_cache[key] = t
    return t


def tempgen_for(source, point_offset, rows, device):
    """(TempGen struct, keep-alive beam tensor) for `source`."""
    beam = beam_table(source, rows, device)
    g = source.tempgen(point_offset=point_offset,
                       beam_ptr=None if beam is None else beam.data_ptr(),
                       beam_steps=0 if beam is None else rows)
    return g, beam


def _scratch(n, device):
    lib = _lib.require()
    nbytes = int(lib.ti64_advance_scratch_bytes(n))
    return _torch().empty((nbytes + 7) // 8, dtype=_torch().float64, device=device)


def advance(fields, n_steps, source, step0=0, params=DEFAULT_PARAMS,
            config=IntegratorConfig(), n_lanes=8, snapshot_every=0, counters=None,
            point_offset=0, stream=None, scratch=None, host_chunk_points=0):
    """Fused advance (K2): equivalent, bit for bit, to

        for s in range(step0, step0 + n_steps):
            fields.temperature_new[:] = T(s + 1)      # source, on device
            step_all(fields, source.dt, params, config, n_lanes)

    with per-point state held in registers across steps.  Returns an
    AdvanceResult whose ``sums`` are the phase-fraction sums after every
    `snapshot_every` steps (and at the end).

    Host-resident fields (``GlobalFields(..., device="host")``) go through
    ti64_advance_host: chunks of `host_chunk_points` points (0: the library's
    default) are staged through device buffers with the host<->device copies
    overlapping the update; ``host_chunk_points=-1`` keeps the zero-copy
    access of the mapped host arrays instead (the scratch argument only
    applies there and to device-resident fields).
    """
    if n_lanes not in SUPPORTED_LANES:
        raise ValueError(f"n_lanes must be one of {SUPPORTED_LANES}")
    if n_steps < 0 or step0 < 0:
        raise ValueError("n_steps and step0 must be non-negative")
    if config.scheme != "explicit":
        return _advance_implicit(fields, n_steps, source, step0, params, config, n_lanes,
                                 snapshot_every, counters, point_offset, stream)
    lib = _lib.require()
    torch = _torch()
    n = fields.n_points
    dev = fields.compute_device
    nsub = num_substeps(float(source.dt), config.dt_sub_max)
    g, beam = tempgen_for(source, point_offset, step0 + n_steps + 1, dev)
    chunk = snapshot_every if snapshot_every > 0 else max(n_steps, 1)
    n_snap = (n_steps + chunk - 1) // chunk if n_steps > 0 else 0
    sums = torch.zeros((max(n_snap, 1), 3), dtype=torch.float64, device=dev)
    cs = counters.cstruct() if counters is not None else None
    fs = fields.cstruct()
    kp, cfg = _kp(params), _cfg(config)
    if fields.host_resident and host_chunk_points >= 0:
        # host arrays: chunks staged through device buffers, the copies of the
        # neighbouring chunks overlapping each chunk's update (ti64_advance_host)
        nbytes = int(_lib.check(lib.ti64_advance_host_scratch_bytes(
            n, int(host_chunk_points), int(n_steps), int(snapshot_every)),
            "ti64_advance_host_scratch_bytes"))
        scratch = torch.empty((nbytes + 7) // 8, dtype=torch.float64, device=dev)
        rc = lib.ti64_advance_host(C.byref(fs), n, C.byref(g), int(step0), int(n_steps),
                                   int(nsub), int(n_lanes), int(snapshot_every), C.byref(kp),
                                   C.byref(cfg), None if cs is None else C.byref(cs),
                                   _lib.ptr(sums), _lib.ptr(scratch), nbytes,
                                   int(host_chunk_points), _lib.stream_handle(stream))
        launches = _lib.check(rc, "ti64_advance_host")
    else:
        scratch = _scratch(n, dev) if scratch is None else scratch
        rc = lib.ti64_advance(C.byref(fs), n, C.byref(g), int(step0), int(n_steps), int(nsub),
                              int(n_lanes), int(snapshot_every), C.byref(kp), C.byref(cfg),
                              None if cs is None else C.byref(cs), _lib.ptr(sums),
                              _lib.ptr(scratch), _lib.stream_handle(stream))
        launches = _lib.check(rc, "ti64_advance")  # >= 0: kernels launched
    _keep_for_stream(stream, beam, sums, scratch)
    del beam
    fields.traffic_bytes += BYTES_PER_POINT * n * n_steps
    fields.steps_taken += n_steps
    return AdvanceResult(sums=sums[:n_snap], counters=counters, steps=n_steps,
                         launches=int(launches))


def init_from_source(source, n, point_offset=0, device=None):
    """GlobalFields with the config's seeded initial state and T(0) (K3)."""
    lib = _lib.require()
    torch = _torch()
    dev = device or _default_device()
    f = GlobalFields.allocate(n, device=dev)
    g, beam = tempgen_for(source, point_offset, 1, dev)
    st = _lib.stream_handle()
    _lib.check(lib.ti64_gen_initial_state(C.byref(g), n, C.byref(f.cstruct()), st),
               "ti64_gen_initial_state")
    _lib.check(lib.ti64_gen_temperature(C.byref(g), n, 0, _lib.ptr(f.temperature_old), st),
               "ti64_gen_temperature")
    f.temperature_new.copy_(f.temperature_old)
    del beam, torch
    return f


def _advance_implicit(fields, n_steps, source, step0, params, config, n_lanes,
                      snapshot_every, counters, point_offset, stream):
    """advance() for the Crank-Nicolson scheme: the literal loop of its
    docstring (K3 generator into temperature_new, then the implicit K1), two
    launches per step plus the snapshot sums.  The implicit step cannot be
    fused across steps the way K2 fuses the explicit one: a failing batch
    must stop the sweep (BatchConvergenceError) before the next step runs."""
    if counters is not None:
        raise ValueError("event counters are only maintained by the fused explicit advance")
    lib = _lib.require()
    torch = _torch()
    n = fields.n_points
    dev = fields.compute_device
    g, beam = tempgen_for(source, point_offset, step0 + n_steps + 1, dev)
    chunk = snapshot_every if snapshot_every > 0 else max(n_steps, 1)
    n_snap = (n_steps + chunk - 1) // chunk if n_steps > 0 else 0
    sums = torch.zeros((max(n_snap, 1), 3), dtype=torch.float64, device=dev)
    scratch = _scratch(n, dev)
    launches = 0
    for k in range(n_steps):
        _lib.check(lib.ti64_gen_temperature(C.byref(g), n, int(step0 + k + 1),
                                            _lib.ptr(fields.temperature_new),
                                            _lib.stream_handle(stream)), "ti64_gen_temperature")
        step_all(fields, source.dt, params, config, n_lanes, stream=stream)
        launches += 2
        if (k + 1) % chunk == 0 or k == n_steps - 1:
            snap = k // chunk
            _lib.check(lib.ti64_phase_sums(_lib.ptr(fields.x_alpha_s),
                                           _lib.ptr(fields.x_alpha_m), _lib.ptr(fields.x_beta),
                                           n, _lib.ptr(sums[snap]), _lib.ptr(scratch),
                                           _lib.stream_handle(stream)), "ti64_phase_sums")
            launches += 2
    _keep_for_stream(stream, beam, sums, scratch)
    del beam
    return AdvanceResult(sums=sums, counters=None, steps=n_steps, launches=launches)


def gen_temperature(source, n, step, point_offset=0, device=None):
    lib = _lib.require()
    dev = device or _default_device()
    out = _torch().empty(n, dtype=_torch().float64, device=dev)
    g, beam = tempgen_for(source, point_offset, step + 1, dev)
    _lib.check(lib.ti64_gen_temperature(C.byref(g), n, int(step), _lib.ptr(out),
                                        _lib.stream_handle()), "ti64_gen_temperature")
    del beam
    return out


def phase_sums(fields, scratch=None):
    """Deterministic fp64 sums (x_alpha_s, x_alpha_m, x_beta) -> tensor(3)."""
    lib = _lib.require()
    torch = _torch()
    out = torch.zeros(3, dtype=torch.float64, device=fields.compute_device)
    scratch = _scratch(fields.n_points, fields.compute_device) if scratch is None else scratch
    _lib.check(lib.ti64_phase_sums(_lib.ptr(fields.x_alpha_s), _lib.ptr(fields.x_alpha_m),
                                   _lib.ptr(fields.x_beta), fields.n_points, _lib.ptr(out),
                                   _lib.ptr(scratch), _lib.stream_handle()), "ti64_phase_sums")
    return out


def histogram(fields, nbins=256, out=None):
    """(3, nbins) int64 counts of floor(x*nbins) (clamped) of xs, xm, xb."""
    lib = _lib.require()
    torch = _torch()
    if out is None:
        out = torch.zeros((3, nbins), dtype=torch.int64, device=fields.compute_device)
    _lib.check(lib.ti64_histogram(_lib.ptr(fields.x_alpha_s), _lib.ptr(fields.x_alpha_m),
                                  _lib.ptr(fields.x_beta), fields.n_points, int(nbins),
                                  _lib.ptr(out), _lib.stream_handle()), "ti64_histogram")
    return out


# --------------------------------------------------------------------------
# element-wise fast math (fastmath.py:246-258 array API, on device)
# --------------------------------------------------------------------------

def _elementwise(fname, *arrays):
    lib = _lib.require()
    torch = _torch()
    is_torch = isinstance(arrays[0], torch.Tensor)
    np_arrs = [a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a for a in arrays]
    b = np.broadcast_arrays(*[np.asarray(a, dtype=np.float64) for a in np_arrs])
    shape = b[0].shape
    dev = _default_device()
    ts = [torch.from_numpy(np.array(x, dtype=np.float64).ravel()).to(dev) for x in b]
    out = torch.empty_like(ts[0])
    fn = getattr(lib, fname)
    _lib.check(fn(*[_lib.ptr(t) for t in ts], _lib.ptr(out), ts[0].numel(),
                  _lib.stream_handle()), fname)
    out = out.reshape(shape)
    if is_torch:
        return out
    res = out.cpu().numpy()
    return float(res) if all(np.ndim(a) == 0 for a in np_arrs) else res


def fast_exp(x):
    return _elementwise("ti64_fast_exp", x)


def fast_ln(x):
    return _elementwise("ti64_fast_ln", x)


def fast_pow(a, x):
    return _elementwise("ti64_fast_pow", a, x)


# --------------------------------------------------------------------------
# temperature histories (integrator.py:303-361), batched
# --------------------------------------------------------------------------

def corrected_beta_state(t0, params=DEFAULT_PARAMS):
    """apply_corrections(PhaseState(0, 0, solid_fraction(T)), T) for an array
    of T (kinetics.py:232-269 with kinetics.py:158-179 / :144-155), the
    reference's default initial state of integrate_history
    (integrator.py:317-319).  Host numpy with the device fast_exp."""
    t = np.asarray(t0, dtype=np.float64)
    p = params
    g = np.clip((t - p.t_sol) / (p.t_liq - p.t_sol), 0.0, 1.0)
    xsol = 1.0 - g
    xs = np.maximum(np.zeros_like(t), 0.0)
    xm = np.maximum(np.zeros_like(t), 0.0)
    ramp = 0.9 * (p.t_alpha_s_start + p.t_alpha_s_reg - t) / p.t_alpha_s_reg
    ramp = np.maximum(ramp, 0.0)
    xs = np.where(t > p.t_alpha_s_start, np.minimum(xs, ramp), xs)
    e1 = np.asarray(fast_exp(-p.k_alpha_eq * (p.t_alpha_s_start - t)))
    xa_eq = np.where(t < p.t_alpha_s_end, 0.9, np.where(t > p.t_alpha_s_start, 0.0, 1.0 - e1))
    xm = np.where(xs + xm > xa_eq, np.maximum(xa_eq - xs, 0.0), xm)
    e2 = np.asarray(fast_exp(-p.k_alpha_m_eq * (p.t_alpha_m_start - t)))
    base = np.where(t > p.t_alpha_m_start, 0.0, np.minimum(1.0 - e2, 0.9))
    xm_eq = base * (0.9 - xs) / 0.9
    xm = np.where(t < p.t_alpha_m_start, np.maximum(xm, xm_eq), xm)
    xa = xs + xm
    scale = np.where(xa > 0.9, 0.9 / np.where(xa > 0.0, xa, 1.0), 1.0)
    xs = xs * scale
    xm = xm * scale
    xb = np.maximum(xsol - xs - xm, 0.0)
    return xs, xm, xb


def run_history(times, temps2d, xs, xm, xb, params=DEFAULT_PARAMS,
                config=IntegratorConfig()):
    """(n_samples, n_points, 3) numpy trajectory; temps2d is (n_samples, n)."""
    lib = _lib.require()
    torch = _torch()
    dev = _default_device()
    ns, n = temps2d.shape
    f = GlobalFields(np.asarray(xs, np.float64), np.asarray(xm, np.float64),
                     np.asarray(xb, np.float64), temps2d[0], temps2d[0], device=dev)
    temps_d = torch.from_numpy(np.ascontiguousarray(temps2d)).to(dev)
    out = torch.empty((ns, n, 3), dtype=torch.float64, device=dev)
    times = np.ascontiguousarray(times, dtype=np.float64)
    fs = f.cstruct()
    kp, cfg = _kp(params), _cfg(config)
    rc = lib.ti64_run_history(C.byref(fs), n, times.ctypes.data_as(C.c_void_p),
                              _lib.ptr(temps_d), ns, C.byref(kp), C.byref(cfg),
                              _lib.ptr(out), _lib.stream_handle())
    _lib.check(rc, "ti64_run_history")
    return out.cpu().numpy()
