"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the CPU oracle.

Loads oracle/libti64oracle.so (built from oracle/ti64_oracle.c by
oracle/Makefile) and exposes numpy-level calls.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may import this
module; the product package never does.

Every function here mirrors a reference entry point (paths relative to
/root/reference/pkg/src/ti64micro/):
  run_range / step_all   batch.py:716-727 / batch.py:762-813
  fast_exp/ln/pow        fastmath.py:181-212
  history                integrator.py:303-361
  stencil_step           thermal.py:205-287
plus the project's own generator / counter definitions.
"""

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2402_17580_b200 import _abi

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libti64oracle.so"

_lib = None


def build():
    """Compile the oracle with oracle/Makefile (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        L.oracle_fast_exp1.restype = D
        L.oracle_fast_exp1.argtypes = [D]
        L.oracle_fast_ln1.restype = D
        L.oracle_fast_ln1.argtypes = [D]
        L.oracle_fast_pow1.restype = D
        L.oracle_fast_pow1.argtypes = [D, D]
        for name in ("oracle_fast_exp", "oracle_fast_ln"):
            getattr(L, name).argtypes = [P, P, I64]
            getattr(L, name).restype = None
        L.oracle_fast_pow.argtypes = [P, P, P, I64]
        L.oracle_fast_pow.restype = None
        L.oracle_run_range.argtypes = [P, I64, I64, I64, I64, D, P, P]
        L.oracle_run_range.restype = I64
        L.oracle_run_range2.argtypes = [P, I64, I64, I64, I64, D, P, P, I32, P]
        L.oracle_run_range2.restype = I64
        L.oracle_step_all.argtypes = [P, I64, I64, I64, D, P, P, I32]
        L.oracle_step_all.restype = I64
        L.oracle_num_substeps.argtypes = [D, D]
        L.oracle_num_substeps.restype = I64
        L.oracle_gen_temperature.argtypes = [P, I64, I64, P, I32]
        L.oracle_gen_temperature.restype = None
        L.oracle_gen_temperature1.argtypes = [P, I64, I64]
        L.oracle_gen_temperature1.restype = D
        L.oracle_gen_initial_state.argtypes = [P, I64, P]
        L.oracle_gen_initial_state.restype = None
        L.oracle_advance.argtypes = [P, I64, P, I64, I64, I64, I64, I64, P, P,
                                     P, P, P, P, I32]
        L.oracle_advance.restype = I64
        L.oracle_advance_points.argtypes = [P, P, I64, P, I64, I64, I64, P, P, P, P, P, I32]
        L.oracle_advance_points.restype = I64
        L.oracle_gen_temperature_points.argtypes = [P, P, I64, I64, I64, P, I32]
        L.oracle_gen_temperature_points.restype = None
        L.oracle_history.argtypes = [P, P, I64, D, D, D, P, P, P]
        L.oracle_history.restype = I64
        L.oracle_stencil_step.argtypes = [P, P, P, P, P, P]
        L.oracle_stencil_step.restype = None
        L.oracle_u01.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.oracle_u01.restype = D
        L.oracle_max_threads.restype = I32
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def max_threads():
    return int(lib().oracle_max_threads())


def fast_exp(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().oracle_fast_exp(_p(x), _p(out), x.size)
    return out


def fast_ln(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().oracle_fast_ln(_p(x), _p(out), x.size)
    return out


def fast_pow(a, x):
    a, x = np.broadcast_arrays(np.asarray(a, np.float64), np.asarray(x, np.float64))
    a = np.ascontiguousarray(a)
    x = np.ascontiguousarray(x)
    out = np.empty_like(a)
    lib().oracle_fast_pow(_p(a), _p(x), _p(out), a.size)
    return out


class HostFields:
    """numpy SoA state with the reference GlobalFields layout (batch.py:99-126)."""

    NAMES = ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old",
             "temperature_new", "seed_tracked", "seed_active", "seed_direction")

    def __init__(self, xs, xm, xb, t_old, t_new, seed_tracked=None,
                 seed_active=None, seed_direction=None):
        n = len(xs)
        self.x_alpha_s = np.array(xs, dtype=np.float64)
        self.x_alpha_m = np.array(xm, dtype=np.float64)
        self.x_beta = np.array(xb, dtype=np.float64)
        self.temperature_old = np.array(t_old, dtype=np.float64)
        self.temperature_new = np.array(t_new, dtype=np.float64)
        self.seed_tracked = (np.zeros(n) if seed_tracked is None
                             else np.array(seed_tracked, dtype=np.float64))
        self.seed_active = (np.zeros(n, np.uint8) if seed_active is None
                            else np.array(seed_active, dtype=np.uint8))
        self.seed_direction = (np.zeros(n, np.uint8) if seed_direction is None
                               else np.array(seed_direction, dtype=np.uint8))

    @classmethod
    def allocate(cls, n, temperature=293.0):
        t = np.full(n, float(temperature))
        return cls(np.zeros(n), np.zeros(n), np.zeros(n), t, t.copy())

    @property
    def n_points(self):
        return len(self.x_alpha_s)

    def copy(self):
        return HostFields(*[getattr(self, k).copy() for k in self.NAMES])

    def states(self):
        return np.stack([self.x_alpha_s, self.x_alpha_m, self.x_beta], axis=1)

    def cstruct(self):
        return _abi.Fields(*[getattr(self, k).ctypes.data for k in self.NAMES])


def run_range(fields, kp, cfg, lanes=8, nsub=1, dt_sub=2e-5, start=0, stop=None):
    stop = fields.n_points if stop is None else stop
    fs = fields.cstruct()
    k, c = _abi.kparams_from(kp), _abi.icfg_from(cfg)
    return int(lib().oracle_run_range(C.byref(fs), start, stop, lanes, nsub,
                                      float(dt_sub), C.byref(k), C.byref(c)))


def run_range_cn(fields, kp, cfg, lanes=8, nsub=1, dt_sub=0.01, record_iters=True):
    """batch.run_range for either scheme over all points (single sweep, like
    step_all with threads=1); returns (rc, iters)."""
    n = fields.n_points
    iters = np.zeros(n, np.int64)
    fs = fields.cstruct()
    k, c = _abi.kparams_from(kp), _abi.icfg_from(cfg)
    rc = int(lib().oracle_run_range2(C.byref(fs), 0, n, lanes, nsub, float(dt_sub),
                                     C.byref(k), C.byref(c), int(bool(record_iters)),
                                     _p(iters)))
    return rc, iters


def num_substeps(dt, dt_sub_max):
    return int(lib().oracle_num_substeps(float(dt), float(dt_sub_max)))


def step_all(fields, dt, kp, cfg, n_lanes=8, threads=1):
    """batch.step_all semantics on HostFields (explicit scheme)."""
    nsub = num_substeps(dt, cfg.dt_sub_max)
    fs = fields.cstruct()
    k, c = _abi.kparams_from(kp), _abi.icfg_from(cfg)
    rc = int(lib().oracle_step_all(C.byref(fs), fields.n_points, n_lanes, nsub,
                                   float(dt) / nsub, C.byref(k), C.byref(c),
                                   int(threads)))
    return rc


def gen_temperature(gen, n, step, threads=1):
    out = np.empty(n)
    lib().oracle_gen_temperature(C.byref(gen), n, step, _p(out), int(threads))
    return out


def gen_initial_state(gen, n, temperature_old=None):
    f = HostFields.allocate(n)
    lib().oracle_gen_initial_state(C.byref(gen), n, C.byref(f.cstruct()))
    return f


def advance(fields, gen, step0, nsteps, kp, cfg, lanes=8, snapshot_every=0,
            threads=1, nsub=None):
    """Reference loop {temperature_new <- T(s+1); step_all} with counters.

    Returns dict(martensite, switches, totals, sums)."""
    n = fields.n_points
    nsub = num_substeps(gen.dt, cfg.dt_sub_max) if nsub is None else nsub
    mart = np.zeros(n, np.uint32)
    sw = np.zeros(n, np.uint32)
    totals = np.zeros(8, np.uint64)
    n_snap = (nsteps // snapshot_every if snapshot_every > 0 else 0)
    if snapshot_every <= 0 or nsteps % snapshot_every != 0:
        n_snap += 1
    sums = np.zeros((max(n_snap, 1), 3))
    fs = fields.cstruct()
    k, c = _abi.kparams_from(kp), _abi.icfg_from(cfg)
    rc = int(lib().oracle_advance(C.byref(fs), n, C.byref(gen), step0, nsteps, nsub,
                                  lanes, snapshot_every, C.byref(k), C.byref(c),
                                  _p(mart), _p(sw), _p(totals), _p(sums),
                                  int(threads)))
    if rc != 0:
        raise RuntimeError(f"oracle_advance rc={rc}")
    return {"martensite": mart, "switches": sw, "totals": totals, "sums": sums}


def advance_points(fields, points, gen, step0, nsteps, kp, cfg, threads=None, nsub=None):
    """oracle_advance for a subset of points given by GLOBAL index (`points`,
    int64): each point alone (width-1 lane batch), OpenMP over points.
    `fields` (HostFields of len(points)) is advanced in place; returns
    dict(martensite, switches, totals)."""
    pts = np.ascontiguousarray(points, dtype=np.int64)
    m = len(pts)
    assert fields.n_points == m
    nsub = num_substeps(gen.dt, cfg.dt_sub_max) if nsub is None else nsub
    threads = max_threads() if threads is None else threads
    mart = np.zeros(m, np.uint32)
    sw = np.zeros(m, np.uint32)
    totals = np.zeros(8, np.uint64)
    fs = fields.cstruct()
    k, c = _abi.kparams_from(kp), _abi.icfg_from(cfg)
    rc = int(lib().oracle_advance_points(C.byref(fs), _p(pts), m, C.byref(gen), int(step0),
                                         int(nsteps), int(nsub), C.byref(k), C.byref(c),
                                         _p(mart), _p(sw), _p(totals), int(threads)))
    if rc != 0:
        raise RuntimeError(f"oracle_advance_points rc={rc}")
    return {"martensite": mart, "switches": sw, "totals": totals}


def gen_temperature_points(gen, points, step0, nsteps, threads=None):
    """(nsteps, m) temperatures of GLOBAL points at steps step0.. (K3's
    definition)."""
    pts = np.ascontiguousarray(points, dtype=np.int64)
    out = np.empty((int(nsteps), len(pts)))
    threads = max_threads() if threads is None else threads
    lib().oracle_gen_temperature_points(C.byref(gen), _p(pts), len(pts), int(step0),
                                        int(nsteps), _p(out), int(threads))
    return out


def gen_initial_points(gen, points):
    """HostFields with the seeded initial state of the given GLOBAL points and
    T_old = T(0) (as init_from_source does for a contiguous shard)."""
    pts = np.ascontiguousarray(points, dtype=np.int64)
    f = HostFields.allocate(len(pts))
    g0 = _abi.TempGen.from_buffer_copy(gen)
    for j, p in enumerate(pts):  # point_offset = p, one point at a time
        g0.point_offset = int(p)
        one = HostFields.allocate(1)
        lib().oracle_gen_initial_state(C.byref(g0), 1, C.byref(one.cstruct()))
        for k in HostFields.NAMES:
            getattr(f, k)[j] = getattr(one, k)[0]
        f.temperature_old[j] = lib().oracle_gen_temperature1(C.byref(g0), 0, 0)
    f.temperature_new[:] = f.temperature_old
    return f


def history(times, temps, state0, kp, cfg):
    times = np.ascontiguousarray(times, np.float64)
    temps = np.ascontiguousarray(temps, np.float64)
    out = np.empty((len(times), 3))
    k, c = _abi.kparams_from(kp), _abi.icfg_from(cfg)
    lib().oracle_history(_p(times), _p(temps), len(times), float(state0[0]),
                         float(state0[1]), float(state0[2]), C.byref(k), C.byref(c),
                         _p(out))
    return out


def stencil_step(src, dst, rc, state, tp, args):
    """thermal.py:205-287 on host arrays (dst and rc updated in place)."""
    for a in (src, dst, rc):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    assert state.dtype == np.uint8 and state.flags.c_contiguous
    lib().oracle_stencil_step(_p(src), _p(dst), _p(rc), _p(state),
                              C.byref(_abi.thermal_from(tp)), C.byref(args))


def u01(seed, point, k):
    return float(lib().oracle_u01(seed, point, k))


os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
