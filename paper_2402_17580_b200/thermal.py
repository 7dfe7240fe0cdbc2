"""Heat-equation stencil path and the coupled layer build, on the GPU.

Mirrors ti64micro/thermal.py: ``ThermalParams`` / ``kernel_tuple``
(thermal.py:50-104), ``HeatSource`` (:107-121), the point-wise helpers
``conductivity`` / ``update_consolidation`` / ``source_term`` /
``surface_losses`` (:124-165), ``stable_dt`` (:168-170), ``ThermalField``
(:177-202), ``step_thermal`` (:321-354, the K4 kernels of
csrc/ti64_stencil.cu on device-resident grids), and the build driver
``BuildGeometry`` / ``BuildSchedule`` / ``allocate_domain`` /
``activate_layer`` / ``run_build`` (:362-589), whose every thermal and
kinetics step runs on the device (step_thermal + step_all on the active
z-prefix, exactly the reference's ``couple``).  ``CoupledDomain`` is the
all-built config-3 block with the fused stencil+kinetics kernel.
"""

import math
from dataclasses import dataclass, replace
from typing import NamedTuple

__all__ = ["KernelThermalParams", "ThermalParams", "DEFAULT_THERMAL", "HeatSource",
           "stable_dt", "STATE_INACTIVE", "STATE_POWDER", "STATE_BUILT", "SIGMA_S",
           "conductivity", "update_consolidation", "source_term", "surface_losses",
           "ThermalField", "step_thermal", "CoupledDomain", "BuildGeometry",
           "BuildSchedule", "allocate_domain", "activate_layer", "cooldown_steps",
           "run_build"]

STATE_INACTIVE = 0
STATE_POWDER = 1
STATE_BUILT = 2

SIGMA_S = 5.670374419e-8


class KernelThermalParams(NamedTuple):
    """thermal.py:50-66."""

    k_ms: float
    k_p: float
    rho_c: float
    t_sol: float
    t_liq: float
    t_inf: float
    emissivity: float
    sigma_s: float
    t_v: float
    c_p: float
    c_t: float
    c_m: float
    h_v: float
    t_h0: float
    t_max_clamp: float
    c_heat: float


@dataclass(frozen=True)
class ThermalParams:
    """Published Ti-6Al-4V thermal set (thermal.py:69-92)."""

    k_ms: float = 28.6
    k_p: float = 0.286
    rho: float = 4090.0
    c: float = 1130.0
    t_sol: float = 1878.0
    t_liq: float = 1928.0
    t_inf: float = 293.0
    emissivity: float = 0.7
    sigma_s: float = SIGMA_S
    t_v: float = 3130.0
    c_p: float = 54e3
    c_t: float = 5.07e4
    c_m: float = 9.15e-4
    molar_mass: float = 0.0478
    h_v: float = 8.84e6
    t_h0: float = 538.0
    t_max_clamp: float = 3130.0 + 1000.0

    def with_overrides(self, **kwargs):
        return replace(self, **kwargs)

    def kernel_tuple(self):
        return KernelThermalParams(
            k_ms=self.k_ms, k_p=self.k_p, rho_c=self.rho * self.c,
            t_sol=self.t_sol, t_liq=self.t_liq, t_inf=self.t_inf,
            emissivity=self.emissivity, sigma_s=self.sigma_s,
            t_v=self.t_v, c_p=self.c_p, c_t=self.c_t, c_m=self.c_m,
            h_v=self.h_v, t_h0=self.t_h0, t_max_clamp=self.t_max_clamp,
            c_heat=self.c)


DEFAULT_THERMAL = ThermalParams()


@dataclass(frozen=True)
class HeatSource:
    """Cylindrical volumetric beam (thermal.py:107-121)."""

    w_eff: float = 180.0
    radius: float = 0.06e-3
    h_powder: float = 0.05e-3

    def __post_init__(self):
        if self.w_eff <= 0 or self.radius <= 0 or self.h_powder <= 0:
            raise ValueError("heat source parameters must be positive")

    @property
    def peak(self):
        return 2.0 * self.w_eff / (math.pi * self.radius**2 * self.h_powder)


def stable_dt(h, params=DEFAULT_THERMAL):
    """Explicit diffusion bound h^2 rho c / (6 k_max) (thermal.py:168-170)."""
    return h * h * params.rho * params.c / (6.0 * params.k_ms)


def _np(a):
    import numpy as np
    return np.asarray(a, dtype=np.float64)


def _ret(out):
    return float(out) if out.ndim == 0 else out


def conductivity(t, r_c, params=DEFAULT_THERMAL):
    """r_p k_p + r_m k_m + r_s k_s with k_m = k_s (thermal.py:124-133)."""
    import numpy as np
    t, r_c = _np(t), _np(r_c)
    g = np.clip((t - params.t_sol) / (params.t_liq - params.t_sol), 0.0, 1.0)
    return _ret((1.0 - r_c) * params.k_p + g * params.k_ms + (r_c - g) * params.k_ms)


def update_consolidation(r_c, t, powder_origin, params=DEFAULT_THERMAL):
    """Running max of the liquid fraction for powder voxels (thermal.py:136-139)."""
    import numpy as np
    g = np.clip((_np(t) - params.t_sol) / (params.t_liq - params.t_sol), 0.0, 1.0)
    return np.where(powder_origin, np.maximum(r_c, g), r_c)


def source_term(x, y, z_below_surface, beam_x, beam_y, source=HeatSource(), params=None):
    """Volumetric beam input at a point (thermal.py:142-148); the exponential
    is the device fast_exp."""
    import numpy as np
    from .batch import fast_exp
    r2 = (_np(x) - beam_x) ** 2 + (_np(y) - beam_y) ** 2
    q = source.peak * _np(fast_exp(-2.0 * r2 / source.radius**2))
    return _ret(np.where(_np(z_below_surface) < source.h_powder, q, 0.0))


def surface_losses(t, params=DEFAULT_THERMAL):
    """Radiative + evaporative flux of exposed top faces (thermal.py:151-165)."""
    import numpy as np
    from .batch import fast_exp
    t = _np(t)
    q_rad = params.emissivity * params.sigma_s * (t**4 - params.t_inf**4)
    tc = np.minimum(t, params.t_max_clamp)
    q_evap = (0.82 * params.c_p * _np(fast_exp(-params.c_t * (1.0 / tc - 1.0 / params.t_v)))
              * np.sqrt(params.c_m / tc) * (params.h_v + params.c * (tc - params.t_h0)))
    return _ret(q_rad + np.where(tc > params.t_v, q_evap, 0.0))


# --------------------------------------------------------------------------
# device-resident field and the K4 step (thermal.py:177-202, :321-354)
# --------------------------------------------------------------------------

class ThermalField:
    """Voxel grid on the GPU (thermal.py:177-202).  temperature_old/new are
    (nz, ny, nx) views of the kinetics GlobalFields' temperature buffers, so
    the thermal -> kinetics hand-off is the in-place roll of step_all, as in
    the reference (thermal.py:424-431)."""

    def __init__(self, temperature_old, temperature_new, r_c, state, h, z_top):
        self.temperature_old = temperature_old
        self.temperature_new = temperature_new
        self.r_c = r_c
        self.state = state
        self.h = float(h)
        self.z_top = int(z_top)

    @property
    def shape(self):
        return tuple(self.state.shape)

    def all_built(self):
        """True when every cell is STATE_BUILT with r_c == 1 (config 3)."""
        return bool((self.state == STATE_BUILT).all().item() and
                    (self.r_c == 1.0).all().item())

    def active_mask(self):
        return self.state != STATE_INACTIVE

    def enthalpy(self, params=DEFAULT_THERMAL):
        """Total rho c T h^3 over active voxels (thermal.py:193-196)."""
        m = self.active_mask()
        return float(params.rho * params.c * self.h**3 * self.temperature_old[m].sum().item())

    def commit_temperatures(self):
        """Adopt temperature_new as current (thermal.py:198-200)."""
        self.temperature_old.copy_(self.temperature_new)


def step_thermal(field, dt, params=DEFAULT_THERMAL, source=None, beam=None, losses=True,
                 bottom_dirichlet=None, nsub=None, all_built=None, stream=None):
    """Advance the thermal field by dt (thermal.py:321-354) with K4.

    temperature_old is left untouched and temperature_new receives the
    result; nsub > 1 alternates through scratch buffers exactly as
    _thermal_substeps (thermal.py:290-318).  Raises ValueError when a forced
    substep count violates the stability bound.
    """
    import ctypes as C
    import torch
    from . import _abi, _lib
    lib = _lib.require()
    dt_ok = stable_dt(field.h, params)
    if nsub is None:
        nsub = max(1, int(math.ceil(dt / dt_ok - 1e-12)))
    if dt / nsub > dt_ok * (1 + 1e-9):
        raise ValueError(f"dt/nsub={dt/nsub:.3e} exceeds stability bound {dt_ok:.3e} s")
    nz, ny, nx = field.shape
    if all_built is None:
        all_built = field.all_built()
    a = _abi.stencil_args(nx, ny, nz, field.z_top, dt / nsub, field.h, beam=beam,
                          source=source, losses=losses, bottom=bottom_dirichlet,
                          all_built=all_built)
    tp = _abi.thermal_from(params.kernel_tuple())
    st = _lib.stream_handle(stream)
    if nsub == 1:
        rc = lib.ti64_stencil_step(_lib.ptr(field.temperature_old),
                                   _lib.ptr(field.temperature_new), _lib.ptr(field.r_c),
                                   _lib.ptr(field.state), C.byref(tp), C.byref(a), st)
        _lib.check(rc, "ti64_stencil_step")
        return field
    bufs = getattr(field, "_substep_bufs", None)
    if bufs is None or bufs[0].shape != field.temperature_old.shape:
        bufs = (torch.empty_like(field.temperature_old), torch.empty_like(field.temperature_old))
        field._substep_bufs = bufs  # reused across macro steps (stream-ordered)
    rc = lib.ti64_thermal_substeps(_lib.ptr(field.temperature_old),
                                   _lib.ptr(field.temperature_new), _lib.ptr(bufs[0]),
                                   _lib.ptr(bufs[1]), _lib.ptr(field.r_c), _lib.ptr(field.state),
                                   C.byref(tp), C.byref(a), int(nsub), st)
    _lib.check(rc, "ti64_thermal_substeps")
    return field


def beam_rows(beams, source):
    """(n, 4) float64 device-table rows (x, y, src_peak, on) of a beam
    schedule, with the arithmetic of _abi.stencil_args (thermal.py:255-261)."""
    import numpy as np
    out = np.zeros((len(beams), 4))
    for k, b in enumerate(beams):
        if b[3]:
            out[k] = (b[0], b[1],
                      2.0 * b[2] / (math.pi * source.radius ** 2 * source.h_powder), 1.0)
    return out


class CoupledDomain:
    """Config 3: a fully built (nz, ny, nx) block, kinetics state at every
    cell, driven per step exactly as run_build's `couple` does
    (thermal.py:541-555): step_thermal(dt) then step_all(dt) on the aliased
    temperature buffers."""

    def __init__(self, nx=512, ny=512, nz=256, h=20e-6, t0=353.0, state0=(0.9, 0.0, 0.1),
                 device=None):
        import numpy as np
        import torch
        from .batch import GlobalFields
        n = nx * ny * nz
        t = torch.full((n,), float(t0), dtype=torch.float64)
        self.fields = GlobalFields(torch.full((n,), float(state0[0]), dtype=torch.float64),
                                   torch.full((n,), float(state0[1]), dtype=torch.float64),
                                   torch.full((n,), float(state0[2]), dtype=torch.float64),
                                   t, t.clone(), device=device)
        dev = self.fields.device
        self.field = ThermalField(self.fields.temperature_old.view(nz, ny, nx),
                                  self.fields.temperature_new.view(nz, ny, nx),
                                  torch.ones((nz, ny, nx), dtype=torch.float64, device=dev),
                                  torch.full((nz, ny, nx), STATE_BUILT, dtype=torch.uint8,
                                             device=dev), h, nz)
        self.shape = (nz, ny, nx)
        self.step = 0
        self._idle_bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
        self._bits_valid = False
        self._split_scratch = None  # the split step's row bitmap / list (allocated on use)
        self._overlap = None  # third temperature buffer, second scratch, kinetics stream
        del np

    def run(self, n_steps, dt, beams, source, kinetics_params=None, integrator_config=None,
            thermal_params=DEFAULT_THERMAL, bottom=353.0, losses=False, n_lanes=8, fused=None,
            split=True, graph=False, overlap=True):
        """n_steps coupled steps; beams[k] = (x, y, power, on) of step k.

        fused=True (default when nx % 32 == 0 and no losses) runs the device
        coupled step with ping-pong temperatures (bit-identical results): with
        split=True the stencil marks hot rows, then the kinetics of hot and
        transformed rows run (split=False: one K4+kinetics kernel);
        fused=False issues step_thermal + step_all per step like the reference.
        graph=True (fused path) reads each step's beam from a device table and
        replays a captured two-step CUDA graph (one host call per two steps;
        same results).  overlap=True (split path, no graph) rotates three
        temperature buffers and runs the row kinetics of step k on a second
        stream beside the stencil of step k+1 (same results)."""
        from .batch import step_all
        from .integrator import IntegratorConfig
        from .kinetics import DEFAULT_PARAMS
        kp = kinetics_params or DEFAULT_PARAMS
        cfg = integrator_config or IntegratorConfig(scheme="explicit")
        nz, ny, nx = self.shape
        if fused is None:
            fused = nx % 32 == 0 and not losses and dt <= cfg.dt_sub_max * (1 + 1e-9)
        if not fused:
            self._bits_valid = False
            for k in range(n_steps):
                step_thermal(self.field, dt, thermal_params, source, beams[k], losses=losses,
                             bottom_dirichlet=bottom, all_built=True)
                step_all(self.fields, dt, kp, cfg, n_lanes=n_lanes)
                self.step += 1
            return self
        return self._run_fused(n_steps, dt, beams, source, kp, cfg, thermal_params, bottom,
                               n_lanes, split, graph, overlap)

    def _run_fused(self, n_steps, dt, beams, source, kp, cfg, thermal_params, bottom, n_lanes,
                   split=True, graph=False, overlap=True):
        import ctypes as C
        from . import _abi, _lib
        lib = _lib.require()
        dt_ok = stable_dt(self.field.h, thermal_params)
        if dt > dt_ok * (1 + 1e-9):
            raise ValueError(f"dt={dt:.3e} exceeds stability bound {dt_ok:.3e} s")
        nz, ny, nx = self.shape
        tp = _abi.thermal_from(thermal_params.kernel_tuple())
        kpc = _abi.kparams_from(kp.kernel_tuple())
        cfgc = _abi.icfg_from(cfg.kernel_tuple())
        fs = self.fields.cstruct()
        st = _lib.stream_handle()
        if split and self._split_scratch is None:
            import torch
            words = _lib.check(lib.ti64_coupled_scratch_words(nx * ny * nz),
                               "ti64_coupled_scratch_words")
            self._split_scratch = torch.zeros(words, dtype=torch.int32,
                                              device=self.fields.device)
        cur, nxt = self.fields.temperature_old, self.fields.temperature_new
        scr = _lib.ptr(self._split_scratch) if split else None

        def call(src, dst, a, stream):
            rc = lib.ti64_coupled_step(_lib.ptr(src), _lib.ptr(dst), C.byref(fs), 0,
                                       _lib.ptr(self._idle_bits), scr, C.byref(tp), C.byref(a),
                                       C.byref(kpc), C.byref(cfgc), int(n_lanes),
                                       0 if self._bits_valid else 1, stream)
            _lib.check(rc, "ti64_coupled_step")
            self._bits_valid = True

        if split and overlap and not graph and n_steps >= 3:
            return self._run_overlapped(n_steps, dt, beams, source, bottom, n_lanes, fs, tp, kpc,
                                        cfgc)
        if graph and n_steps >= 3:
            import torch
            dev = self.fields.device
            tab = torch.from_numpy(beam_rows(beams[:n_steps], source)).to(dev)
            ctr = torch.zeros(1, dtype=torch.int64, device=dev)
            a = _abi.stencil_args(nx, ny, nz, nz, dt, self.field.h, beam=None, source=None,
                                  losses=False, bottom=bottom, all_built=True)
            a.src_r2inv = 1.0 / source.radius ** 2
            a.beam_tab_d, a.step_d = tab.data_ptr(), ctr.data_ptr()

            def step(src, dst, stream):
                call(src, dst, a, stream)
                _lib.check(lib.ti64_step_counter_add(_lib.ptr(ctr), 1, stream),
                           "ti64_step_counter_add")

            step(cur, nxt, st)  # eager first step (initialises the idle bits)
            cur, nxt = nxt, cur
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                cs = _lib.stream_handle()
                step(cur, nxt, cs)
                step(nxt, cur, cs)
            for _ in range((n_steps - 1) // 2):
                g.replay()
            if (n_steps - 1) % 2:
                step(cur, nxt, st)
                cur, nxt = nxt, cur
            torch.cuda.current_stream().synchronize()  # keep tab / ctr alive to the end
            del g
            self.step += n_steps
        else:
            for k in range(n_steps):
                a = _abi.stencil_args(nx, ny, nz, nz, dt, self.field.h, beam=beams[k],
                                      source=source, losses=False, bottom=bottom, all_built=True)
                call(cur, nxt, a, st)
                cur, nxt = nxt, cur
                self.step += 1
        # the reference ends a step with temperature_old == temperature_new
        if cur is self.fields.temperature_new:
            self.fields.temperature_old.copy_(cur)
        else:
            self.fields.temperature_new.copy_(cur)
        self.fields.traffic_bytes += 72 * self.fields.n_points * n_steps
        self.fields.steps_taken += n_steps
        return self


    def _run_overlapped(self, n_steps, dt, beams, source, bottom, n_lanes, fs, tp, kpc, cfgc):
        """The split coupled step with the row kinetics of step k on a second
        stream beside the stencil of step k+1 (ti64_coupled_step_streams): three
        temperature buffers in rotation, two scratch sets, one event per step
        ordering stencil(k+2) behind kinetics(k)."""
        import ctypes as C

        import torch
        from . import _abi, _lib
        lib = _lib.require()
        nz, ny, nx = self.shape
        dev = self.fields.device
        if self._overlap is None:
            self._overlap = (torch.empty_like(self.fields.temperature_old),
                             torch.zeros_like(self._split_scratch), torch.cuda.Stream(device=dev),
                             [torch.cuda.Event() for _ in range(3)])
        extra, scratch2, kin, events = self._overlap
        main = torch.cuda.current_stream()
        bufs = [self.fields.temperature_old, self.fields.temperature_new, extra]
        scr = [_lib.ptr(self._split_scratch), _lib.ptr(scratch2)]
        st, ks = _lib.stream_handle(main), _lib.stream_handle(kin)
        kin.wait_stream(main)  # earlier work on the fields (and the idle bits) is done
        for k in range(n_steps):
            a = _abi.stencil_args(nx, ny, nz, nz, dt, self.field.h, beam=beams[k], source=source,
                                  losses=False, bottom=bottom, all_built=True)
            if k >= 2:
                main.wait_event(events[(k - 2) % 3])  # kinetics(k-2) read B[(k+1) % 3]
            rc = lib.ti64_coupled_step_streams(
                _lib.ptr(bufs[k % 3]), _lib.ptr(bufs[(k + 1) % 3]), C.byref(fs), 0,
                _lib.ptr(self._idle_bits), scr[k % 2], C.byref(tp), C.byref(a), C.byref(kpc),
                C.byref(cfgc), int(n_lanes), 0 if self._bits_valid else 1, st, ks)
            _lib.check(rc, "ti64_coupled_step_streams")
            self._bits_valid = True
            events[k % 3].record(kin)
        main.wait_stream(kin)
        final = bufs[n_steps % 3]
        # the reference ends a step with temperature_old == temperature_new
        for t in (self.fields.temperature_old, self.fields.temperature_new):
            if t is not final:
                t.copy_(final)
        self.step += n_steps
        self.fields.traffic_bytes += 72 * self.fields.n_points * n_steps
        self.fields.steps_taken += n_steps
        return self


# --------------------------------------------------------------------------
# layer build (thermal.py:362-589)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class BuildGeometry:
    """Axis-aligned box part centred on a box base plate, SI units
    (thermal.py:362-403)."""

    plate_size: tuple = (1.2e-3, 1.2e-3, 0.2e-3)
    part_size: tuple = (1.0e-3, 1.0e-3, 0.25e-3)
    voxel: float = 0.05e-3

    def __post_init__(self):
        if self.voxel <= 0:
            raise ValueError("voxel size must be positive")
        for a, b in zip(self.part_size[:2], self.plate_size[:2]):
            if a > b + 1e-12:
                raise ValueError("part footprint must fit on the plate")

    @property
    def grid(self):
        h = self.voxel
        return (int(round(self.plate_size[0] / h)), int(round(self.plate_size[1] / h)),
                int(round(self.plate_size[2] / h)), int(round(self.part_size[2] / h)))

    @property
    def part_box(self):
        nx, ny, _, _ = self.grid
        h = self.voxel
        px = int(round(self.part_size[0] / h))
        py = int(round(self.part_size[1] / h))
        ix0, iy0 = (nx - px) // 2, (ny - py) // 2
        return (ix0, ix0 + px), (iy0, iy0 + py)

    @property
    def part_extent(self):
        (ix0, ix1), (iy0, iy1) = self.part_box
        h = self.voxel
        return (ix0 * h, iy0 * h, ix1 * h, iy1 * h)


@dataclass(frozen=True)
class BuildSchedule:
    """Time-stepping schedule of the layer build (thermal.py:406-417)."""

    dt_active: float = 2e-5
    interlayer_dwell: float = 1.0
    initial_dwell_steps: int = 2000
    growth_every: int = 10
    dt_max: float = 0.1
    final_cooldown: float = 100.0
    preheat: float = 293.0
    room: float = 293.0


def _fresh_solid(t, kinetics_params):
    from .batch import corrected_beta_state
    xs, xm, xb = corrected_beta_state([float(t)], kinetics_params)
    return float(xs[0]), float(xm[0]), float(xb[0])


def allocate_domain(geometry, schedule, kinetics_params=None, device=None):
    """Plate active (built, r_c = 1), part inactive; kinetics fields on every
    voxel with the thermal temperatures as views of theirs; plate
    microstructure = fresh solid corrected at the preheat (thermal.py:420-438)."""
    import torch
    from .batch import GlobalFields
    from .kinetics import DEFAULT_PARAMS
    kp = kinetics_params or DEFAULT_PARAMS
    nx, ny, nz_plate, n_layers = geometry.grid
    nz = nz_plate + n_layers
    fields = GlobalFields.allocate(nz * ny * nx, temperature=schedule.preheat, device=device)
    dev = fields.device
    state = torch.zeros((nz, ny, nx), dtype=torch.uint8, device=dev)
    state[:nz_plate] = STATE_BUILT
    r_c = torch.zeros((nz, ny, nx), dtype=torch.float64, device=dev)
    r_c[:nz_plate] = 1.0
    field = ThermalField(fields.temperature_old.view(nz, ny, nx),
                         fields.temperature_new.view(nz, ny, nx), r_c, state,
                         geometry.voxel, nz_plate)
    xs, xm, xb = _fresh_solid(schedule.preheat, kp)
    fields.x_alpha_s.fill_(xs)
    fields.x_alpha_m.fill_(xm)
    fields.x_beta.fill_(xb)
    return field, fields


def activate_layer(field, fields, geometry, schedule, kinetics_params=None):
    """Next powder layer at the preheat temperature, r_c = 0, fresh solid
    microstructure; ValueError once the build is complete (thermal.py:441-463)."""
    from .kinetics import DEFAULT_PARAMS
    nx, ny, nz_plate, n_layers = geometry.grid
    if field.z_top >= nz_plate + n_layers:
        raise ValueError("build complete: no layer left to activate")
    (ix0, ix1), (iy0, iy1) = geometry.part_box
    z = field.z_top
    field.state[z, iy0:iy1, ix0:ix1] = STATE_POWDER
    field.r_c[z, iy0:iy1, ix0:ix1] = 0.0
    field.temperature_old[z, iy0:iy1, ix0:ix1] = schedule.preheat
    field.temperature_new[z, iy0:iy1, ix0:ix1] = schedule.preheat
    nzz, nyy, nxx = field.shape
    xs, xm, xb = _fresh_solid(schedule.preheat, kinetics_params or DEFAULT_PARAMS)
    for arr, v in ((fields.x_alpha_s, xs), (fields.x_alpha_m, xm), (fields.x_beta, xb)):
        arr.view(nzz, nyy, nxx)[z, iy0:iy1, ix0:ix1] = v
    field.z_top = z + 1
    return field


def _active_prefix(field, fields):
    """GlobalFields over the active z-prefix, sharing storage (thermal.py:466-474)."""
    from .batch import GlobalFields
    nz, ny, nx = field.shape
    m = field.z_top * ny * nx
    return GlobalFields(*[getattr(fields, k)[:m] for k in (
        "x_alpha_s", "x_alpha_m", "x_beta", "temperature_old", "temperature_new",
        "seed_tracked", "seed_active", "seed_direction")], device=fields.device)


def cooldown_steps(duration, schedule, initial_steps):
    """Macro step sizes of one cool-down phase: `initial_steps` at dt_active,
    then doubling every growth_every steps up to dt_max, the last step cut to
    land on `duration` (thermal.py:477-495)."""
    steps = []
    t = 0.0
    dt = schedule.dt_active
    count = 0
    while t < duration - 1e-12:
        if count > initial_steps and (count - initial_steps) % schedule.growth_every == 0:
            dt = min(dt * 2.0, schedule.dt_max)
        dt_eff = min(dt, duration - t)
        steps.append(dt_eff)
        t += dt_eff
        count += 1
    return steps


def run_build(geometry, scan_path, schedule=BuildSchedule(), thermal_params=DEFAULT_THERMAL,
              kinetics_params=None, integrator_config=None, source=None, n_lanes=8,
              threads=1, probe_points=(), snapshot_hook=None, probe_hook=None, device=None):
    """Coupled scan-resolved build (thermal.py:498-589), every step on the GPU.

    Per layer: activate the powder layer, trace the layer's segments at
    dt_active, then the interlayer cool-down with growing steps; finally a
    cool-down with the bottom held at room temperature.  Each macro step is
    the reference's ``couple``: step_thermal (K4, losses on) then step_all
    on the active z-prefix, which consumes the (T_n, T_n+1) pair in place.

    Returns (field, fields, probes): probes maps probe index -> list of
    (t, T, x_alpha_s, x_alpha_m, x_beta) rows, gathered on the device every
    step and copied to the host once at the end; ``probes.timings`` holds
    the phase wall-clock split (synchronised at phase ends; the device work
    is asynchronous, so thermal_s / kinetics_s are not split and stay 0).
    ``threads`` is accepted and ignored.
    """
    import math
    import time as _time

    import torch

    from .batch import step_all
    from .integrator import IntegratorConfig
    from .kinetics import DEFAULT_PARAMS
    from .scanpath import beam_position, beam_timeline

    kp = kinetics_params or DEFAULT_PARAMS
    cfg = integrator_config or IntegratorConfig(scheme="explicit")
    source = source or HeatSource(h_powder=geometry.voxel)
    field, fields = allocate_domain(geometry, schedule, kp, device=device)
    nx, ny, nz_plate, n_layers = geometry.grid
    dev = fields.device

    class ProbeSet(dict):
        timings = None

    probes = ProbeSet({i: [] for i in range(len(probe_points))})
    probes.timings = {"active_s": 0.0, "cooldown_s": 0.0, "final_s": 0.0,
                      "thermal_s": 0.0, "kinetics_s": 0.0}
    pidx = []
    for (px, py, pz) in probe_points:
        ix = min(nx - 1, max(0, int(px / geometry.voxel)))
        iy = min(ny - 1, max(0, int(py / geometry.voxel)))
        iz = min(nz_plate + n_layers - 1, max(0, int(pz / geometry.voxel)))
        pidx.append((iz, iy, ix))
    flat = torch.tensor([(iz * ny + iy) * nx + ix for iz, iy, ix in pidx], dtype=torch.int64,
                        device=dev)
    rows = []   # (t_now, probes inside the active prefix, device row (n_probes, 5))
    t_now = 0.0
    counts = [0, 0]
    state_flat = field.state.view(-1)

    prefix = {}  # the active z-prefix view changes only when a layer is activated

    def couple(dt, beam, bottom, phase):
        nonlocal t_now
        step_thermal(field, dt, thermal_params, source, beam, losses=True,
                     bottom_dirichlet=bottom, all_built=False)
        counts[0] += 1
        if field.z_top not in prefix:
            prefix.clear()
            prefix[field.z_top] = _active_prefix(field, fields)
        step_all(prefix[field.z_top], dt, kp, cfg, n_lanes=n_lanes)
        counts[1] += 1
        t_now += dt
        if probe_hook is not None:
            probe_hook(t_now, field, fields)
        elif len(pidx):
            rows.append((t_now, [iz < field.z_top for iz, _, _ in pidx],
                         torch.stack([state_flat[flat].double(), fields.temperature_old[flat],
                                      fields.x_alpha_s[flat], fields.x_alpha_m[flat],
                                      fields.x_beta[flat]], 1)))

    def timed(phase, fn):
        torch.cuda.synchronize(dev)
        w0 = _time.perf_counter()
        fn()
        torch.cuda.synchronize(dev)
        probes.timings[phase] += _time.perf_counter() - w0

    for layer in range(n_layers):
        activate_layer(field, fields, geometry, schedule, kp)
        segments = scan_path.layer_segments(layer)
        if segments:
            spans = beam_timeline(segments)
            t_active = spans[-1][1]
            n_steps = max(1, int(math.ceil(t_active / schedule.dt_active - 1e-12)))

            def active():
                for k in range(n_steps):
                    tq = min((k + 0.5) * schedule.dt_active, t_active)
                    couple(schedule.dt_active, beam_position(segments, tq, spans),
                           schedule.preheat, "active_s")
            timed("active_s", active)

        def dwell():
            for dt in cooldown_steps(scan_path.dwell, schedule, schedule.initial_dwell_steps):
                couple(dt, None, schedule.preheat, "cooldown_s")
        timed("cooldown_s", dwell)
        if snapshot_hook is not None:
            snapshot_hook(f"layer_{layer:04d}", t_now, field, fields)

    def final():
        for dt in cooldown_steps(schedule.final_cooldown, schedule, 0):
            couple(dt, None, schedule.room, "final_s")
    timed("final_s", final)
    if snapshot_hook is not None:
        snapshot_hook("final", t_now, field, fields)
    assert counts[0] == counts[1], "coupling order violated"
    if rows:
        vals = torch.stack([r[2] for r in rows]).cpu().numpy()  # one copy for the run
        for k, (t, live, _) in enumerate(rows):
            for pi in range(len(pidx)):
                if live[pi] and vals[k, pi, 0] != STATE_INACTIVE:
                    probes[pi].append((t, float(vals[k, pi, 1]), float(vals[k, pi, 2]),
                                       float(vals[k, pi, 3]), float(vals[k, pi, 4])))
    return field, fields, probes
