"""Heat-equation stencil path (config 3) — parameters and field container.

Mirrors the subset of ti64micro/thermal.py that the coupled config needs:
``ThermalParams`` / ``kernel_tuple`` (thermal.py:50-104), ``HeatSource``
(thermal.py:107-121), ``stable_dt`` (thermal.py:168-170), ``ThermalField``
(thermal.py:177-202) and ``step_thermal`` (thermal.py:321-354), the latter
running the K4 kernel (csrc/ti64_stencil.cu) on device-resident grids.
"""

import math
from dataclasses import dataclass, replace
from typing import NamedTuple

__all__ = ["KernelThermalParams", "ThermalParams", "DEFAULT_THERMAL", "HeatSource",
           "stable_dt", "STATE_INACTIVE", "STATE_POWDER", "STATE_BUILT", "SIGMA_S"]

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
    cur = field.temperature_old
    bufs = [None, None]
    for s in range(nsub):
        if s == nsub - 1:
            dst = field.temperature_new
        else:
            if bufs[s % 2] is None:
                bufs[s % 2] = torch.empty_like(field.temperature_old)
            dst = bufs[s % 2]
        rc = lib.ti64_stencil_step(_lib.ptr(cur), _lib.ptr(dst), _lib.ptr(field.r_c),
                                   _lib.ptr(field.state), C.byref(tp), C.byref(a), st)
        _lib.check(rc, "ti64_stencil_step")
        cur = dst
    return field


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
        del np

    def run(self, n_steps, dt, beams, source, kinetics_params=None, integrator_config=None,
            thermal_params=DEFAULT_THERMAL, bottom=353.0, losses=False, n_lanes=8, fused=None):
        """n_steps coupled steps; beams[k] = (x, y, power, on) of step k.

        fused=True (default when nx % 32 == 0 and no losses) runs the single-pass
        K4+kinetics kernel with ping-pong temperatures (bit-identical results);
        fused=False issues step_thermal + step_all per step like the reference."""
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
                               n_lanes)

    def _run_fused(self, n_steps, dt, beams, source, kp, cfg, thermal_params, bottom, n_lanes):
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
        cur, nxt = self.fields.temperature_old, self.fields.temperature_new
        for k in range(n_steps):
            a = _abi.stencil_args(nx, ny, nz, nz, dt, self.field.h, beam=beams[k],
                                  source=source, losses=False, bottom=bottom, all_built=True)
            rc = lib.ti64_coupled_step(_lib.ptr(cur), _lib.ptr(nxt), C.byref(fs),
                                       _lib.ptr(self._idle_bits), C.byref(tp), C.byref(a),
                                       C.byref(kpc), C.byref(cfgc), int(n_lanes),
                                       0 if self._bits_valid else 1, st)
            _lib.check(rc, "ti64_coupled_step")
            self._bits_valid = True
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
