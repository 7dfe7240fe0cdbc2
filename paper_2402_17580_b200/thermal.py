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
