"""ctypes mirrors of the POD structs in include/ti64_b200.h.

Pure layout definitions (no library loading, no GPU).  Field order follows
the reference NamedTuples they mirror: KernelKineticsParams
(ti64micro/kinetics.py:41-62), KernelIntegratorConfig (batch.py:82-92),
KernelThermalParams (thermal.py:50-66).
"""

import ctypes as C

__all__ = [
    "KParams", "ICfg", "Fields", "TempGen", "Counters", "Thermal",
    "StencilArgs", "kparams_from", "icfg_from", "thermal_from",
    "SCHEME_EXPLICIT", "SCHEME_CRANK_NICOLSON",
    "SEED_NONE", "SEED_BETA_TO_ALPHA_S", "SEED_ALPHA_S_TO_BETA",
    "SRC_PULSE", "SRC_ROSENTHAL", "SRC_PULSE_TRAIN", "SRC_PULSE_SWEEP",
    "TOTALS_FIELDS",
]

SCHEME_EXPLICIT = 0
SCHEME_CRANK_NICOLSON = 1
SEED_NONE = 0
SEED_BETA_TO_ALPHA_S = 1
SEED_ALPHA_S_TO_BETA = 2

SRC_PULSE = 1
SRC_ROSENTHAL = 2
SRC_PULSE_TRAIN = 3
SRC_PULSE_SWEEP = 4

# order of ti64_counters.totals_d
TOTALS_FIELDS = ("point_updates", "n_form", "n_grow_or_am", "n_grow", "n_am",
                 "n_dissolve", "martensite_events", "phase_switches")

_KP_FIELDS = ("t_liq", "t_sol", "t_as_start", "t_as_end", "t_am_start", "t_inf",
              "k_alpha_eq", "k_alpha_m_eq", "k1", "k2", "k3", "f", "t_as_reg",
              "exp_as_lo", "exp_as_hi", "exp_b_lo", "exp_b_hi", "c_alpha_s", "c_beta")


class KParams(C.Structure):
    _fields_ = [(n, C.c_double) for n in _KP_FIELDS]


class ICfg(C.Structure):
    _fields_ = [("scheme", C.c_int64), ("dt_sub_max", C.c_double),
                ("eps_abs", C.c_double), ("eps_rel", C.c_double),
                ("max_fixed_point_iters", C.c_int64),
                ("initiation_threshold", C.c_double), ("stuck_tol", C.c_double),
                ("max_halvings", C.c_int64)]


class Fields(C.Structure):
    _fields_ = [("x_alpha_s", C.c_void_p), ("x_alpha_m", C.c_void_p),
                ("x_beta", C.c_void_p), ("temperature_old", C.c_void_p),
                ("temperature_new", C.c_void_p), ("seed_tracked", C.c_void_p),
                ("seed_active", C.c_void_p), ("seed_direction", C.c_void_p)]


class TempGen(C.Structure):
    _fields_ = [("kind", C.c_int32), ("max_pulses", C.c_int32),
                ("seed", C.c_uint64), ("point_offset", C.c_int64),
                ("dt", C.c_double), ("base", C.c_double),
                ("p", C.c_double * 16), ("beam_d", C.c_void_p),
                ("beam_steps", C.c_int64), ("nx", C.c_int64), ("ny", C.c_int64),
                ("nz", C.c_int64), ("h", C.c_double), ("pf", C.c_float * 8)]


class Counters(C.Structure):
    _fields_ = [("martensite_d", C.c_void_p), ("switches_d", C.c_void_p),
                ("totals_d", C.c_void_p)]


_TH_FIELDS = ("k_ms", "k_p", "rho_c", "t_sol", "t_liq", "t_inf", "emissivity",
              "sigma_s", "t_v", "c_p", "c_t", "c_m", "h_v", "t_h0", "t_max_clamp",
              "c_heat")


class Thermal(C.Structure):
    _fields_ = [(n, C.c_double) for n in _TH_FIELDS]


class StencilArgs(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("z_top", C.c_int64), ("dt", C.c_double), ("h", C.c_double),
                ("beam_x", C.c_double), ("beam_y", C.c_double),
                ("source_on", C.c_int32), ("losses_on", C.c_int32),
                ("bc_bottom_on", C.c_int32), ("all_built", C.c_int32),
                ("src_peak", C.c_double), ("src_r2inv", C.c_double),
                ("bc_bottom", C.c_double), ("z_base", C.c_int64),
                ("nz_stored", C.c_int64), ("z_begin", C.c_int64), ("z_end", C.c_int64),
                ("beam_tab_d", C.c_void_p), ("step_d", C.c_void_p)]


def stencil_args(nx, ny, nz, z_top, dt, h, beam=None, source=None, losses=False,
                 bottom=None, all_built=False, slab=None):
    """StencilArgs for a whole grid (slab=None) or a z-slab
    slab=(z_base, nz_stored, z_begin, z_end)."""
    import math
    a = StencilArgs(nx=nx, ny=ny, nz=nz, z_top=z_top, dt=dt, h=h)
    if beam is not None and source is not None and beam[3]:
        a.beam_x, a.beam_y = beam[0], beam[1]
        a.src_peak = 2.0 * beam[2] / (math.pi * source.radius ** 2 * source.h_powder)
        a.src_r2inv = 1.0 / source.radius ** 2
        a.source_on = 1
    else:
        a.src_r2inv = 1.0
    a.losses_on = 1 if losses else 0
    a.bc_bottom_on = 0 if bottom is None else 1
    a.bc_bottom = 0.0 if bottom is None else float(bottom)
    a.all_built = 1 if all_built else 0
    if slab is None:
        slab = (0, nz, 0, z_top)
    a.z_base, a.nz_stored, a.z_begin, a.z_end = slab
    return a


def kparams_from(kernel_tuple):
    """KernelKineticsParams (or any object with its fields) -> KParams."""
    return KParams(*[float(getattr(kernel_tuple, n)) for n in _KP_FIELDS])


def icfg_from(kernel_tuple):
    """KernelIntegratorConfig -> ICfg."""
    k = kernel_tuple
    return ICfg(int(k.scheme), float(k.dt_sub_max), float(k.eps_abs),
                float(k.eps_rel), int(k.max_fixed_point_iters),
                float(k.initiation_threshold), float(k.stuck_tol),
                int(k.max_halvings))


def thermal_from(kernel_tuple):
    """KernelThermalParams -> Thermal."""
    return Thermal(*[float(getattr(kernel_tuple, n)) for n in _TH_FIELDS])
