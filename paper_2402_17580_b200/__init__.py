"""paper_2402_17580_b200 — B200-native (sm_100a) per-point Ti-6Al-4V
microstructure update: a drop-in for ti64micro's ``step_all`` path (explicit and Crank-Nicolson)
(reference: ti64micro/__init__.py:11-41 exports).

Importing needs no GPU; every compute call runs in libti64b200.so on an
sm_100 device and raises ``Ti64Unavailable`` otherwise (no CPU fallback).
"""

__version__ = "0.1.0"

from .kinetics import (
    DEFAULT_PARAMS,
    KineticsParams,
    PhaseRates,
    PhaseState,
    X_ALPHA_MAX,
    apply_corrections,
    compute_rates,
    liquid_fraction,
    x_alpha_eq,
    x_alpha_m_eq,
)
from .errors import FixedPointDivergence
from .integrator import (
    IntegratorConfig,
    SeedingState,
    integrate_history,
    integrate_interval,
    initiate_diffusion,
    analytic_beta_growth,
    step_crank_nicolson,
    wrms_norm,
    step_explicit,
)
from .batch import (
    BYTES_PER_POINT,
    SUPPORTED_LANES,
    AdvanceResult,
    BatchConvergenceError,
    EventCounters,
    blend,
    branch_dispatch,
    GlobalFields,
    advance,
    fast_exp,
    fast_ln,
    fast_pow,
    histogram,
    init_from_source,
    phase_sums,
    step_all,
)
from .sources import PulseHistory, PulseSweep, PulseTrain, RosenthalRaster, source_for_config
from ._lib import Ti64Error, Ti64Unavailable

from .fastmath import estrin_eval

__all__ = [
    "fast_exp", "fast_ln", "fast_pow", "estrin_eval",
    "liquid_fraction", "x_alpha_eq", "x_alpha_m_eq", "compute_rates", "apply_corrections",
    "PhaseRates", "blend", "branch_dispatch",
    "KineticsParams", "PhaseState", "DEFAULT_PARAMS", "X_ALPHA_MAX",
    "IntegratorConfig", "SeedingState",
    "step_explicit", "step_crank_nicolson", "integrate_interval", "integrate_history",
    "FixedPointDivergence", "wrms_norm", "initiate_diffusion", "analytic_beta_growth",
    "GlobalFields", "step_all", "BatchConvergenceError", "SUPPORTED_LANES", "BYTES_PER_POINT",
    "advance", "AdvanceResult", "EventCounters", "phase_sums", "histogram",
    "init_from_source",
    "PulseHistory", "RosenthalRaster", "PulseTrain", "PulseSweep", "source_for_config",
    "Ti64Error", "Ti64Unavailable",
]
