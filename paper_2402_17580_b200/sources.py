"""Seeded temperature-history generators (K3) — host-side descriptors.

The reference integrates whatever temperatures the caller writes into
``temperature_new`` before each ``step_all`` (ti64micro/batch.py:762,
thermal.py:541-555).  The BASELINE configs prescribe synthetic histories
instead; here they are generated ON DEVICE, per point and per step, from a
counter-based RNG keyed by (seed, global point index, draw), so a point's
history is independent of how points are sharded across GPUs.

Each class only builds the ``ti64_tempgen`` descriptor (include/ti64_b200.h);
the arithmetic lives in csrc/ti64_sources.cuh and is defined in DESIGN.md §3.
Per-step beam positions of the moving source (config 1) are a host-side
table, like the reference's host-side ``scanpath.beam_position``
(scanpath.py:206-212).
"""

import math
from dataclasses import dataclass

import numpy as np

from . import _abi

__all__ = ["PulseHistory", "RosenthalRaster", "PulseTrain", "PulseSweep",
           "source_for_config"]


def _fill(gen, values):
    for i, v in enumerate(values):
        gen.p[i] = float(v)


@dataclass(frozen=True)
class PulseHistory:
    """Config 0: T_i(t) = base + A_i exp(-((t - t_i) / w_i)^2), one pulse."""

    seed: int = 0
    dt: float = 1e-5
    base: float = 300.0
    amp: tuple = (900.0, 1900.0)
    center: tuple = (0.02, 0.15)
    width: tuple = (2e-4, 5e-3)

    kind = _abi.SRC_PULSE
    max_pulses = 1

    def tempgen(self, point_offset=0, beam_ptr=None, beam_steps=0):
        g = _abi.TempGen()
        g.kind, g.max_pulses, g.seed = self.kind, 1, self.seed
        g.point_offset, g.dt, g.base = point_offset, self.dt, self.base
        _fill(g, (*self.amp, *self.center, *self.width))
        return g

    def beam_table(self, n_rows):
        return None


@dataclass(frozen=True)
class RosenthalRaster:
    """Config 1: quasi-steady Rosenthal point source rastering the top plane.

    T = ambient + (eta P / (2 pi k)) / R * exp(-(v / (2 alpha)) (R + xi)),
    capped at ``cap``; xi is the coordinate along the beam's travel
    direction, R the distance to the beam.  Lattice point p -> (i, j, k) =
    (p % nx, (p // nx) % ny, p // (nx ny)) at (i h, j h) with depth k h below
    the scanned plane.  Raster: tracks along x over the lattice width, 100 um
    hatch in y, serpentine direction, restarting at y = 0 after the last
    track.
    """

    dt: float = 2e-5
    nx: int = 128
    ny: int = 128
    nz: int = 64
    h: float = 20e-6
    power: float = 200.0
    absorptivity: float = 0.35
    speed: float = 1.0
    hatch: float = 100e-6
    ambient: float = 353.0
    conductivity: float = 7.0
    diffusivity: float = 3e-6
    cap: float = 3000.0
    seed: int = 0

    kind = _abi.SRC_ROSENTHAL
    max_pulses = 0

    @property
    def n_points(self):
        return self.nx * self.ny * self.nz

    @property
    def track_length(self):
        return self.nx * self.h

    @property
    def n_tracks(self):
        return int(self.track_length / self.hatch + 1e-9) + 1

    def beam_table(self, n_rows):
        """(n_rows, 3) float64: beam (x, y, dir) at t_n = n dt."""
        out = np.empty((n_rows, 3))
        L = self.track_length
        for n in range(n_rows):
            t = float(n) * self.dt
            s = t * self.speed
            q = math.floor(s / L)
            within = s - q * L
            d = 1.0 if q % 2 == 0 else -1.0
            out[n, 0] = within if d > 0 else L - within
            out[n, 1] = float(q % self.n_tracks) * self.hatch
            out[n, 2] = d
        return out

    def straight_runs(self, tab):
        """Per row r: how many rows from r on (r included) continue one
        straight pass — same y, same direction, x advancing by exactly
        dir * speed * dt (to 1e-12 m).  The kernel's multi-step rest bound is
        only applied inside such a run."""
        n = len(tab)
        step = self.speed * self.dt
        run = np.ones(n, np.int64)
        if n > 1:
            ok = ((tab[1:, 1] == tab[:-1, 1]) & (tab[1:, 2] == tab[:-1, 2]) &
                  (np.abs(tab[1:, 0] - tab[:-1, 0] - tab[:-1, 2] * step) <= 1e-12))
            for r in range(n - 2, -1, -1):
                if ok[r]:
                    run[r] = run[r + 1] + 1
        return np.minimum(run, 1 << 24)

    def packed_beam(self, n_rows):
        """Device layout of the beam table: the (n_rows, 3) doubles, padded to
        an even count, then n_rows float32 rows (x, y, dir, run) for the
        kernel's FP32 filters (run = straight_runs); one float64 array."""
        tab = self.beam_table(n_rows)
        nd = 3 * n_rows + (3 * n_rows) % 2
        out = np.zeros(nd + 2 * n_rows)
        out[:3 * n_rows] = tab.ravel()
        f = np.zeros((n_rows, 4), np.float32)
        f[:, :3] = tab
        f[:, 3] = self.straight_runs(tab)
        out[nd:] = f.view(np.float64).ravel()
        return out

    def noop_threshold(self):
        """(arg_noop_f32, T_noop): for vk*(R+xi) >= arg_noop the source term
        (coef/R)*fast_exp(-arg) < ulp(base)/4, so T == min(base, cap) bit for
        bit (R >= arg/(2 vk) bounds coef/R; fast_exp's relative error is
        < 1e-9).  arg_noop_f32 adds a margin far above the FP32 estimate's
        error on this lattice."""
        coef, vk = self._coef_vk()
        quarter_ulp = math.ulp(self.ambient) / 4.0
        arg = 1.0
        while 2.0 * vk * coef / arg * math.exp(-arg) * 1.01 >= quarter_ulp:
            arg += 1.0
        extent = math.sqrt((self.nx * self.h) ** 2 + (self.ny * self.h) ** 2 +
                           (self.nz * self.h) ** 2) + self.track_length + \
            self.n_tracks * self.hatch
        margin = max(1.0, 64.0 * vk * 1.2e-7 * extent)
        return arg + margin, min(self.ambient, self.cap)

    def _coef_vk(self):
        coef = self.absorptivity * self.power / (2.0 * math.pi * self.conductivity)
        vk = self.speed / (2.0 * self.diffusivity)
        return coef, vk

    def tempgen(self, point_offset=0, beam_ptr=None, beam_steps=0):
        g = _abi.TempGen()
        g.kind, g.max_pulses, g.seed = self.kind, 0, self.seed
        g.point_offset, g.dt, g.base = point_offset, self.dt, self.ambient
        coef, vk = self._coef_vk()
        thr, t_noop = self.noop_threshold()
        _fill(g, (coef, vk, self.cap, thr, t_noop))
        g.beam_d = beam_ptr
        g.beam_steps = beam_steps
        g.nx, g.ny, g.nz, g.h = self.nx, self.ny, self.nz, self.h
        # FP32 constants of the kernel's estimates: vk, coef, vk*log2(e),
        # arg_noop/vk (the no-op filter compares R against arg_noop/vk - xi)
        g.pf[0] = vk
        g.pf[1] = coef
        g.pf[2] = vk * 1.4426950408889634
        g.pf[3] = thr / vk
        g.pf[4] = self.speed * self.dt  # beam advance per row inside a straight run
        return g


@dataclass(frozen=True)
class PulseTrain:
    """Config 2: base + sum_k A_k exp(-((t - t_k)/w_k)^2), 10 re-scan pulses.

    A_k = (A_1 * 0.6^k) * U(0.9, 1.1) with A_1 ~ U(1500, 2500) and 0.6^k
    formed by repeated multiplication; t_k = (t0 + 0.04 k) + U(-2, 2) ms;
    w_k ~ U(0.5, 3) ms.  Initial x_alpha_s ~ U(0.8, 0.95), x_beta = 1 - x_alpha_s.
    """

    seed: int = 2
    dt: float = 1e-5
    base: float = 353.0
    n_pulses: int = 10
    amp1: tuple = (1500.0, 2500.0)
    jitter_amp: tuple = (0.9, 1.1)
    t0: float = 0.02
    spacing: float = 0.04
    jitter_t: tuple = (-2e-3, 2e-3)
    width: tuple = (5e-4, 3e-3)
    decay: float = 0.6
    xs0: tuple = (0.8, 0.95)

    kind = _abi.SRC_PULSE_TRAIN

    @property
    def max_pulses(self):
        return self.n_pulses

    def tempgen(self, point_offset=0, beam_ptr=None, beam_steps=0):
        g = _abi.TempGen()
        g.kind, g.max_pulses, g.seed = self.kind, self.n_pulses, self.seed
        g.point_offset, g.dt, g.base = point_offset, self.dt, self.base
        _fill(g, (*self.amp1, *self.jitter_amp, self.t0, self.spacing,
                  *self.jitter_t, *self.width, self.decay, *self.xs0))
        return g

    def beam_table(self, n_rows):
        return None


@dataclass(frozen=True)
class PulseSweep:
    """Config 4: 1..20 pulses per point, amplitudes U(600, 3000) K, centres
    U(0, 1) s, widths log-uniform on [1e-4, 1e-2] s (w = fast_exp(U(ln lo, ln hi)))."""

    seed: int = 4
    dt: float = 1e-5
    base: float = 300.0
    n_pulses_max: int = 20
    amp: tuple = (600.0, 3000.0)
    center: tuple = (0.0, 1.0)
    width: tuple = (1e-4, 1e-2)

    kind = _abi.SRC_PULSE_SWEEP

    @property
    def max_pulses(self):
        return self.n_pulses_max

    def tempgen(self, point_offset=0, beam_ptr=None, beam_steps=0):
        g = _abi.TempGen()
        g.kind, g.max_pulses, g.seed = self.kind, self.n_pulses_max, self.seed
        g.point_offset, g.dt, g.base = point_offset, self.dt, self.base
        _fill(g, (*self.amp, *self.center, math.log(self.width[0]),
                  math.log(self.width[1])))
        return g

    def beam_table(self, n_rows):
        return None


def source_for_config(cfg):
    """Generator of BASELINE.json config `cfg` (0, 1, 2 or 4)."""
    return {0: PulseHistory(), 1: RosenthalRaster(), 2: PulseTrain(),
            4: PulseSweep()}[cfg]
