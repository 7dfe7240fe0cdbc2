// ti64_sources.cuh — on-device seeded temperature-history generators (K3).
//
// Definitions are shared bit for bit with the checker in
// oracle/ti64_oracle.c (oracle_gen_temperature1).  Per-point parameters come
// from a counter-based splitmix64 hash of (seed, global point index, draw),
// so a point's history does not depend on sharding or launch shape.
//
// Pulse sums skip pulses whose contribution is provably an exact no-op:
// outside a conservative step window |t - t_c| > wk w around its centre,
// A*fast_exp(-u^2) < ulp(base)/2 <= ulp(running sum)/2 (every term is >= 0),
// so adding it cannot change a bit (wk from the amplitude
// bound and the base, pulse_window_k in ti64_kernels.cu).
#pragma once
#include "ti64_fastmath.cuh"
#include "../../include/ti64_b200.h"

#ifndef PULSE_CACHE
#define PULSE_CACHE 1
#endif

namespace ti64 {

__host__ __device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

__device__ __forceinline__ double u01(uint64_t seed, uint64_t point, uint64_t k) {
  const uint64_t b = splitmix(splitmix(seed ^ splitmix(point)) ^ (k * 0xD1B54A32D192ED03ULL));
  return __dmul_rn(__ull2double_rn(b >> 11), 0x1.0p-53);
}

// u01 with the point's key h = splitmix(seed ^ splitmix(point)) formed once
__device__ __forceinline__ uint64_t point_key(uint64_t seed, uint64_t point) {
  return splitmix(seed ^ splitmix(point));
}
__device__ __forceinline__ double u01_keyed(uint64_t h, uint64_t k) {
  const uint64_t b = splitmix(h ^ (k * 0xD1B54A32D192ED03ULL));
  return __dmul_rn(__ull2double_rn(b >> 11), 0x1.0p-53);
}

__device__ __forceinline__ double unif(double lo, double hi, double u) {
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
}

// single-MUFU FP32 approximations (used only for conservative estimates)
__device__ __forceinline__ float exp2f_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrtf_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// (double)n exactly, n in [0, 2^52): one DADD instead of an I2F conversion
__device__ __forceinline__ double step_to_double(int64_t n) {
  return __dsub_rn(__hiloint2double(0x43300000 | (int)(n >> 32), (int)(uint32_t)n),
                   4503599627370496.0);
}

// Gaussian pulse contribution a*fast_exp(-u^2), u = (t - tc)*inv_w.
// -u*u is never NaN and <= 0; below -708 fast_exp is exactly 0.
template <class C = CoefBank>
__device__ __forceinline__ double add_pulse(double s, double a, double tc, double inv_w,
                                            double t, const C& c = C()) {
  const double u = __dmul_rn(__dsub_rn(t, tc), inv_w);
  const double uu = __dmul_rn(u, u);
  if (uu > 708.0) return __dadd_rn(s, 0.0);  // a * 0.0 == +0.0
  return __dadd_rn(s, __dmul_rn(a, exp_core(-uu, c)));
}

// Up to MAXP Gaussian pulses per point (configs 0, 2, 4).  Pulse k is only
// evaluated on steps [lo_k, hi_k]; a live mask plus the next step at which
// it changes keep the per-step cost at the live pulses.
template <int MAXP>
struct PulseSet {
  static constexpr int MAX_PULSES = MAXP;
  double base;
  double a[MAXP], tc[MAXP], inv_w[MAXP];
  int lo[MAXP], hi[MAXP];
  int np;
  unsigned live;
  int64_t next_event;
#if PULSE_CACHE
  // the lowest live pulse (the first term of the sum) in registers: usually
  // the only live one, so the per-step sum needs no local-memory loads
  double ca, ctc, ciw;
#endif

  // wk (> 0): half-width of the live window in widths, from the host
  // (pulse_window_k): outside it a*fast_exp(-u^2) < ulp(base)/2, an exact no-op.
  // Only pulses whose live window meets the caller's step range [n_lo, n_hi]
  // are kept (appended in pulse order, so the sum keeps its association): a
  // pulse that is never live in the range is never added to the sum, and the
  // per-thread table (local memory) holds the few pulses of a launch window
  // instead of every pulse of the point.
  __device__ __forceinline__ void add(double ak, double tck, double w, double dt, double wk,
                                      int64_t n_lo, int64_t n_hi) {
    // conservative window: outside it |t - tc| >= wk w - O(ulp) (2-step margin)
    const double l = floor((tck - wk * w) / dt) - 2.0;
    const double h = ceil((tck + wk * w) / dt) + 2.0;
    const int li = l < -1.0e9 ? -1000000000 : (l > 1.0e9 ? 1000000000 : (int)l);
    const int hi_ = h < -1.0e9 ? -1000000000 : (h > 1.0e9 ? 1000000000 : (int)h);
    if ((int64_t)hi_ < n_lo || (int64_t)li > n_hi) return;
    const int k = np++;
    a[k] = ak;
    tc[k] = tck;
    inv_w[k] = div_rn(1.0, w);
    lo[k] = li;
    hi[k] = hi_;
  }

  __device__ __forceinline__ void rescan(int64_t n) {
    live = 0u;
    int64_t nxt = INT64_MAX;
    for (int k = 0; k < np; ++k) {
      if (n >= lo[k] && n <= hi[k]) {
        live |= 1u << k;
        nxt = min(nxt, (int64_t)hi[k] + 1);
      } else if (n < lo[k]) {
        nxt = min(nxt, (int64_t)lo[k]);
      }
    }
    next_event = nxt;
#if PULSE_CACHE
    if (live) {
      const int k = __ffs(live) - 1;
      ca = a[k];
      ctc = tc[k];
      ciw = inv_w[k];
    }
#endif
  }

  // FP32 estimate of T - base (relative error < 1e-5; u is formed in FP64
  // so the only FP32 error is in the exponential and the product).
  __device__ __forceinline__ float excess_estimate(int64_t n, double dt) {
    if (n >= next_event || n < 0) rescan(n);
    unsigned m = live;
    if (m == 0u) return 0.0f;
    const double t = __dmul_rn(step_to_double(n), dt);
    float e = 0.0f;
#if PULSE_CACHE
    {
      const float u = (float)__dmul_rn(__dsub_rn(t, ctc), ciw);
      e += (float)ca * exp2f_approx(-u * u * 1.44269504f);
      m &= m - 1;
    }
#endif
    while (m) {
      const int k = __ffs(m) - 1;
      m &= m - 1;
      const float u = (float)__dmul_rn(__dsub_rn(t, tc[k]), inv_w[k]);
      e += (float)a[k] * exp2f_approx(-u * u * 1.44269504f);
    }
    return e;
  }

  template <class C = CoefBank>
  __device__ __forceinline__ double temp(int64_t n, double dt, const C& c = C()) {
    if (n >= next_event || n < 0) rescan(n);
    double s = base;
    unsigned m = live;
    if (m == 0u) return s;  // every pulse is an exact no-op: T == base
    const double t = __dmul_rn(step_to_double(n), dt);
#if PULSE_CACHE
    s = add_pulse(s, ca, ctc, ciw, t, c);
    m &= m - 1;
#endif
    while (m) {
      const int k = __ffs(m) - 1;
      m &= m - 1;
      s = add_pulse(s, a[k], tc[k], inv_w[k], t, c);
    }
    return s;
  }
};

// A pulse visitor with PulseSet's add() signature for the work-class order of
// the fused advance: "will this point get hot (T near T_alpha_s,end or above)
// within the coming launch window?"  A pulse of amplitude above `thr` reaches
// base + thr inside |t - t_c| <= rw w (rw from the largest amplitude, host
// side); live_soon: some pulse is live (off the base temperature) within the
// window.  Only scheduling hints: overlapping smaller pulses are ignored and
// no result depends on them.
template <int MAXP>
struct HotProbe {
  static constexpr int MAX_PULSES = MAXP;
  double base;
  int np;
  unsigned live;
  int64_t next_event;
  double thr, rw, t_lo, t_hi;
  float inv_thr;
  bool hot, live_soon;
  __device__ __forceinline__ void add(double ak, double tck, double w, double, double wk,
                                      int64_t, int64_t) {
    const double rl = wk * w;  // the live window (PulseSet::add), without its 2-step margin
    live_soon |= (tck + rl >= t_lo) & (tck - rl <= t_hi);
    if (ak > thr) {
      // radius of the pulse's own amplitude (FP32: a hint), capped by rw
      const float q = sqrtf(__logf((float)ak * inv_thr)) * 1.02f + 0.02f;
      const double r = (double)fminf(q, (float)rw) * w;
      hot |= (tck + r >= t_lo) & (tck - r <= t_hi);
    }
  }
};

// live-window half-width of the pulse kinds (g.pf[7], set by the library's
// entry points from pulse_window_k); 26.7 (u^2 > 708: fast_exp is exactly 0)
// is exact for any base and amplitude
__device__ __forceinline__ double window_k(const ti64_tempgen& g) {
  const double k = (double)g.pf[7];
  return k > 0.0 ? k : 26.7;
}

// A pulse centred farther than g.pf[6] seconds (the library's bound on the
// live half-width wk w of any pulse of the generator, + 4 steps; 0: unknown)
// from the step range [n_lo, n_hi] is not live anywhere in it: add() would
// drop it, so its amplitude and width need not be drawn at all.
__device__ __forceinline__ bool pulse_out_of_reach(double tc, const ti64_tempgen& g,
                                                   int64_t n_lo, int64_t n_hi) {
  const double reach = (double)g.pf[6];
  return (reach > 0.0) & ((tc + reach < __dmul_rn((double)n_lo, g.dt)) |
                          (tc - reach > __dmul_rn((double)n_hi, g.dt)));
}

// config 0 (TI64_SRC_PULSE): p = {A_lo, A_hi, tc_lo, tc_hi, w_lo, w_hi}
template <class PS>
__device__ __forceinline__ void init_pulse1(PS& ps, const ti64_tempgen& g,
                                            uint64_t pt, int64_t n_lo, int64_t n_hi) {
  ps.base = g.base;
  ps.np = 0;
  const double tc = unif(g.p[2], g.p[3], u01(g.seed, pt, 1));
  if (!pulse_out_of_reach(tc, g, n_lo, n_hi)) {
    const double a = unif(g.p[0], g.p[1], u01(g.seed, pt, 0));
    const double w = unif(g.p[4], g.p[5], u01(g.seed, pt, 2));
    ps.add(a, tc, w, g.dt, window_k(g), n_lo, n_hi);
  }
  ps.next_event = -1;
  ps.live = 0u;
}

// config 2 (TI64_SRC_PULSE_TRAIN): p = {A1_lo, A1_hi, j_lo, j_hi, t0, spacing,
// tj_lo, tj_hi, w_lo, w_hi, decay, xs_lo, xs_hi}
template <class PS>
__device__ __forceinline__ void init_train(PS& ps, const ti64_tempgen& g,
                                           uint64_t pt, int64_t n_lo, int64_t n_hi) {
  ps.base = g.base;
  const int npt = g.max_pulses < PS::MAX_PULSES ? g.max_pulses : PS::MAX_PULSES;
  ps.np = 0;
  const double a1 = unif(g.p[0], g.p[1], u01(g.seed, pt, 0));
  double scale = 1.0;
  for (int k = 0; k < npt; ++k) {
    const double tc = __dadd_rn(__dadd_rn(g.p[4], __dmul_rn(g.p[5], (double)k)),
                                unif(g.p[6], g.p[7], u01(g.seed, pt, 2 + 3 * k)));
    if (!pulse_out_of_reach(tc, g, n_lo, n_hi)) {
      const double a = __dmul_rn(__dmul_rn(a1, scale),
                                 unif(g.p[2], g.p[3], u01(g.seed, pt, 1 + 3 * k)));
      const double w = unif(g.p[8], g.p[9], u01(g.seed, pt, 3 + 3 * k));
      ps.add(a, tc, w, g.dt, window_k(g), n_lo, n_hi);
    }
    scale = __dmul_rn(scale, g.p[10]);
  }
  ps.next_event = -1;
  ps.live = 0u;
}

// config 4 (TI64_SRC_PULSE_SWEEP): p = {A_lo, A_hi, c_lo, c_hi, lnw_lo, lnw_hi}
template <class PS>
__device__ __forceinline__ void init_sweep(PS& ps, const ti64_tempgen& g,
                                           uint64_t pt, int64_t n_lo, int64_t n_hi) {
  ps.base = g.base;
  const uint64_t h = point_key(g.seed, pt);
  int np_ = 1 + (int)__dmul_rn(u01_keyed(h, 0), (double)g.max_pulses);
  np_ = np_ < PS::MAX_PULSES ? np_ : PS::MAX_PULSES;
  ps.np = 0;
  // pass 1: the centres only (one draw per pulse); pass 2: each lane draws
  // amplitude and width of ITS pulses within reach, in pulse order -- lanes
  // work on different pulses at once instead of every lane waiting through
  // all 20 pulse slots for the few lanes that need one (MAX_PULSES <= 32)
  unsigned near = 0u;
  for (int k = 0; k < np_; ++k) {
    const double tc = unif(g.p[2], g.p[3], u01_keyed(h, 2 + 3 * k));
    if (!pulse_out_of_reach(tc, g, n_lo, n_hi)) near |= 1u << k;
  }
  while (near) {
    const int k = __ffs(near) - 1;
    near &= near - 1u;
    const double tc = unif(g.p[2], g.p[3], u01_keyed(h, 2 + 3 * k));
    const double a = unif(g.p[0], g.p[1], u01_keyed(h, 1 + 3 * k));
    const double w = fast_exp(unif(g.p[4], g.p[5], u01_keyed(h, 3 + 3 * k)));
    ps.add(a, tc, w, g.dt, window_k(g), n_lo, n_hi);
  }
  ps.next_event = -1;
  ps.live = 0u;
}

// config 1 (TI64_SRC_ROSENTHAL): p = {coef, v/(2 alpha), cap, arg_noop_f32,
// T_noop}.  beam_d holds beam_steps rows of 3 doubles (x, y, dir), padded to
// an even count, followed by beam_steps rows of 4 floats (x, y, dir, 0) for
// the FP32 no-op filter (sources.RosenthalRaster.packed_beam).
//
// No-op filter: when vk*(R + xi) >= arg_noop the Rosenthal term
// (coef/R)*fast_exp(-arg) is below a quarter-ulp of `base` (host-derived bound,
// sources.py), so T == min(base, cap) exactly.  An FP32 estimate of the
// argument (error < 1e-2 on this lattice) against arg_noop + 1 selects that
// case without any FP64 work; everything else takes the exact FP64 path.
struct Rosenthal {
  double x, y, dd;
  float xf, yf, ddf;

  __device__ __forceinline__ void init(const ti64_tempgen& g, uint64_t pt) {
    const int64_t p = (int64_t)pt;
    const int64_t i = p % g.nx;
    const int64_t j = (p / g.nx) % g.ny;
    const int64_t k = p / (g.nx * g.ny);
    x = __dmul_rn((double)i, g.h);
    y = __dmul_rn((double)j, g.h);
    const double d = __dmul_rn((double)k, g.h);
    dd = __dmul_rn(d, d);
    xf = (float)x;
    yf = (float)y;
    ddf = (float)dd;
  }

  static __device__ __forceinline__ const float4* ftab(const ti64_tempgen& g) {
    return reinterpret_cast<const float4*>(g.beam_d + ((3 * g.beam_steps + 1) & ~1LL));
  }

  // FP32 geometry of step row bf: returns s = R^2 and sets xi
  __device__ __forceinline__ float geom(const float4& bf, float& xif) const {
    xif = (xf - bf.x) * bf.z;
    const float etaf = yf - bf.y;
    return fmaf(xif, xif, fmaf(etaf, etaf, ddf));
  }

  // FP32 estimate of T - base (pf = {vk, coef, vk*log2e, ...}); relative
  // error ~1e-4 on this lattice (coordinates carry 1e-9 m error), NaN when
  // the point sits on the beam (caller then takes the exact path).
  __device__ __forceinline__ float excess_estimate(const float4* bfp, const ti64_tempgen& g) const {
    const float4 bf = __ldg(bfp);
    float xif;
    const float sf = geom(bf, xif);
    const float rq = rsqrtf_approx(sf);
    const float rf = sf * rq;
    return g.pf[1] * rq * exp2f_approx(-g.pf[2] * (rf + xif));
  }

  // exact T at the step rows (bfp float row, b double row)
  template <class C = CoefBank>
  __device__ __forceinline__ double temp(const float4* bfp, const double* b,
                                         const ti64_tempgen& g, const C& cf = C()) const {
    {
      // no-op filter: vk (R + xi) > arg_noop  <=>  R > c := arg_noop/vk - xi
      const float4 bf = __ldg(bfp);
      float xif;
      const float sf = geom(bf, xif);
      const float c = g.pf[3] - xif;
      if (c <= 0.0f || sf > c * c) return g.p[4];
    }
    const double bx = __ldg(b), by = __ldg(b + 1), dir = __ldg(b + 2);
    const double xi = __dmul_rn(__dsub_rn(x, bx), dir);
    const double eta = __dsub_rn(y, by);
    const double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(xi, xi), __dmul_rn(eta, eta)), dd));
    const double arg = __dmul_rn(g.p[1], __dadd_rn(r, xi));  // >= 0
    double tt;
    if (arg > 708.0) {
      tt = g.base;  // fast_exp == 0 exactly; (coef/r)*0 == +0 (r > 0 here)
    } else {
      tt = __dadd_rn(g.base, __dmul_rn(div_rn(g.p[0], r), exp_core(-arg, cf)));
    }
    return tt > g.p[2] ? g.p[2] : tt;
  }
};

}  // namespace ti64
