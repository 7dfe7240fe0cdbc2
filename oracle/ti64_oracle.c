/*
 * ti64_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker and the CPU
 * baseline of bench.py).  Never linked into, loaded by or called from the
 * product path (paper_2402_17580_b200/); only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * A plain-C, literal restatement of the reference's explicit per-point
 * microstructure update, ti64micro (reference @ /root/reference/pkg/src/
 * ti64micro, numba/LLVM).  Every function cites the reference lines it
 * follows.  Bit parity with the reference is pinned by the tests/golden npz fixtures,
 * generated from the reference itself by tests/golden/make_golden.py and
 * checked in tests/test_oracle_golden.py.
 *
 * Arithmetic contract (reference Appendix A of SURVEY.md): one rounding per
 * + - * /, explicit fma() exactly where fastmath.py calls _fma, IEEE div and
 * sqrt, no contraction (build with -ffp-contract=off, never -ffast-math).
 *
 * The lane-batched structure of _range_body (batch.py:467-695) is kept:
 * lane arrays of width `lanes`, three-scenario branch dispatch, masked tail
 * batches, the two seeding passes and the per-batch seed write-back.  The
 * temperature generators and event counters are this project's own
 * definitions, restated here once for the checker.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/ti64_b200.h"

#if defined(__FAST_MATH__)
#error "the oracle must not be compiled with -ffast-math"
#endif

/* ------------------------------------------------------------------------ */
/* fastmath.py:53-107 tables and constants                                    */
/* ------------------------------------------------------------------------ */
static const double A_EXP[8] = {
    1.213071811889e-10,  3.068528102657e-1,  -2.40226342399359e-1,
    -5.55053313414954e-2, -9.6135243288483e-3, -1.34288475963084e-3,
    -1.43131744483589e-4, -2.1595656126349e-5};
static const double B_LN[12] = {
    1.84775672096293e-10, 1.44269504084132,     -0.721347520143005,
    0.480898345526187,    -0.360675000332004,   0.288048466919235,
    -0.235306287368882,   0.183102904829435,    -0.1209962689793,
    0.0591503811592113,   -0.0181149492489989,  0.00254488675605743};
static const double LOG2E = 1.4426950408889634;
static const double LN2 = 0.6931471805599453;
static const double SCALE = 4503599627370496.0; /* 2**52 */
static const double INV_SCALE = 1.0 / 4503599627370496.0;
static const double BIAS = 1023.0;
static const double ARG_MIN = -708.0;
static const double ARG_MAX = 709.0;
static const int64_t MANT_MASK = 0x000FFFFFFFFFFFFFLL;

static inline double i2f(int64_t i) { double d; memcpy(&d, &i, 8); return d; }
static inline int64_t f2i(double d) { int64_t i; memcpy(&i, &d, 8); return i; }
/* numpy's np.nan as a numba constant */
static inline double qnan(void) { return i2f(0x7FF8000000000000LL); }

/* fastmath.py:161-168 _k_exp (Estrin, explicit FMAs) */
static inline double k_exp(double y) {
  double y2 = y * y;
  double y4 = y2 * y2;
  double hi = fma(fma(A_EXP[7], y, A_EXP[6]), y2, fma(A_EXP[5], y, A_EXP[4]));
  double lo = fma(fma(A_EXP[3], y, A_EXP[2]), y2, fma(A_EXP[1], y, A_EXP[0]));
  return fma(hi, y4, lo);
}

/* fastmath.py:171-178 _k_ln */
static inline double k_ln(double m) {
  double m2 = m * m;
  double m4 = m2 * m2;
  double q0 = fma(fma(B_LN[3], m, B_LN[2]), m2, fma(B_LN[1], m, B_LN[0]));
  double q1 = fma(fma(B_LN[7], m, B_LN[6]), m2, fma(B_LN[5], m, B_LN[4]));
  double q2 = fma(fma(B_LN[11], m, B_LN[10]), m2, fma(B_LN[9], m, B_LN[8]));
  return fma(fma(q2, m4, q1), m4, q0);
}

/* fastmath.py:181-193 fast_exp_scalar */
double oracle_fast_exp1(double x) {
  int below = x < ARG_MIN;
  int above = x > ARG_MAX;
  int isn = x != x;
  double xs = (below || above || isn) ? 0.0 : x;
  double y = xs * LOG2E;
  double yf = y - floor(y);
  double z = i2f((int64_t)((y - k_exp(yf) + BIAS) * SCALE));
  z = below ? 0.0 : z;
  z = above ? DBL_MAX : z;
  return isn ? qnan() : z;
}

/* fastmath.py:196-206 fast_ln_scalar */
double oracle_fast_ln1(double x) {
  int bad = !(x > 0.0);
  double xs = bad ? 1.0 : x;
  xs = xs < DBL_MIN ? DBL_MIN : xs;
  int64_t bits = f2i(xs);
  double e = (double)(bits >> 52) - BIAS;
  double m = (double)(bits & MANT_MASK) * INV_SCALE;
  double z = LN2 * (e + k_ln(m));
  return bad ? qnan() : z;
}

/* fastmath.py:209-212 fast_pow_scalar */
double oracle_fast_pow1(double a, double x) {
  return oracle_fast_exp1(x * oracle_fast_ln1(a));
}

void oracle_fast_exp(const double* x, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = oracle_fast_exp1(x[i]);
}
void oracle_fast_ln(const double* x, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = oracle_fast_ln1(x[i]);
}
void oracle_fast_pow(const double* a, const double* x, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = oracle_fast_pow1(a[i], x[i]);
}

/* ------------------------------------------------------------------------ */
/* batch.py lane helpers                                                      */
/* ------------------------------------------------------------------------ */
#define XA_MAX 0.9
#define POW_FLOOR 1e-300
#define MAXL 8

/* batch.py:215-226 _lane_tfuncs */
static void lane_tfuncs(int L, const double* T, double* g, double* xsol,
                        double* xaeq, double* kas, const ti64_kparams* kp) {
  for (int j = 0; j < L; ++j) {
    double gg = (T[j] - kp->t_sol) / (kp->t_liq - kp->t_sol);
    gg = gg < 0.0 ? 0.0 : (gg > 1.0 ? 1.0 : gg);
    g[j] = gg;
    xsol[j] = 1.0 - gg;
    double ramp = 1.0 - oracle_fast_exp1(-kp->k_alpha_eq * (kp->t_as_start - T[j]));
    double ae = T[j] < kp->t_as_end ? XA_MAX : (T[j] > kp->t_as_start ? 0.0 : ramp);
    xaeq[j] = ae;
    kas[j] = kp->k1 / (1.0 + oracle_fast_exp1(-kp->k3 * (T[j] - kp->k2)));
  }
}

/* batch.py:229-236 _lane_tfuncs_rates */
static void lane_tfuncs_rates(int L, const double* T, double* xaeq, double* kas,
                              const ti64_kparams* kp) {
  for (int j = 0; j < L; ++j) {
    double ramp = 1.0 - oracle_fast_exp1(-kp->k_alpha_eq * (kp->t_as_start - T[j]));
    double ae = T[j] < kp->t_as_end ? XA_MAX : (T[j] > kp->t_as_start ? 0.0 : ramp);
    xaeq[j] = ae;
    kas[j] = kp->k1 / (1.0 + oracle_fast_exp1(-kp->k3 * (T[j] - kp->k2)));
  }
}

/* batch.py:239-244 _lane_xmeq_base */
static void lane_xmeq_base(int L, const double* T, double* out, const ti64_kparams* kp) {
  for (int j = 0; j < L; ++j) {
    double v = 1.0 - oracle_fast_exp1(-kp->k_alpha_m_eq * (kp->t_am_start - T[j]));
    out[j] = v < XA_MAX ? v : XA_MAX;
  }
}

/* batch.py:247-291 _lane_rates (three-scenario dispatch) */
static void lane_rates(int L, const double* xs, const double* xm, const double* xaeq,
                       const double* kas, double* ds, double* dm, double* pxs,
                       double* pa, double* pb, double* pc, double* pd,
                       const ti64_kparams* kp) {
  int n_grow = 0, n_am = 0, n_dis = 0;
  for (int j = 0; j < L; ++j) {
    double xa = xs[j] + xm[j];
    n_grow += ((xa < xaeq[j]) & (xs[j] > 0.0)) ? 1 : 0;
    n_am += ((xm[j] > 0.0) & (xs[j] > 0.0)) ? 1 : 0;
    n_dis += ((xa > xaeq[j]) & (xa < XA_MAX)) ? 1 : 0;
  }
  if (n_grow > 0 || n_am > 0)
    for (int j = 0; j < L; ++j) {
      double b = xs[j] > POW_FLOOR ? xs[j] : POW_FLOOR;
      pxs[j] = oracle_fast_pow1(b, kp->exp_as_lo);
    }
  if (n_grow > 0)
    for (int j = 0; j < L; ++j) {
      double d = xaeq[j] - (xs[j] + xm[j]);
      double b = d > POW_FLOOR ? d : POW_FLOOR;
      pa[j] = oracle_fast_pow1(b, kp->exp_as_hi);
    }
  if (n_am > 0)
    for (int j = 0; j < L; ++j) {
      double b = xm[j] > POW_FLOOR ? xm[j] : POW_FLOOR;
      pb[j] = oracle_fast_pow1(b, kp->exp_as_hi);
    }
  if (n_dis > 0)
    for (int j = 0; j < L; ++j) {
      double xa = xs[j] + xm[j];
      double b = XA_MAX - xa;
      b = b > POW_FLOOR ? b : POW_FLOOR;
      pc[j] = oracle_fast_pow1(b, kp->exp_b_lo);
      double d = xa - xaeq[j];
      b = d > POW_FLOOR ? d : POW_FLOOR;
      pd[j] = oracle_fast_pow1(b, kp->exp_b_hi);
    }
  for (int j = 0; j < L; ++j) {
    double xa = xs[j] + xm[j];
    double r1 = ((xa < xaeq[j]) & (xs[j] > 0.0)) ? kas[j] * pxs[j] * pa[j] : 0.0;
    double r2 = ((xm[j] > 0.0) & (xs[j] > 0.0)) ? kas[j] * pxs[j] * pb[j] : 0.0;
    double r3 = ((xa > xaeq[j]) & (xa < XA_MAX)) ? kp->f * kas[j] * pc[j] * pd[j] : 0.0;
    ds[j] = r1 + r2 - r3;
    dm[j] = -r2;
  }
}

/* batch.py:294-321 _lane_corrections */
static void lane_corrections(int L, const double* xs_in, const double* xm_in,
                             const double* T, const double* xaeq, const double* xsol,
                             const double* xmeqb, int any_form, int any_reg,
                             double* oxs, double* oxm, double* oxb,
                             const ti64_kparams* kp) {
  for (int j = 0; j < L; ++j) {
    double xs = xs_in[j] > 0.0 ? xs_in[j] : 0.0;
    double xm = xm_in[j] > 0.0 ? xm_in[j] : 0.0;
    if (any_reg) {
      double ramp = XA_MAX * (kp->t_as_start + kp->t_as_reg - T[j]) / kp->t_as_reg;
      ramp = ramp > 0.0 ? ramp : 0.0;
      double cap = ramp < xs ? ramp : xs;
      xs = T[j] > kp->t_as_start ? cap : xs;
    }
    double diss = xaeq[j] - xs;
    diss = diss > 0.0 ? diss : 0.0;
    xm = xs + xm > xaeq[j] ? diss : xm;
    if (any_form) {
      double xmeq = xmeqb[j] * (XA_MAX - xs) * (1.0 / XA_MAX);
      double grown = xmeq > xm ? xmeq : xm;
      xm = T[j] < kp->t_am_start ? grown : xm;
    }
    double xa = xs + xm;
    double sc = xa > XA_MAX ? XA_MAX / xa : 1.0;
    xs = xs * sc;
    xm = xm * sc;
    double xb = xsol[j] - xs - xm;
    oxs[j] = xs;
    oxm[j] = xm;
    oxb[j] = xb > 0.0 ? xb : 0.0;
  }
}

/* batch.py:324-354 _seed_advance */
static void seed_advance(int direction, double tracked, double xaeq, double kas,
                         double xsol, double dt, const ti64_kparams* kp,
                         double threshold, double* o_tr, int* o_act, double* o_xs,
                         double* o_xm, double* o_xb) {
  double delta, k, c;
  if (direction == TI64_SEED_BETA_TO_ALPHA_S) {
    delta = xaeq;
    k = kas;
    c = kp->c_alpha_s;
  } else {
    delta = XA_MAX - xaeq;
    k = kp->f * kas;
    c = kp->c_beta;
  }
  double xi = tracked / delta;
  xi = xi < 0.0 ? 0.0 : xi;
  xi = xi > 1.0 - 1e-12 ? 1.0 - 1e-12 : xi;
  double term = xi > 0.0 ? oracle_fast_pow1(xi / (1.0 - xi), 1.0 / c) : 0.0;
  double denom = delta * k * dt + c * term;
  double nt = delta / (1.0 + oracle_fast_pow1(c / denom, c));
  *o_act = !(nt * dt > threshold);
  *o_tr = nt;
  if (direction == TI64_SEED_BETA_TO_ALPHA_S) {
    *o_xs = nt;
    *o_xm = 0.0;
    *o_xb = xsol - nt;
  } else {
    *o_xs = XA_MAX - nt;
    *o_xm = 0.0;
    *o_xb = 0.1 + nt;
  }
}

/* batch.py:419-464 _seed_pass */
static int seed_pass(int L, double* lxs, double* lxm, double* lxb, double* ltr,
                     uint8_t* lac, uint8_t* ldr, const double* pt1, const double* g1,
                     const double* xsol1, const double* xaeq1, const double* kas1,
                     double* exs, double* exm, double* exb, double dt,
                     const ti64_icfg* cfg, const ti64_kparams* kp, int do_advance) {
  int n_seed = 0;
  double tol = cfg->stuck_tol;
  for (int j = 0; j < L; ++j) {
    double t1 = pt1[j];
    double xaeq = xaeq1[j];
    int melting = g1[j] > 0.0;
    if (lac[j] != 0) {
      if (ldr[j] == TI64_SEED_BETA_TO_ALPHA_S) {
        if (xaeq <= 0.0 || t1 < kp->t_am_start || melting) lac[j] = 0;
      } else {
        if (xaeq >= XA_MAX - 1e-12 || melting) lac[j] = 0;
      }
    } else {
      if (fabs(lxm[j]) <= tol && !melting) {
        if (fabs(lxs[j]) <= tol && fabs(lxb[j] - xsol1[j]) <= tol && xaeq > 0.0 &&
            t1 >= kp->t_am_start) {
          lac[j] = 1;
          ldr[j] = TI64_SEED_BETA_TO_ALPHA_S;
          ltr[j] = lxs[j] > 0.0 ? lxs[j] : 0.0;
        } else if (fabs(lxs[j] - XA_MAX) <= tol && fabs(lxb[j] - 0.1) <= tol &&
                   xaeq < XA_MAX - 1e-12) {
          lac[j] = 1;
          ldr[j] = TI64_SEED_ALPHA_S_TO_BETA;
          ltr[j] = lxb[j] > 0.1 ? lxb[j] - 0.1 : 0.0;
        }
      }
    }
    if (lac[j] != 0) {
      n_seed += 1;
      if (do_advance) {
        double tr, sxs, sxm, sxb;
        int act;
        seed_advance(ldr[j], ltr[j], xaeq1[j], kas1[j], xsol1[j], dt, kp,
                     cfg->initiation_threshold, &tr, &act, &sxs, &sxm, &sxb);
        ltr[j] = tr;
        lac[j] = act ? 1 : 0;
        exs[j] = sxs;
        exm[j] = sxm;
        exb[j] = sxb;
      }
    }
  }
  return n_seed;
}

/* batch.py:357-416 _cn_substep: Crank-Nicolson fixed point with per-lane
 * WRMS freeze; returns all-converged, writes the iteration count */
static int cn_substep(int L, const double* lxs, const double* lxm, const double* pt1,
                      const double* xsol1, const double* xaeq1, const double* kas1,
                      const double* xmeqb1, const double* dsn, const double* dmn, double* dsi,
                      double* dmi, double* dsx, double* dmx, double* cxs, double* cxm,
                      double* cxb, double* pxs, double* pa, double* pb, double* pc, double* pd,
                      double* exs, double* exm, double* exb, double* sxs, double* sxm,
                      double* sxb, uint8_t* conv, double* itc, double dt,
                      const ti64_icfg* cfg, const ti64_kparams* kp, int* iters_out) {
  int any_form = 0, any_reg = 0;
  for (int j = 0; j < L; ++j) {
    any_form += pt1[j] < kp->t_am_start;
    any_reg += pt1[j] > kp->t_as_start;
    conv[j] = 0;
  }
  lane_corrections(L, lxs, lxm, pt1, xaeq1, xsol1, xmeqb1, any_form > 0, any_reg > 0, cxs, cxm,
                   cxb, kp);
  lane_rates(L, cxs, cxm, xaeq1, kas1, dsi, dmi, pxs, pa, pb, pc, pd, kp);
  double half = 0.5 * dt;
  int iters = 0;
  for (;;) {
    for (int j = 0; j < L; ++j) {
      exs[j] = lxs[j] + half * (dsi[j] + dsn[j]);
      exm[j] = lxm[j] + half * (dmi[j] + dmn[j]);
    }
    lane_corrections(L, exs, exm, pt1, xaeq1, xsol1, xmeqb1, any_form > 0, any_reg > 0, cxs,
                     cxm, cxb, kp);
    lane_rates(L, cxs, cxm, xaeq1, kas1, dsx, dmx, pxs, pa, pb, pc, pd, kp);
    iters += 1;
    int n_open = 0;
    for (int j = 0; j < L; ++j) {
      if (conv[j] == 0) {
        double rs = half * (dsx[j] - dsi[j]);
        double rm = half * (dmx[j] - dmi[j]);
        double ws = 1.0 / (cfg->eps_abs + fabs(cxs[j]) * cfg->eps_rel);
        double wm = 1.0 / (cfg->eps_abs + fabs(cxm[j]) * cfg->eps_rel);
        double e = 0.5 * ((rs * ws) * (rs * ws) + (rm * wm) * (rm * wm));
        sxs[j] = cxs[j];
        sxm[j] = cxm[j];
        sxb[j] = cxb[j];
        dsi[j] = dsx[j];
        dmi[j] = dmx[j];
        itc[j] += 1.0;
        if (e < 1.0)
          conv[j] = 1;
        else
          n_open += 1;
      }
    }
    if (n_open == 0 || iters >= cfg->max_fixed_point_iters) {
      for (int j = 0; j < L; ++j) {
        exs[j] = sxs[j];
        exm[j] = sxm[j];
        exb[j] = sxb[j];
      }
      *iters_out = iters;
      return n_open == 0;
    }
  }
}

/* batch.py:467-695 _range_body, both schemes (explicit: pieces stay 1 since
 * the explicit step never fails; implicit: halving retries with state
 * rollback, batch.py:568-674).  iters_out (may be NULL) receives the
 * per-point implicit iteration counts when record_iters. */
int64_t oracle_run_range2(const ti64_fields* f, int64_t start, int64_t stop, int64_t lanes,
                          int64_t nsub, double dt_sub, const ti64_kparams* kp,
                          const ti64_icfg* cfg, int32_t record_iters, int64_t* iters_out) {
  if (lanes < 1 || lanes > MAXL) return TI64_EINVAL;
  const int explicit_ = cfg->scheme == TI64_SCHEME_EXPLICIT;
  const int L = (int)lanes;
  double lxs[MAXL], lxm[MAXL], lxb[MAXL], lt0[MAXL], lt1[MAXL], st0[MAXL], st1[MAXL];
  double pt0[MAXL], pt1[MAXL];
  double g1[MAXL], xsol1[MAXL], xaeq1[MAXL], kas1[MAXL], xmeqb1[MAXL];
  double xaeq0[MAXL], kas0[MAXL], ltr[MAXL], dsn[MAXL], dmn[MAXL];
  double dsi[MAXL], dmi[MAXL], dsx[MAXL], dmx[MAXL], cxs[MAXL], cxm[MAXL], cxb[MAXL];
  double pxs[MAXL] = {0}, pa[MAXL] = {0}, pb[MAXL] = {0}, pc[MAXL] = {0}, pd[MAXL] = {0};
  double exs[MAXL], exm[MAXL], exb[MAXL], sxs[MAXL], sxm[MAXL], sxb[MAXL], itc[MAXL];
  double bxs[MAXL], bxm[MAXL], bxb[MAXL], btr[MAXL];
  uint8_t lac[MAXL], ldr[MAXL], bac[MAXL], bdr[MAXL], conv[MAXL];
  memset(xmeqb1, 0, sizeof xmeqb1);
  memset(xaeq1, 0, sizeof xaeq1);
  memset(kas1, 0, sizeof kas1);
  memset(sxs, 0, sizeof sxs);
  memset(sxm, 0, sizeof sxm);
  memset(sxb, 0, sizeof sxb);
  const double inv_nsub = 1.0 / (double)nsub;
  const double stuck_tol = cfg->stuck_tol;
  for (int64_t base = start; base < stop; base += lanes) {
    int64_t w = stop - base;
    w = w > lanes ? lanes : w;
    int n_seed_in = 0;
    for (int j = 0; j < L; ++j) {
      int64_t i = j < w ? base + j : base;
      lxs[j] = f->x_alpha_s[i];
      lxm[j] = f->x_alpha_m[i];
      lxb[j] = f->x_beta[i];
      lt0[j] = f->temperature_old[i];
      lt1[j] = f->temperature_new[i];
      uint8_t ac = f->seed_active[i];
      n_seed_in += ac != 0;
      lac[j] = ac;
      ldr[j] = ac != 0 ? f->seed_direction[i] : 0;
      ltr[j] = ac != 0 ? f->seed_tracked[i] : 0.0;
      if (!explicit_) itc[j] = 0.0;
    }
    int seed_out = n_seed_in > 0;
    int failed = 0;
    for (int64_t k = 0; k < nsub; ++k) {
      int last_sub = k == nsub - 1;
      const double *s0v, *s1v;
      if (nsub == 1) {
        s0v = lt0;
        s1v = lt1;
      } else {
        double f0 = (double)k * inv_nsub;
        double f1 = (double)(k + 1) * inv_nsub;
        for (int j = 0; j < L; ++j) {
          double d = lt1[j] - lt0[j];
          st0[j] = lt0[j] + d * f0;
          st1[j] = last_sub ? lt1[j] : lt0[j] + d * f1;
        }
        s0v = st0;
        s1v = st1;
      }
      if (!explicit_)
        for (int j = 0; j < L; ++j) {
          bxs[j] = lxs[j];
          bxm[j] = lxm[j];
          bxb[j] = lxb[j];
          btr[j] = ltr[j];
          bac[j] = lac[j];
          bdr[j] = ldr[j];
        }
      int halv = 0;
      for (;;) {
        int64_t pieces = (int64_t)1 << halv;
        double inv_p = 1.0 / (double)pieces;
        int ok = 1;
        for (int64_t p = 0; p < pieces; ++p) {
          const double *p0v, *p1v;
          if (pieces == 1) {
            p0v = s0v;
            p1v = s1v;
          } else {
            double pf0 = (double)p * inv_p;
            double pf1 = (double)(p + 1) * inv_p;
            int last_p = p == pieces - 1;
            for (int j = 0; j < L; ++j) {
              double dts = s1v[j] - s0v[j];
              pt0[j] = s0v[j] + dts * pf0;
              pt1[j] = last_p ? s1v[j] : s0v[j] + dts * pf1;
            }
            p0v = pt0;
            p1v = pt1;
          }
          if (k == 0 && p == 0) {
            lane_tfuncs_rates(L, p0v, xaeq0, kas0, kp);
          } else if (halv == 0 || p > 0) {
            for (int j = 0; j < L; ++j) {
              xaeq0[j] = xaeq1[j];
              kas0[j] = kas1[j];
            }
          } else {
            lane_tfuncs_rates(L, p0v, xaeq0, kas0, kp);
          }
          lane_tfuncs(L, p1v, g1, xsol1, xaeq1, kas1, kp);
          int n_form = 0, n_reg = 0, n_watch = 0;
          for (int j = 0; j < L; ++j) {
            n_form += p1v[j] < kp->t_am_start;
            n_reg += p1v[j] > kp->t_as_start;
            int watch = (lac[j] != 0) |
                        ((fabs(lxm[j]) <= stuck_tol) &
                         ((fabs(lxs[j]) <= stuck_tol) | (fabs(lxs[j] - XA_MAX) <= stuck_tol)));
            n_watch += watch;
          }
          if (n_form > 0) lane_xmeq_base(L, p1v, xmeqb1, kp);
          int n_seed = 0;
          if (n_watch > 0)
            n_seed = seed_pass(L, lxs, lxm, lxb, ltr, lac, ldr, p1v, g1, xsol1, xaeq1, kas1,
                               exs, exm, exb, 0.0, cfg, kp, 0);
          double dt_p = dt_sub * inv_p;
          int its = 0;
          if (n_seed < L) {
            lane_rates(L, lxs, lxm, xaeq0, kas0, dsn, dmn, pxs, pa, pb, pc, pd, kp);
            if (explicit_) {
              for (int j = 0; j < L; ++j) {
                exs[j] = lxs[j] + dt_p * dsn[j];
                exm[j] = lxm[j] + dt_p * dmn[j];
              }
              lane_corrections(L, exs, exm, p1v, xaeq1, xsol1, xmeqb1, n_form > 0, n_reg > 0,
                               exs, exm, exb, kp);
            } else {
              ok = cn_substep(L, lxs, lxm, p1v, xsol1, xaeq1, kas1, xmeqb1, dsn, dmn, dsi, dmi,
                              dsx, dmx, cxs, cxm, cxb, pxs, pa, pb, pc, pd, exs, exm, exb, sxs,
                              sxm, sxb, conv, itc, dt_p, cfg, kp, &its);
            }
          }
          if (n_seed > 0) {
            seed_pass(L, lxs, lxm, lxb, ltr, lac, ldr, p1v, g1, xsol1, xaeq1, kas1, exs, exm,
                      exb, dt_p, cfg, kp, 1);
            seed_out = 1;
          }
          for (int j = 0; j < L; ++j) {
            lxs[j] = exs[j];
            lxm[j] = exm[j];
            lxb[j] = exb[j];
          }
          if (!ok) break;
        }
        if (ok) break;
        halv += 1;
        if (halv > cfg->max_halvings) {
          failed = 1;
          break;
        }
        for (int j = 0; j < L; ++j) {
          lxs[j] = bxs[j];
          lxm[j] = bxm[j];
          lxb[j] = bxb[j];
          ltr[j] = btr[j];
          lac[j] = bac[j];
          ldr[j] = bdr[j];
        }
      }
      if (failed) break;
    }
    for (int64_t j = 0; j < w; ++j) {
      int64_t i = base + j;
      f->x_alpha_s[i] = lxs[j];
      f->x_alpha_m[i] = lxm[j];
      f->x_beta[i] = lxb[j];
      f->temperature_old[i] = lt1[j];
    }
    if (record_iters && !explicit_ && iters_out)
      for (int64_t j = 0; j < w; ++j) iters_out[base + j] = (int64_t)itc[j];
    if (seed_out)
      for (int64_t j = 0; j < w; ++j) {
        int64_t i = base + j;
        f->seed_tracked[i] = ltr[j];
        f->seed_active[i] = lac[j];
        f->seed_direction[i] = ldr[j];
      }
    if (failed) return base + 1;
  }
  return 0;
}

/* explicit-scheme entry kept for the existing callers */
int64_t oracle_run_range(const ti64_fields* f, int64_t start, int64_t stop,
                         int64_t lanes, int64_t nsub, double dt_sub,
                         const ti64_kparams* kp, const ti64_icfg* cfg) {
  return oracle_run_range2(f, start, stop, lanes, nsub, dt_sub, kp, cfg, 0, NULL);
}

/* batch.py:750-755 _num_substeps */
int64_t oracle_num_substeps(double dt, double dt_sub_max) {
  if (dt <= dt_sub_max * (1.0 + 1e-9)) return 1;
  return (int64_t)ceil(dt / dt_sub_max - 1e-12);
}

/* step_all's threaded split (batch.py:784-796): lane-aligned chunks, so the
 * lane batches are the same as the single-threaded sweep. */
int64_t oracle_step_all(const ti64_fields* f, int64_t n, int64_t lanes,
                        int64_t nsub, double dt_sub, const ti64_kparams* kp,
                        const ti64_icfg* cfg, int32_t threads) {
  if (threads <= 1 || n <= 4 * lanes) return oracle_run_range(f, 0, n, lanes, nsub, dt_sub, kp, cfg);
  int64_t nchunks = (int64_t)threads * 8;
  int64_t nb = (n + lanes - 1) / lanes;
  if (nchunks > nb) nchunks = nb;
  int64_t rc_all = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) reduction(max : rc_all)
#endif
  for (int64_t c = 0; c < nchunks; ++c) {
    int64_t b0 = (nb * c) / nchunks * lanes;
    int64_t b1 = (nb * (c + 1)) / nchunks * lanes;
    if (b1 > n) b1 = n;
    int64_t rc = oracle_run_range(f, b0, b1, lanes, nsub, dt_sub, kp, cfg);
    if (rc > rc_all) rc_all = rc;
  }
  return rc_all;
}

/* ------------------------------------------------------------------------ */
/* Seeded temperature generators (not in the reference)        */
/* ------------------------------------------------------------------------ */
static inline uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
static inline double u01(uint64_t seed, uint64_t point, uint64_t k) {
  uint64_t b = splitmix(splitmix(seed ^ splitmix(point)) ^ (k * 0xD1B54A32D192ED03ULL));
  return (double)(b >> 11) * 0x1.0p-53;
}
static inline double unif(double lo, double hi, double u) { return lo + (hi - lo) * u; }

double oracle_u01(uint64_t seed, uint64_t point, uint64_t k) { return u01(seed, point, k); }

/* Gaussian pulse a * exp(-((t - tc) * inv_w)^2) with the fast exp */
static inline double pulse(double a, double tc, double inv_w, double t) {
  double u = (t - tc) * inv_w;
  return a * oracle_fast_exp1(-(u * u));
}

/* One point's generator with its seeded parameters drawn once (the per-step
 * arithmetic is the definition; drawing once only saves the hashes). */
#define PG_MAXP 64
typedef struct {
  int np;
  double a[PG_MAXP], tc[PG_MAXP], inv_w[PG_MAXP];
  double x, y, dd;
} pointgen;

static void pointgen_init(const ti64_tempgen* g, uint64_t pt, pointgen* q) {
  const double* p = g->p;
  q->np = 0;
  switch (g->kind) {
    case TI64_SRC_PULSE: {
      double a = unif(p[0], p[1], u01(g->seed, pt, 0));
      double tc = unif(p[2], p[3], u01(g->seed, pt, 1));
      double w = unif(p[4], p[5], u01(g->seed, pt, 2));
      q->np = 1;
      q->a[0] = a;
      q->tc[0] = tc;
      q->inv_w[0] = 1.0 / w;
      break;
    }
    case TI64_SRC_ROSENTHAL: {
      int64_t i = (int64_t)pt % g->nx;
      int64_t j = ((int64_t)pt / g->nx) % g->ny;
      int64_t k = (int64_t)pt / (g->nx * g->ny);
      double d = (double)k * g->h;
      q->x = (double)i * g->h;
      q->y = (double)j * g->h;
      q->dd = d * d;
      break;
    }
    case TI64_SRC_PULSE_TRAIN: {
      double a1 = unif(p[0], p[1], u01(g->seed, pt, 0));
      double scale = 1.0;
      int np_ = g->max_pulses < PG_MAXP ? g->max_pulses : PG_MAXP;
      for (int kk = 0; kk < np_; ++kk) {
        q->a[kk] = a1 * scale * unif(p[2], p[3], u01(g->seed, pt, 1 + 3 * kk));
        q->tc[kk] = p[4] + p[5] * (double)kk + unif(p[6], p[7], u01(g->seed, pt, 2 + 3 * kk));
        q->inv_w[kk] = 1.0 / unif(p[8], p[9], u01(g->seed, pt, 3 + 3 * kk));
        scale = scale * p[10];
      }
      q->np = np_;
      break;
    }
    case TI64_SRC_PULSE_SWEEP: {
      int np_ = 1 + (int)(u01(g->seed, pt, 0) * (double)g->max_pulses);
      if (np_ > PG_MAXP) np_ = PG_MAXP;
      for (int kk = 0; kk < np_; ++kk) {
        q->a[kk] = unif(p[0], p[1], u01(g->seed, pt, 1 + 3 * kk));
        q->tc[kk] = unif(p[2], p[3], u01(g->seed, pt, 2 + 3 * kk));
        q->inv_w[kk] = 1.0 / oracle_fast_exp1(unif(p[4], p[5], u01(g->seed, pt, 3 + 3 * kk)));
      }
      q->np = np_;
      break;
    }
    default:
      break;
  }
}

/* T at time step `step` (t = step * dt): base + the pulses in order k = 1..K,
 * or the capped Rosenthal term */
static double pointgen_temp(const ti64_tempgen* g, const pointgen* q, int64_t step) {
  const double t = (double)step * g->dt;
  const double* p = g->p;
  if (g->kind == TI64_SRC_ROSENTHAL) {
    const double* b = g->beam_d + 3 * step;
    double xi = (q->x - b[0]) * b[2];
    double eta = q->y - b[1];
    double r = sqrt(xi * xi + eta * eta + q->dd);
    double tt = g->base + p[0] / r * oracle_fast_exp1(-(p[1] * (r + xi)));
    return tt > p[2] ? p[2] : tt;
  }
  if (g->kind < TI64_SRC_PULSE || g->kind > TI64_SRC_PULSE_SWEEP) return qnan();
  double s = g->base;
  for (int kk = 0; kk < q->np; ++kk) s = s + pulse(q->a[kk], q->tc[kk], q->inv_w[kk], t);
  return s;
}

double oracle_gen_temperature1(const ti64_tempgen* g, int64_t local, int64_t step) {
  pointgen q;
  pointgen_init(g, (uint64_t)(g->point_offset + local), &q);
  return pointgen_temp(g, &q, step);
}

/* T at steps step0 .. step0+nsteps-1 of the points with GLOBAL indices
 * pts[0..m): out is (nsteps, m) row-major (the CPU legs' inputs, generated
 * outside their timed regions). */
void oracle_gen_temperature_points(const ti64_tempgen* g, const int64_t* pts, int64_t m,
                                   int64_t step0, int64_t nsteps, double* out,
                                   int32_t threads) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
#endif
  for (int64_t j = 0; j < m; ++j) {
    pointgen q;
    pointgen_init(g, (uint64_t)pts[j], &q);
    for (int64_t s = 0; s < nsteps; ++s) out[s * m + j] = pointgen_temp(g, &q, step0 + s);
  }
}

void oracle_gen_temperature(const ti64_tempgen* g, int64_t n, int64_t step, double* out,
                            int32_t threads) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
#endif
  for (int64_t i = 0; i < n; ++i) out[i] = oracle_gen_temperature1(g, i, step);
}

void oracle_gen_initial_state(const ti64_tempgen* g, int64_t n, const ti64_fields* f) {
  for (int64_t i = 0; i < n; ++i) {
    double xs = 0.9, xb = 0.1;
    if (g->kind == TI64_SRC_PULSE_TRAIN) {
      uint64_t pt = (uint64_t)(g->point_offset + i);
      xs = unif(g->p[11], g->p[12], u01(g->seed, pt, 63));
      xb = 1.0 - xs;
    }
    f->x_alpha_s[i] = xs;
    f->x_alpha_m[i] = 0.0;
    f->x_beta[i] = xb;
    f->seed_tracked[i] = 0.0;
    f->seed_active[i] = 0;
    f->seed_direction[i] = 0;
  }
}

/* ------------------------------------------------------------------------ */
/* Advance loop with event counters (definitions: DESIGN.md §3)              */
/* ------------------------------------------------------------------------ */
static inline int argmax3(double a, double b, double c) {
  return (a >= b && a >= c) ? 0 : (b >= c ? 1 : 2);
}

/* x_alpha_eq at T, batch.py:223-224 arithmetic */
static inline double xaeq_of(double T, const ti64_kparams* kp) {
  double ramp = 1.0 - oracle_fast_exp1(-kp->k_alpha_eq * (kp->t_as_start - T));
  return T < kp->t_as_end ? XA_MAX : (T > kp->t_as_start ? 0.0 : ramp);
}

/* Reference loop: temperature_new <- T(s+1); step_all (run_range over all
 * points, lane batches of `lanes`).  Counters per DESIGN.md §3; totals:
 * {updates, form, grow|am, grow, am, dissolve, martensite, switches}.
 * sums[snap][3] at every snapshot_every steps (and the end). */
int64_t oracle_advance(const ti64_fields* f, int64_t n, const ti64_tempgen* g,
                       int64_t step0, int64_t nsteps, int64_t nsub, int64_t lanes,
                       int64_t snapshot_every, const ti64_kparams* kp,
                       const ti64_icfg* cfg, uint32_t* mart, uint32_t* sw,
                       uint64_t* totals, double* sums, int32_t threads) {
  double* xm_prev = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int* am_prev = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  int64_t snap = 0;
  double dt = g->dt;
  for (int64_t s = 0; s < nsteps; ++s) {
    int64_t step = step0 + s;
    oracle_gen_temperature(g, n, step + 1, f->temperature_new, threads);
    uint64_t c_form = 0, c_ga = 0, c_g = 0, c_a = 0, c_d = 0;
    for (int64_t i = 0; i < n; ++i) {
      double xs = f->x_alpha_s[i], xm = f->x_alpha_m[i];
      double xa = xs + xm;
      double xe0 = xaeq_of(f->temperature_old[i], kp);
      int grow = (xa < xe0) & (xs > 0.0);
      int am = (xm > 0.0) & (xs > 0.0);
      int dis = (xa > xe0) & (xa < XA_MAX);
      c_form += f->temperature_new[i] < kp->t_am_start;
      c_ga += grow | am;
      c_g += grow;
      c_a += am;
      c_d += dis;
      xm_prev[i] = xm;
      am_prev[i] = argmax3(xs, xm, f->x_beta[i]);
    }
    int64_t rc = oracle_step_all(f, n, lanes, nsub, dt / (double)nsub, kp, cfg, threads);
    if (rc != 0) {
      free(xm_prev);
      free(am_prev);
      return rc;
    }
    uint64_t c_m = 0, c_s = 0;
    for (int64_t i = 0; i < n; ++i) {
      int m = f->x_alpha_m[i] > xm_prev[i];
      int w = argmax3(f->x_alpha_s[i], f->x_alpha_m[i], f->x_beta[i]) != am_prev[i];
      if (mart) mart[i] += (uint32_t)m;
      if (sw) sw[i] += (uint32_t)w;
      c_m += m;
      c_s += w;
    }
    if (totals) {
      totals[0] += (uint64_t)n;
      totals[1] += c_form;
      totals[2] += c_ga;
      totals[3] += c_g;
      totals[4] += c_a;
      totals[5] += c_d;
      totals[6] += c_m;
      totals[7] += c_s;
    }
    int at_snap = (snapshot_every > 0 && (s + 1) % snapshot_every == 0) || s + 1 == nsteps;
    if (at_snap && sums) {
      double a = 0.0, b = 0.0, c = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        a += f->x_alpha_s[i];
        b += f->x_alpha_m[i];
        c += f->x_beta[i];
      }
      sums[3 * snap + 0] = a;
      sums[3 * snap + 1] = b;
      sums[3 * snap + 2] = c;
    }
    if (at_snap) ++snap;
  }
  free(xm_prev);
  free(am_prev);
  return 0;
}

/* The reference loop of oracle_advance for a SUBSET of points given by their
 * GLOBAL indices pts[0..m) (e.g. every 1024th point of a config).  Points are
 * independent: consecutive subset points are grouped into lane batches of 8
 * (the reference's default width) and each group runs the whole loop alone;
 * explicit-scheme states are lane-width and batch-composition invariant
 * (test_batch.py:79-85), while the seed arrays of INACTIVE points are
 * batch-dependent residue (batch.py:687-692) and are not compared.
 * f holds the m points' state (in/out); counters as oracle_advance
 * (per-point mart/sw may be NULL; totals[8] may be NULL). */
#define AP_LANES 8
int64_t oracle_advance_points(const ti64_fields* f, const int64_t* pts, int64_t m,
                              const ti64_tempgen* g, int64_t step0, int64_t nsteps,
                              int64_t nsub, const ti64_kparams* kp, const ti64_icfg* cfg,
                              uint32_t* mart, uint32_t* sw, uint64_t* totals,
                              int32_t threads) {
  int64_t rc_all = 0;
  uint64_t t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0, t5 = 0, t6 = 0, t7 = 0;
  const double dt_sub = g->dt / (double)nsub;
  const int64_t ngroups = (m + AP_LANES - 1) / AP_LANES;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads > 0 ? threads : 1) \
    reduction(max : rc_all) reduction(+ : t0, t1, t2, t3, t4, t5, t6, t7)
#endif
  for (int64_t gi = 0; gi < ngroups; ++gi) {
    const int64_t j0 = gi * AP_LANES;
    const int w = (int)(m - j0 < AP_LANES ? m - j0 : AP_LANES);
    pointgen q[AP_LANES];
    double xs[AP_LANES], xm[AP_LANES], xb[AP_LANES], to[AP_LANES], tn[AP_LANES], tr[AP_LANES];
    uint8_t ac[AP_LANES], dr[AP_LANES];
    uint32_t mc[AP_LANES] = {0}, sc[AP_LANES] = {0};
    for (int l = 0; l < w; ++l) {
      const int64_t j = j0 + l;
      pointgen_init(g, (uint64_t)pts[j], &q[l]);
      xs[l] = f->x_alpha_s[j];
      xm[l] = f->x_alpha_m[j];
      xb[l] = f->x_beta[j];
      to[l] = f->temperature_old[j];
      tn[l] = f->temperature_new[j];
      tr[l] = f->seed_tracked[j];
      ac[l] = f->seed_active[j];
      dr[l] = f->seed_direction[j];
    }
    ti64_fields fg = {xs, xm, xb, to, tn, tr, ac, dr};
    int failed = 0;
    for (int64_t s = 0; s < nsteps && !failed; ++s) {
      double xm_prev[AP_LANES];
      int am_prev[AP_LANES];
      for (int l = 0; l < w; ++l) {
        tn[l] = pointgen_temp(g, &q[l], step0 + s + 1);
        const double xa = xs[l] + xm[l];
        const double xe0 = xaeq_of(to[l], kp);
        const int grow = (xa < xe0) & (xs[l] > 0.0);
        const int am = (xm[l] > 0.0) & (xs[l] > 0.0);
        const int dis = (xa > xe0) & (xa < XA_MAX);
        t1 += tn[l] < kp->t_am_start;
        t2 += grow | am;
        t3 += grow;
        t4 += am;
        t5 += dis;
        xm_prev[l] = xm[l];
        am_prev[l] = argmax3(xs[l], xm[l], xb[l]);
      }
      const int64_t rc = oracle_run_range(&fg, 0, w, AP_LANES, nsub, dt_sub, kp, cfg);
      if (rc != 0) {
        if (rc_all < j0 + rc) rc_all = j0 + rc;
        failed = 1;
      }
      for (int l = 0; l < w; ++l) {
        mc[l] += xm[l] > xm_prev[l];
        sc[l] += argmax3(xs[l], xm[l], xb[l]) != am_prev[l];
      }
    }
    for (int l = 0; l < w; ++l) {
      const int64_t j = j0 + l;
      f->x_alpha_s[j] = xs[l];
      f->x_alpha_m[j] = xm[l];
      f->x_beta[j] = xb[l];
      f->temperature_old[j] = to[l];
      f->temperature_new[j] = tn[l];
      f->seed_tracked[j] = tr[l];
      f->seed_active[j] = ac[l];
      f->seed_direction[j] = dr[l];
      if (mart) mart[j] += mc[l];
      if (sw) sw[j] += sc[l];
      t6 += mc[l];
      t7 += sc[l];
    }
    t0 += (uint64_t)nsteps * (uint64_t)w;
  }
  if (totals) {
    totals[0] += t0;
    totals[1] += t1;
    totals[2] += t2;
    totals[3] += t3;
    totals[4] += t4;
    totals[5] += t5;
    totals[6] += t6;
    totals[7] += t7;
  }
  return rc_all;
}

/* integrator.py:328-361 _history_kernel for one point (times strictly
 * increasing, checked by the caller); out is (n_samples, 3). */
int64_t oracle_history(const double* times, const double* temps, int64_t ns,
                       double xs0, double xm0, double xb0, const ti64_kparams* kp,
                       const ti64_icfg* cfg, double* out) {
  double xs = xs0, xm = xm0, xb = xb0, t0 = temps[0], t1 = 0.0, tr = 0.0;
  uint8_t ac = 0, dr = 0;
  ti64_fields f = {&xs, &xm, &xb, &t0, &t1, &tr, &ac, &dr};
  out[0] = xs0;
  out[1] = xm0;
  out[2] = xb0;
  for (int64_t k = 1; k < ns; ++k) {
    double dt = times[k] - times[k - 1];
    t1 = temps[k];
    int64_t nsub = oracle_num_substeps(dt, cfg->dt_sub_max);
    int64_t rc = oracle_run_range(&f, 0, 1, 1, nsub, dt / (double)nsub, kp, cfg);
    if (rc != 0) {
      for (int64_t q = k; q < ns; ++q) out[3 * q] = out[3 * q + 1] = out[3 * q + 2] = qnan();
      return rc;
    }
    out[3 * k + 0] = xs;
    out[3 * k + 1] = xm;
    out[3 * k + 2] = xb;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* thermal.py:205-287 _stencil_step, literal                                  */
/* ------------------------------------------------------------------------ */
#define STATE_INACTIVE 0
#define STATE_POWDER 1

/* Arrays hold global planes [z_base, z_base + nz_stored) (the whole grid
 * when z_base = 0, nz_stored = nz); planes [z_begin, z_end) are updated.
 * The slab form exists so tests can check the z-slab decomposition of the
 * multi-GPU driver against the whole-grid reference. */
void oracle_stencil_step(const double* src, double* dst, double* rc,
                         const uint8_t* state, const ti64_thermal* tp,
                         const ti64_stencil_args* a) {
  const int64_t nz = a->nz, ny = a->ny, nx = a->nx;
  const int64_t zb = a->z_base;
#define IDX(z, y, x) ((((z) - zb) * ny + (y)) * nx + (x))
  double inv_rch2 = a->dt / (tp->rho_c * a->h * a->h);
  double inv_rch = a->dt / (tp->rho_c * a->h);
  double inv_rc = a->dt / tp->rho_c;
  double dk = tp->k_ms - tp->k_p;
  double t4inf = pow(tp->t_inf, 4.0);
  /* every cell writes only its own dst entry: planes run in parallel (the
   * reference's serial loop order does not affect any result) */
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int64_t z = a->z_begin; z < a->z_end; ++z)
    for (int64_t y = 0; y < ny; ++y)
      for (int64_t x = 0; x < nx; ++x) {
        if (state[IDX(z, y, x)] == STATE_INACTIVE) continue;
        double t0 = src[IDX(z, y, x)];
        double g0 = (t0 - tp->t_sol) / (tp->t_liq - tp->t_sol);
        g0 = g0 < 0.0 ? 0.0 : (g0 > 1.0 ? 1.0 : g0);
        double rc0 = rc[IDX(z, y, x)];
        rc0 = rc0 > g0 ? rc0 : g0;
        double k0 = tp->k_p + rc0 * dk;
        double flux = 0.0;
        for (int face = 0; face < 6; ++face) {
          int64_t zz = z, yy = y, xx = x;
          switch (face) {
            case 0: xx = x - 1; break;
            case 1: xx = x + 1; break;
            case 2: yy = y - 1; break;
            case 3: yy = y + 1; break;
            case 4: zz = z - 1; break;
            default: zz = z + 1; break;
          }
          if (xx < 0 || xx >= nx || yy < 0 || yy >= ny || zz < 0 || zz >= nz) continue;
          if (state[IDX(zz, yy, xx)] == STATE_INACTIVE) continue;
          double t1 = src[IDX(zz, yy, xx)];
          double g1 = (t1 - tp->t_sol) / (tp->t_liq - tp->t_sol);
          g1 = g1 < 0.0 ? 0.0 : (g1 > 1.0 ? 1.0 : g1);
          double rc1 = rc[IDX(zz, yy, xx)];
          rc1 = rc1 > g1 ? rc1 : g1;
          double k1 = tp->k_p + rc1 * dk;
          double kf = 2.0 * k0 * k1 / (k0 + k1);
          flux += kf * (t1 - t0);
        }
        double t_new = t0 + inv_rch2 * flux;
        if (a->source_on != 0 && z == a->z_top - 1) {
          double xc = ((double)x + 0.5) * a->h;
          double yc = ((double)y + 0.5) * a->h;
          double r2 = (xc - a->beam_x) * (xc - a->beam_x) + (yc - a->beam_y) * (yc - a->beam_y);
          double arg = -2.0 * r2 * a->src_r2inv;
          if (arg > -40.0) t_new += inv_rc * a->src_peak * oracle_fast_exp1(arg);
        }
        if (a->losses_on != 0) {
          int exposed = z == nz - 1 || state[IDX(z + 1, y, x)] == STATE_INACTIVE;
          if (exposed) {
            double q = tp->emissivity * tp->sigma_s * (t0 * t0 * t0 * t0 - t4inf);
            double tc = t0 < tp->t_max_clamp ? t0 : tp->t_max_clamp;
            if (tc > tp->t_v)
              q += 0.82 * tp->c_p * oracle_fast_exp1(-tp->c_t * (1.0 / tc - 1.0 / tp->t_v)) *
                   sqrt(tp->c_m / tc) * (tp->h_v + tp->c_heat * (tc - tp->t_h0));
            t_new -= inv_rch * q;
          }
        }
        dst[IDX(z, y, x)] = t_new;
      }
  if (a->bc_bottom_on != 0 && a->z_begin == 0 && a->z_end > 0)
    for (int64_t y = 0; y < ny; ++y)
      for (int64_t x = 0; x < nx; ++x)
        if (state[IDX(0, y, x)] != STATE_INACTIVE) dst[IDX(0, y, x)] = a->bc_bottom;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int64_t z = a->z_begin; z < a->z_end; ++z)
    for (int64_t y = 0; y < ny; ++y)
      for (int64_t x = 0; x < nx; ++x)
        if (state[IDX(z, y, x)] == STATE_POWDER) {
          double g1 = (dst[IDX(z, y, x)] - tp->t_sol) / (tp->t_liq - tp->t_sol);
          g1 = g1 < 0.0 ? 0.0 : (g1 > 1.0 ? 1.0 : g1);
          if (g1 > rc[IDX(z, y, x)]) rc[IDX(z, y, x)] = g1;
        }
#undef IDX
}

int32_t oracle_max_threads(void) {
#ifdef _OPENMP
  return (int32_t)omp_get_max_threads();
#else
  return 1;
#endif
}
