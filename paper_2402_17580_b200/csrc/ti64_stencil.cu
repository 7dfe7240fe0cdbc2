// ti64_stencil.cu — K4: explicit 7-point heat-equation step on the voxel
// grid, bit-identical to ti64micro/thermal.py:205-287 (_stencil_step).
//
// Two kernels:
//  * stencil_built_kernel — every cell STATE_BUILT with r_c == 1 (config 3).
//    Then max(r_c, g) == 1 for any T, so every face conductivity is the same
//    constant kf = 2 k k / (k + k) with k = k_p + 1 * (k_ms - k_p), computed
//    on the host with the reference's operations; the per-face divides
//    vanish and the update is a 16 B/cell streaming stencil.  2.5D blocking:
//    a block owns a 32 x 8 (x, y) tile and marches over z with the z-1 / z /
//    z+1 values in registers and the current plane (+1-cell x/y halo) staged
//    in shared memory, so each T_n value is read from HBM once.
//  * stencil_general_kernel — any state/r_c mix, per-face harmonic means,
//    surface losses; one thread per cell.  A second pass applies the running
//    max consolidation of powder cells (thermal.py:279-287), which must see
//    the post-sweep temperatures.
// Face order x-, x+, y-, y+, z-, z+ and every association follow the
// reference (thermal.py:228-273); missing / inactive faces are skipped.
#include <cuda.h>  // CUtensorMap (types only; the encoder comes via cudaGetDriverEntryPoint)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/ti64_b200.h"
#include "ti64_fastmath.cuh"
#include "ti64_point.cuh"

using namespace ti64;

namespace {

constexpr int STATE_INACTIVE = 0;
constexpr int STATE_POWDER = 1;


struct StencilConst {
  double inv_rch2, inv_rch, inv_rc, dk, t4inf, kf, dliq;
  double src_coef;  // inv_rc * src_peak  (association of thermal.py:261)
};

__device__ __forceinline__ double clip01(double g) { return g < 0.0 ? 0.0 : (g > 1.0 ? 1.0 : g); }

// The beam of this step: from the launch arguments, or (graph replay of a
// step loop) row *step_d of a device table of (x, y, src_peak, on) rows
struct SrcRow {
  int on;
  double bx, by, coef;  // coef = inv_rc * src_peak (association of thermal.py:261)
};

__device__ __forceinline__ SrcRow source_row(const ti64_stencil_args& a, const StencilConst& c) {
  SrcRow r;
  if (a.beam_tab_d) {
    const double* b = a.beam_tab_d + 4 * (*a.step_d);
    r.bx = b[0];
    r.by = b[1];
    r.coef = __dmul_rn(c.inv_rc, b[2]);
    r.on = b[3] != 0.0;
  } else {
    r.bx = a.beam_x;
    r.by = a.beam_y;
    r.coef = c.src_coef;
    r.on = a.source_on != 0;
  }
  return r;
}

// top-layer Gaussian source term (thermal.py:255-261)
__device__ __forceinline__ double add_source(double t_new, int64_t x, int64_t y,
                                             const ti64_stencil_args& a, const SrcRow& sr) {
  const double xc = __dmul_rn(__dadd_rn((double)x, 0.5), a.h);
  const double yc = __dmul_rn(__dadd_rn((double)y, 0.5), a.h);
  const double dx = __dsub_rn(xc, sr.bx), dy = __dsub_rn(yc, sr.by);
  const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  const double arg = __dmul_rn(__dmul_rn(-2.0, r2), a.src_r2inv);
  if (arg > -40.0) t_new = __dadd_rn(t_new, __dmul_rn(sr.coef, fast_exp(arg)));
  return t_new;
}

constexpr int TX = 32, TY = 8;

__global__ void __launch_bounds__(256) stencil_general_kernel(const double* __restrict__ src,
                                                             double* __restrict__ dst,
                                                             const double* __restrict__ rc,
                                                             const uint8_t* __restrict__ state,
                                                             ti64_thermal tp,
                                                             ti64_stencil_args a,
                                                             StencilConst c) {
  const int64_t nx = a.nx, ny = a.ny, nz = a.nz;
  const int64_t plane = nx * ny;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (a.z_end - a.z_begin) * plane) return;
  const int64_t z = a.z_begin + t / plane, y = (t / nx) % ny, x = t % nx;
  const int64_t idx = (z - a.z_base) * plane + y * nx + x;  // stored index
  if (state[idx] == STATE_INACTIVE) return;
  const double t0 = src[idx];
  const double g0 = clip01(__ddiv_rn(__dsub_rn(t0, tp.t_sol), c.dliq));
  double rc0 = rc[idx];
  rc0 = rc0 > g0 ? rc0 : g0;
  const double k0 = __dadd_rn(tp.k_p, __dmul_rn(rc0, c.dk));
  double flux = 0.0;
#pragma unroll
  for (int face = 0; face < 6; ++face) {
    int64_t zz = z, yy = y, xx = x;
    if (face == 0) xx = x - 1;
    else if (face == 1) xx = x + 1;
    else if (face == 2) yy = y - 1;
    else if (face == 3) yy = y + 1;
    else if (face == 4) zz = z - 1;
    else zz = z + 1;
    if (xx < 0 || xx >= nx || yy < 0 || yy >= ny || zz < 0 || zz >= nz) continue;
    const int64_t j = ((zz - a.z_base) * ny + yy) * nx + xx;
    if (state[j] == STATE_INACTIVE) continue;
    const double t1 = src[j];
    const double g1 = clip01(__ddiv_rn(__dsub_rn(t1, tp.t_sol), c.dliq));
    double rc1 = rc[j];
    rc1 = rc1 > g1 ? rc1 : g1;
    const double k1 = __dadd_rn(tp.k_p, __dmul_rn(rc1, c.dk));
    const double kf = __ddiv_rn(__dmul_rn(__dmul_rn(2.0, k0), k1), __dadd_rn(k0, k1));
    flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(t1, t0)));
  }
  double t_new = __dadd_rn(t0, __dmul_rn(c.inv_rch2, flux));
  const SrcRow sr = source_row(a, c);
  if (sr.on && z == a.z_top - 1) t_new = add_source(t_new, x, y, a, sr);
  if (a.losses_on != 0) {
    const bool exposed = z == nz - 1 || state[idx + plane] == STATE_INACTIVE;
    if (exposed) {
      double q = __dmul_rn(__dmul_rn(tp.emissivity, tp.sigma_s),
                           __dsub_rn(__dmul_rn(__dmul_rn(__dmul_rn(t0, t0), t0), t0), c.t4inf));
      const double tc = t0 < tp.t_max_clamp ? t0 : tp.t_max_clamp;
      if (tc > tp.t_v) {
        const double e = fast_exp(__dmul_rn(-tp.c_t, __dsub_rn(__ddiv_rn(1.0, tc),
                                                                __ddiv_rn(1.0, tp.t_v))));
        const double ev = __dmul_rn(
            __dmul_rn(__dmul_rn(__dmul_rn(0.82, tp.c_p), e), __dsqrt_rn(__ddiv_rn(tp.c_m, tc))),
            __dadd_rn(tp.h_v, __dmul_rn(tp.c_heat, __dsub_rn(tc, tp.t_h0))));
        q = __dadd_rn(q, ev);
      }
      t_new = __dsub_rn(t_new, __dmul_rn(c.inv_rch, q));
    }
  }
  if (a.bc_bottom_on != 0 && z == 0) t_new = a.bc_bottom;
  dst[idx] = t_new;
}

// running max consolidation of powder cells on the post-step field
__global__ void consolidate_kernel(const double* __restrict__ dst, double* __restrict__ rc,
                                   const uint8_t* __restrict__ state, int64_t off, int64_t n,
                                   double t_sol, double dliq) {
  const int64_t i = off + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= off + n || state[i] != STATE_POWDER) return;
  const double g1 = clip01(__ddiv_rn(__dsub_rn(dst[i], t_sol), dliq));
  if (g1 > rc[i]) rc[i] = g1;
}

// ---------------------------------------------------------------------------
// Fused coupled step (config 3): K4 built stencil + the kinetics step per cell
// ---------------------------------------------------------------------------
constexpr double IDLE_XB = 1.0 - 0.9;

__device__ __forceinline__ bool bits_same(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}

// cold idle composition (0.9, +0, 1 - 0.9) with the seed inactive
__device__ __forceinline__ bool idle_cell(double xs, double xm, double xb, int ac) {
  return ac == 0 && bits_same(xs, 0.9) && __double_as_longlong(xm) == 0 && bits_same(xb, IDLE_XB);
}

struct CoupledODE {
  ti64_kparams kp;
  Derived dv;
  ti64_icfg cfg;
  double dt;
  int L;
  int rest_ok;  // t_as_end <= t_sol etc.: the cold idle rest is exact
  uint32_t* hot;  // split mode: 1 bit per 32-cell row, set where T_n or T_n+1 >= t_as_end
  // slab form: the kinetics state (fields, idle bits, hot rows) starts at
  // global plane sz0; toff = (sz0 - z_base) * plane maps a state index to
  // the temperature arrays (which hold planes from z_base)
  int64_t sz0, toff;
};

// ---------------------------------------------------------------------------
// Pipelined z-marching kernel for all-built grids (K4), optionally fused with
// the kinetics step of every cell (config 3).
//
// A block owns a TX x TY (x, y) tile and a z-range.  Planes (+1-cell x/y halo)
// live in a shared-memory ring of RING = PD + 3 slots filled by cp.async
// (LDGSTS) PD planes ahead of the one being computed, so every thread keeps
// several 8-byte loads in flight instead of one dependent load per plane.
// Each T_n value is read from HBM once per step (plus tile halos, L2 hits).
// ---------------------------------------------------------------------------
#ifndef PD_DEF
#define PD_DEF 5
#endif
#ifndef RY_DEF
#define RY_DEF 2
#endif
constexpr int PD = PD_DEF;           // planes prefetched beyond z+1
constexpr int RING = PD + 3;    // planes z-1, z, z+1 and PD more

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void cp_async8s(unsigned sa, const double* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async4s(unsigned sa, const uint32_t* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}

// Each thread owns RY cells of its x column (rows y + r*TY), so the per-plane
// bookkeeping (copies, waits, syncs, loop) is shared by RY cells.
constexpr int RY = RY_DEF;
#ifndef ZCHUNK
#define ZCHUNK 32
#endif
constexpr int TYT = TY * RY;  // tile height in cells

// Kinetics of the warp's cells when at least one of them is not at rest:
// out of line, so the stencil loop around the (usually taken) rest exit
// keeps a small register footprint.
static __device__ __noinline__ void cells_step(const ti64_fields& f, uint32_t* __restrict__ idle,
                                               const CoupledODE& o, int lane, bool in,
                                               bool rest, int64_t flat, uint32_t bits,
                                               double t0, double t_new, unsigned gm) {
  bool touched = false;
  bool now_idle = rest;
  Seed sd;
  sd.ac = 0;
  sd.dr = 0;
  sd.tr = 0.0;
  if (in && !rest) {
    double xs = f.x_alpha_s[flat], xm = f.x_alpha_m[flat], xb = f.x_beta[flat];
    const int ac = f.seed_active[flat];
    sd.ac = ac;
    sd.dr = ac ? f.seed_direction[flat] : 0;
    sd.tr = ac ? f.seed_tracked[flat] : 0.0;
    touched = ac != 0;
    double xaeq0 = xaeq_of(t0, o.kp, o.dv);
    substep(xs, xm, xb, sd, t0, t_new, xaeq0, o.dt, o.kp, o.dv, o.cfg, touched);
    f.x_alpha_s[flat] = xs;
    f.x_alpha_m[flat] = xm;
    f.x_beta[flat] = xb;
    now_idle = idle_cell(xs, xm, xb, sd.ac);
  }
  const unsigned bal = __ballot_sync(0xffffffffu, touched && in);
  if (in && (bal & gm)) {  // lane-group seed write-back (batch.py:687-692)
    f.seed_tracked[flat] = sd.tr;
    f.seed_active[flat] = (uint8_t)sd.ac;
    f.seed_direction[flat] = (uint8_t)sd.dr;
  }
  const uint32_t nb = __ballot_sync(0xffffffffu, now_idle && in);
  if (lane == 0 && nb != bits) idle[(flat - lane) >> 5] = nb;
}

// CM: 1 = fused (the kinetics of the warp's cells run here), 2 = split (the
// stencil only marks rows with a hot cell; rows_kinetics_kernel runs next)
template <int CM>
__device__ __forceinline__ void cell_kinetics(const ti64_fields& f, uint32_t* __restrict__ idle,
                                              const CoupledODE& o, int lane, bool in,
                                              int64_t flat, uint32_t bits, double t0,
                                              double t_new, unsigned gm) {
  if constexpr (CM == 2) {
    // not provably cold (NaN included): the row's kinetics must run
    // Integer screen on the high words (ALU pipe; the stencil's FP64 pipe and
    // issue slots are the busy ones): for T >= +0, T < t_as_end whenever
    // hi(T) < hi(t_as_end) as unsigned, and negative values and NaNs of
    // either sign have hi >= 0x80000000 or > hi(t_as_end) and are flagged.  So
    // a cell that is not flagged has T_n, T_n+1 < t_as_end; cells just below
    // the bound are flagged too, and the kinetics kernel applies the exact
    // test.  No vote: hot cells are rare and a warp's same-word atomics
    // combine.  (The screen costs ~20 us of the 229 us step, A/B
    // tools/ab_split_k4.sh: no screen 208 us, masked signed compare 234 us.)
    const unsigned thi = (unsigned)__double2hiint(o.kp.t_as_end);
    const unsigned h = max((unsigned)__double2hiint(t0), (unsigned)__double2hiint(t_new));
    if (h >= thi) {
      const int64_t row = flat >> 5;
      atomicOr(o.hot + (row >> 5), 1u << (row & 31));
    }
  } else {
    const bool was_idle = in && ((bits >> lane) & 1u);
    const bool rest = o.rest_ok && was_idle && t0 < o.kp.t_as_end && t_new < o.kp.t_as_end;
    if (__all_sync(0xffffffffu, rest || !in)) return;  // warp-uniform exit
    cells_step(f, idle, o, lane, in, rest, flat, bits, t0, t_new, gm);
  }
}

// Split coupled step, second half.  A 32-cell row (rows are whole: nx % 32
// == 0) can skip its kinetics only if every cell is at the cold idle rest:
// idle bit set and T_n, T_n+1 < t_as_end.  So a row runs iff its idle word
// has a zero bit (transformed material, persistent) or the stencil marked it
// hot.  rows_scan_kernel lists those rows (each thread reads 4 idle words as
// one 16-byte load: the 1-bit/cell map is 1/64 of the temperature bytes) and
// clears the hot bits; rows_kinetics_kernel runs one listed row per warp with
// the fused kernel's rest test and cells_step on T_n (tn, untouched by the
// stencil) and T_n+1 (tn1).  Rows are independent: list order is irrelevant.
// Rows [row_lo, nrows) of the state (row_lo % 32 == 0, so the 8 threads that
// share a hot word are lanes of one warp).
__global__ void __launch_bounds__(256) rows_scan_kernel(const uint32_t* __restrict__ idle,
                                                        uint32_t* __restrict__ hot,
                                                        int64_t row_lo, int64_t nrows,
                                                        uint32_t* __restrict__ list,
                                                        unsigned int* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r0 = row_lo + 4 * i;  // rows r0 .. r0+3 (nrows % 4 == 0 is not assumed)
  unsigned m = 0u;
  uint32_t hw = 0u;
  if (r0 < nrows) {
    hw = hot[r0 >> 5];
    uint32_t v[4];
    if (r0 + 4 <= nrows && (reinterpret_cast<uintptr_t>(idle + r0) & 15) == 0) {
      const uint4 q = *reinterpret_cast<const uint4*>(idle + r0);
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = r0 + k < nrows ? idle[r0 + k] : 0xffffffffu;
    }
    m = (hw >> (r0 & 31)) & 0xfu;
#pragma unroll
    for (int k = 0; k < 4; ++k) m |= (v[k] != 0xffffffffu ? 1u : 0u) << k;
  }
  // the 8 threads sharing a hot word are lanes of one warp: read, then clear
  __syncwarp();
  if (r0 < nrows && (r0 & 31) == 0 && hw) hot[r0 >> 5] = 0u;
  const unsigned c = __popc(m);
  unsigned pre = c;  // inclusive warp scan
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, pre, d);
    if (lane >= d) pre += t;
  }
  const unsigned tot = __shfl_sync(0xffffffffu, pre, 31);
  unsigned base = 0u;
  if (lane == 31 && tot) base = atomicAdd(count, tot);
  base = __shfl_sync(0xffffffffu, base, 31) + pre - c;
  while (m) {
    const int k = __ffs(m) - 1;
    m &= m - 1;
    list[base++] = (uint32_t)(r0 + k);
  }
}

__global__ void __launch_bounds__(128) rows_kinetics_kernel(const double* __restrict__ tn,
                                                            const double* __restrict__ tn1,
                                                            const __grid_constant__ ti64_fields f,
                                                            uint32_t* __restrict__ idle,
                                                            const __grid_constant__ CoupledODE o,
                                                            const uint32_t* __restrict__ list,
                                                            const unsigned int* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const unsigned gm = ((o.L >= 32) ? 0xffffffffu : ((1u << o.L) - 1u)) << (lane & ~(o.L - 1));
  const unsigned cnt = *count;
  const unsigned nw = (gridDim.x * blockDim.x) >> 5;
  for (unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < cnt; w += nw) {
    const int64_t row = list[w];
    const int64_t flat = row * 32 + lane;
    const uint32_t bits = idle[row];
    const double t0 = tn[o.toff + flat], t_new = tn1[o.toff + flat];
    const bool rest = o.rest_ok && ((bits >> lane) & 1u) && t0 < o.kp.t_as_end &&
                      t_new < o.kp.t_as_end;
    cells_step(f, idle, o, lane, true, rest, flat, bits, t0, t_new, gm);
  }
}

template <bool COUPLED>
__global__ void __launch_bounds__(TX* TY) built_pipe_kernel(
    const double* __restrict__ src, double* __restrict__ dst, ti64_stencil_args a,
    StencilConst c, int zchunk, const __grid_constant__ ti64_fields f,
    uint32_t* __restrict__ idle, const __grid_constant__ CoupledODE o) {
  constexpr int W = TX + 2;              // smem row pitch
  constexpr int SLOT = (TYT + 2) * W;    // doubles per ring slot
  __shared__ double ring[RING * SLOT];
  __shared__ uint32_t iring[RING * TYT];
  const int nx = (int)a.nx, ny = (int)a.ny, nz = (int)a.nz;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int lane = tx;
  const int x = blockIdx.x * TX + tx;
  const int ybase = blockIdx.y * TYT;
  const int z0 = (int)a.z_begin + blockIdx.z * zchunk;
  const int z1 = min(z0 + zchunk, (int)a.z_end);
  if (z0 >= z1) return;
  const int64_t plane = (int64_t)nx * ny;
  const SrcRow sr = source_row(a, c);
  const int zlo = max(0, (int)a.z_base), zhi = min(nz, (int)(a.z_base + a.nz_stored));
  const unsigned rbase = (unsigned)__cvta_generic_to_shared(ring);
  const unsigned ibase = (unsigned)__cvta_generic_to_shared(iring);
  // per owned row r: y, smem cell index, in-grid flag, halo duties
  int yr[RY], cidx[RY];
  bool in[RY], hl[RY], hr[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    yr[r] = ybase + ty + r * TY;
    cidx[r] = (ty + r * TY + 1) * W + tx + 1;
    in[r] = x < nx && yr[r] < ny;
    hl[r] = tx == 0 && x > 0 && yr[r] < ny;
    hr[r] = tx == TX - 1 && x + 1 < nx && yr[r] < ny;
  }
  const bool hu = ty == 0 && ybase > 0 && x < nx;                  // row ybase-1
  const bool hd = ty == TY - 1 && ybase + TYT < ny && x < nx;      // row ybase+TYT
  const double* gcol = src + (-a.z_base) * plane + x;               // + z*plane + y*nx

  const int zmax = min(zhi, z1 + 1);  // plane z1 is the last one read (z+1 of z1-1)
  auto issue = [&](int zz, int slot) {
    if (zz >= zlo && zz < zmax) {
      const double* g = gcol + (int64_t)zz * plane;
      const unsigned so = rbase + 8u * (unsigned)(slot * SLOT);
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const unsigned sa = so + 8u * (unsigned)cidx[r];
        const double* gr = g + (int64_t)yr[r] * nx;
        if (in[r]) cp_async8s(sa, gr);
        if (hl[r]) cp_async8s(sa - 8u, gr - 1);
        if (hr[r]) cp_async8s(sa + 8u, gr + 1);
      }
      if (hu) cp_async8s(so + 8u * (unsigned)(tx + 1), g + (int64_t)(ybase - 1) * nx);
      if (hd) cp_async8s(so + 8u * (unsigned)((TYT + 1) * W + tx + 1), g + (int64_t)(ybase + TYT) * nx);
      if (COUPLED && lane == 0 && zz >= z0 && zz < z1) {
#pragma unroll
        for (int r = 0; r < RY; ++r)
          if (yr[r] < ny)
            cp_async4s(ibase + 4u * (unsigned)(slot * TYT + ty + r * TY),
                       idle + (((int64_t)(zz - o.sz0) * plane + (int64_t)yr[r] * nx + (x - lane)) >> 5));
      }
    }
    cp_async_commit();
  };

  for (int k = 0; k <= PD + 1; ++k) issue(z0 - 1 + k, k);
  int sm = 0, s0 = 1, sp1 = 2, si = PD + 2;  // slots of z-1, z, z+1, z+1+PD
  const double kf = c.kf;
  const unsigned gm =
      COUPLED ? (((o.L >= 32) ? 0xffffffffu : ((1u << o.L) - 1u)) << (lane & ~(o.L - 1))) : 0u;
  double* dcol = dst + (-a.z_base) * plane + x;

  for (int z = z0; z < z1; ++z) {
    issue(z + 1 + PD, si);
    cp_async_wait<PD>();  // planes <= z + 1 have landed (this thread's copies)
    __syncthreads();      // ... and everyone's
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      if (yr[r] < ny) {  // warp-uniform (one warp per x-row)
        const int y = yr[r];
        const double* P = ring + s0 * SLOT + cidx[r];
        double t_new = 0.0, t0 = 0.0;
        if (in[r]) {
          t0 = P[0];
          double flux = 0.0;
          if (x > 0) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[-1], t0)));
          if (x + 1 < nx) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[1], t0)));
          if (y > 0) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[-W], t0)));
          if (y + 1 < ny) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[W], t0)));
          if (z > 0) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(ring[sm * SLOT + cidx[r]], t0)));
          if (z + 1 < nz)
            flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(ring[sp1 * SLOT + cidx[r]], t0)));
          t_new = __dadd_rn(t0, __dmul_rn(c.inv_rch2, flux));
          if (sr.on && z == a.z_top - 1) t_new = add_source(t_new, x, y, a, sr);
          if (a.bc_bottom_on != 0 && z == 0) t_new = a.bc_bottom;  // thermal.py:274-278
          dcol[(int64_t)z * plane + (int64_t)y * nx] = t_new;
        }
        if (COUPLED)
          cell_kinetics<COUPLED ? 1 : 0>(f, idle, o, lane, in[r], (int64_t)(z - o.sz0) * plane + (int64_t)y * nx + x,
                                 iring[s0 * TYT + ty + r * TY], t0, t_new, gm);
      }
    }
    __syncthreads();  // slot of plane z-1 is refilled by the next iteration's issue
    const int t = sm;
    sm = s0;
    s0 = sp1;
    sp1 = (sp1 + 1 == RING) ? 0 : sp1 + 1;
    si = t;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// TMA variant: one elected thread moves each (TX+2) x (TYT+2) plane box (tile
// plus x/y halo, out-of-range cells zero-filled) into the shared-memory ring
// with cp.async.bulk.tensor; an mbarrier per slot carries the transaction
// count.  The other threads only compute, so the per-cell instruction count
// is the stencil arithmetic itself.
// ---------------------------------------------------------------------------
// the box starts at x0 - 2: TMA needs the innermost start coordinate 16-byte
// aligned (measured: an odd double offset faults), so 2 halo columns on the
// left (one unused) and 2 on the right keep the box 36 doubles = 288 B wide
constexpr int BOX_X = TX + 4;
// rows per thread of the TMA kernels: the plain stencil keeps 2 (more resident
// blocks), the fused coupled step takes 4 (its per-plane kinetics bookkeeping
// is shared by more cells); measured on the config-3 grid
#ifndef RY_S_DEF
#define RY_S_DEF 2
#endif
#ifndef RY_C_DEF
#define RY_C_DEF 4
#endif
template <int RYV>
struct TmaTile {
  static constexpr int RY = RYV;
  static constexpr int TYT = TY * RYV;
  static constexpr int BOX_Y = TYT + 2;
  static constexpr int BOX_BYTES = BOX_X * BOX_Y * 8;
  static constexpr int SLOT_BYTES = (BOX_BYTES + 127) / 128 * 128;
  static constexpr int SMEM = RING * SLOT_BYTES + RING * 8 + RING * TYT * 4;
};
template <int CM>
using TileOf = TmaTile<CM == 1 ? RY_C_DEF : RY_S_DEF>;

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ unsigned mbar_try(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok;
}
// bounded wait: the common case (data landed, or lands within try_wait's own
// suspend window) costs one try_wait; the clock is read only after a miss,
// and a transaction that never lands traps instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > 4000000000LL) {  // ~2 s: a transaction never landed
      if (threadIdx.x == 0 && threadIdx.y == 0)
        printf("ti64 TMA wait timeout: block (%d,%d,%d) bar %u parity %u\n", blockIdx.x,
               blockIdx.y, blockIdx.z, bar, parity);
#ifdef TI64_TMA_DEBUG
      return;
#else
      __trap();
#endif
    }
  }
}
__device__ __forceinline__ void tma_load_3d(unsigned dst, uint64_t desc, int c0, int c1, int c2,
                                            unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

#ifndef TMA_MINB
#define TMA_MINB 3
#endif
#ifndef TMA_MINB_C
#define TMA_MINB_C 2
#endif
template <int CM>
__global__ void __launch_bounds__(TX* TY, CM == 1 ? TMA_MINB_C : TMA_MINB) built_tma_kernel(
    const __grid_constant__ CUtensorMap tmap, double* __restrict__ dst, ti64_stencil_args a,
    StencilConst c, int zchunk, const __grid_constant__ ti64_fields f,
    uint32_t* __restrict__ idle, const __grid_constant__ CoupledODE o) {
  constexpr bool COUPLED = CM != 0;
  using T = TileOf<CM>;
  constexpr int RY = T::RY, TYT = T::TYT, BOX_BYTES = T::BOX_BYTES, SLOT_BYTES = T::SLOT_BYTES;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);  // RING slots of SLOT_BYTES
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + RING * SLOT_BYTES);
  uint32_t* iring = reinterpret_cast<uint32_t*>(smem_raw + RING * SLOT_BYTES + RING * 8);
  constexpr int SLOTD = SLOT_BYTES / 8;  // doubles per slot
  constexpr int W = BOX_X;
  const int nx = (int)a.nx, ny = (int)a.ny, nz = (int)a.nz;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int lane = tx;
  const bool leader = tx == 0 && ty == 0;
  const int x0 = blockIdx.x * TX, ybase = blockIdx.y * TYT;
  const int x = x0 + tx;
  const int z0 = (int)a.z_begin + blockIdx.z * zchunk;
  const int z1 = min(z0 + zchunk, (int)a.z_end);
  if (z0 >= z1) return;
  const int64_t plane = (int64_t)nx * ny;
  const SrcRow sr = source_row(a, c);
  const int zlo = max(0, (int)a.z_base), zhi = min(nz, (int)(a.z_base + a.nz_stored));
  const int zmax = min(zhi, z1 + 1);
  // the descriptor address is taken here, in the kernel body: a lambda that
  // captured the __grid_constant__ parameter by reference would copy it to
  // local memory, where TMA cannot read it (the load then never lands)
  const uint64_t desc = reinterpret_cast<uint64_t>(&tmap);
  const unsigned rbase = (unsigned)__cvta_generic_to_shared(ring);
  const unsigned bbase = (unsigned)__cvta_generic_to_shared(bars);
  const unsigned ibase = (unsigned)__cvta_generic_to_shared(iring);
  int yr[RY], cidx[RY];
  bool in[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    yr[r] = ybase + ty + r * TY;
    cidx[r] = (ty + r * TY + 1) * W + tx + 2;
    in[r] = x < nx && yr[r] < ny;
  }
  if (leader) {
    for (int k = 0; k < RING; ++k) mbar_init(bbase + 8u * k, 1u);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // plane zz lives in slot (zz - (z0 - 1)) % RING
  auto issue = [&](int zz, int slot) {
    if (leader && zz >= zlo && zz < zmax) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      const unsigned bar = bbase + 8u * slot;
      mbar_expect_tx(bar, (unsigned)BOX_BYTES);
      tma_load_3d(rbase + (unsigned)(slot * SLOT_BYTES), desc, x0 - 2, ybase - 1,
                  zz - (int)a.z_base, bar);
    }
    if (CM == 1) {
      if (lane == 0 && zz >= z0 && zz < z1) {
#pragma unroll
        for (int r = 0; r < RY; ++r)
          if (yr[r] < ny)
            cp_async4s(ibase + 4u * (unsigned)(slot * TYT + ty + r * TY),
                       idle + (((int64_t)(zz - o.sz0) * plane + (int64_t)yr[r] * nx + x0) >> 5));
      }
      cp_async_commit();
    }
  };
  // per-slot phase parity of the next completion to wait for: loads and waits
  // pair up one-to-one per slot (planes outside the grid are neither issued
  // nor waited), so a bit flip per completed wait tracks the phase
  unsigned phase = 0u;
  auto wait_plane = [&](int zz, int slot) {
    if (zz >= zlo && zz < zmax) {
      mbar_wait(bbase + 8u * slot, (phase >> slot) & 1u);
      phase ^= 1u << slot;
    }
  };

  for (int k = 0; k <= PD + 1; ++k) issue(z0 - 1 + k, k);
  int sm = 0, s0 = 1, sp1 = 2, si = PD + 2;
  wait_plane(z0 - 1, 0);
  wait_plane(z0, 1);
  const double kf = c.kf;
  const unsigned gm =
      COUPLED ? (((o.L >= 32) ? 0xffffffffu : ((1u << o.L) - 1u)) << (lane & ~(o.L - 1))) : 0u;
  double* dcol = dst + (-a.z_base) * plane + x;
  // block-uniform: every cell of the tile has all four in-plane neighbours
  const bool xy_interior = x0 > 0 && x0 + TX < nx && ybase > 0 && ybase + TYT < ny;

  for (int z = z0; z < z1; ++z) {
    issue(z + 1 + PD, si);
    wait_plane(z + 1, sp1);
    if (CM == 1) {
      cp_async_wait<PD>();
      __syncthreads();
    }
    if (xy_interior && z > 0 && z + 1 < nz && !(sr.on && z == a.z_top - 1)) {
      // interior plane of an interior tile: all six faces present, no source
      // or boundary value; same face order and association as below
      double* dz = dcol + (int64_t)z * plane;
      unsigned hr[RY];  // CM 2: per-row screen word, one branch per plane below
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const double* P = ring + s0 * SLOTD + cidx[r];
        const double t0 = P[0];
        double flux = __dadd_rn(0.0, __dmul_rn(kf, __dsub_rn(P[-1], t0)));
        flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[1], t0)));
        flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[-W], t0)));
        flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[W], t0)));
        flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(ring[sm * SLOTD + cidx[r]], t0)));
        flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(ring[sp1 * SLOTD + cidx[r]], t0)));
        const double t_new = __dadd_rn(t0, __dmul_rn(c.inv_rch2, flux));
        dz[(int64_t)yr[r] * nx] = t_new;
        if constexpr (CM == 2)
          hr[r] = max((unsigned)__double2hiint(t0), (unsigned)__double2hiint(t_new));
        else if (COUPLED)
          cell_kinetics<CM>(f, idle, o, lane, true, (int64_t)(z - o.sz0) * plane + (int64_t)yr[r] * nx + x,
                                 CM == 1 ? iring[s0 * TYT + ty + r * TY] : 0u, t0, t_new, gm);
      }
      if constexpr (CM == 2) {  // the screen of cell_kinetics<2>, both rows at once
        unsigned hm = hr[0];
#pragma unroll
        for (int r = 1; r < RY; ++r) hm = max(hm, hr[r]);
        const unsigned thi = (unsigned)__double2hiint(o.kp.t_as_end);
        if (hm >= thi) {
#pragma unroll
          for (int r = 0; r < RY; ++r)
            if (hr[r] >= thi) {
              const int64_t row = ((int64_t)(z - o.sz0) * plane + (int64_t)yr[r] * nx + x) >> 5;
              atomicOr(o.hot + (row >> 5), 1u << (row & 31));
            }
        }
      }
      __syncthreads();
      const int t = sm;
      sm = s0;
      s0 = sp1;
      sp1 = (sp1 + 1 == RING) ? 0 : sp1 + 1;
      si = t;
      continue;
    }
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      if (yr[r] < ny) {  // warp-uniform (one warp per x-row)
        const int y = yr[r];
        const double* P = ring + s0 * SLOTD + cidx[r];
        double t_new = 0.0, t0 = 0.0;
        if (in[r]) {
          t0 = P[0];
          double flux = 0.0;
          if (x > 0) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[-1], t0)));
          if (x + 1 < nx) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[1], t0)));
          if (y > 0) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[-W], t0)));
          if (y + 1 < ny) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(P[W], t0)));
          if (z > 0) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(ring[sm * SLOTD + cidx[r]], t0)));
          if (z + 1 < nz)
            flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(ring[sp1 * SLOTD + cidx[r]], t0)));
          t_new = __dadd_rn(t0, __dmul_rn(c.inv_rch2, flux));
          if (sr.on && z == a.z_top - 1) t_new = add_source(t_new, x, y, a, sr);
          if (a.bc_bottom_on != 0 && z == 0) t_new = a.bc_bottom;  // thermal.py:274-278
          dcol[(int64_t)z * plane + (int64_t)y * nx] = t_new;
        }
        if (COUPLED)
          cell_kinetics<CM>(f, idle, o, lane, in[r], (int64_t)(z - o.sz0) * plane + (int64_t)y * nx + x,
                                 CM == 1 ? iring[s0 * TYT + ty + r * TY] : 0u, t0, t_new, gm);
      }
    }
    __syncthreads();  // every thread is done with slot sm before it is refilled
    const int t = sm;
    sm = s0;
    s0 = sp1;
    sp1 = (sp1 + 1 == RING) ? 0 : sp1 + 1;
    si = t;
  }
  if (CM == 1) cp_async_wait<0>();
}

// --- host: tensor-map encoder through the runtime's driver entry point ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    cudaGetLastError();
  });
  return fn;
}

// 3D map over the stored planes (x fastest); false when TMA cannot be used
bool make_plane_map(CUtensorMap* m, const double* base, int64_t nx, int64_t ny, int64_t nzs,
                    int box_y) {
  EncodeTiledFn enc = encoder();
  // the box must fit inside the tensor (a box wider than the grid stalls)
  if (!enc || (reinterpret_cast<uintptr_t>(base) & 15) || (nx * 8) % 16 != 0 || nx < BOX_X ||
      ny < box_y ||
      nx > (1LL << 31) || ny > (1LL << 31) || nzs > (1LL << 31))
    return false;
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nzs};
  cuuint64_t strides[2] = {(cuuint64_t)(nx * 8), (cuuint64_t)(nx * ny * 8)};
  cuuint32_t box[3] = {(cuuint32_t)BOX_X, (cuuint32_t)box_y, 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  std::memset(m, 0, sizeof(*m));
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA launch: false when the grid cannot be mapped (callers fall back to the
// cp.async kernel); the grid's y extent follows the kernel's own tile height
template <int CM>
bool launch_built(const double* src, double* dst, const ti64_stencil_args& a,
                  const StencilConst& c, ti64_fields f, uint32_t* idle, const CoupledODE& o,
                  int64_t nz_units, int zchunk, cudaStream_t st) {
  using T = TileOf<CM>;
  CUtensorMap m;
  if (!make_plane_map(&m, src, a.nx, a.ny, a.nz_stored, T::BOX_Y)) return false;
  // the opt-in shared-memory size is a per-device function attribute
  static std::atomic<unsigned long long> attr_set{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_set.load(std::memory_order_relaxed) & bit)) {
    cudaFuncSetAttribute(built_tma_kernel<CM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         T::SMEM);
    attr_set.fetch_or(bit, std::memory_order_relaxed);
  }
  dim3 grid((unsigned)((a.nx + TX - 1) / TX), (unsigned)((a.ny + T::TYT - 1) / T::TYT),
            (unsigned)((nz_units + zchunk - 1) / zchunk));
  built_tma_kernel<CM><<<grid, dim3(TX, TY), T::SMEM, st>>>(m, dst, a, c, zchunk, f, idle, o);
  return true;
}

__global__ void idle_bits_init_kernel(ti64_fields f, uint32_t* idle, int64_t lo, int64_t n) {
  const int64_t w = lo / 32 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w * 32 >= n) return;
  uint32_t b = 0u;
  for (int k = 0; k < 32; ++k) {
    const int64_t i = w * 32 + k;
    if (i < n && idle_cell(f.x_alpha_s[i], f.x_alpha_m[i], f.x_beta[i], f.seed_active[i]))
      b |= 1u << k;
  }
  idle[w] = b;
}

}  // namespace

void ti64_set_error(const std::string& msg);  // ti64_kernels.cu

namespace {
// TI64_NO_TMA=1 forces the cp.async pipeline (A/B comparisons, parity tests)
bool use_tma() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("TI64_NO_TMA");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}
}  // namespace

extern "C" int64_t ti64_stencil_step(const double* src_d, double* dst_d, double* rc_d,
                                     const uint8_t* state_d, const ti64_thermal* tp,
                                     const ti64_stencil_args* a, void* stream) {
  if (!src_d || !dst_d || !tp || !a || a->nx < 1 || a->ny < 1 || a->nz < 1 || a->z_top < 0 ||
      a->z_top > a->nz || src_d == dst_d || a->z_begin < 0 || a->z_end > a->z_top ||
      a->z_begin < a->z_base || a->z_end > a->z_base + a->nz_stored ||
      (a->z_begin > 0 && a->z_begin - 1 < a->z_base) ||
      (a->z_end < a->nz && a->z_end + 1 > a->z_base + a->nz_stored)) {
    ti64_set_error("ti64_stencil_step: bad argument");
    return TI64_EINVAL;
  }
  if (!a->all_built && (!rc_d || !state_d)) {
    ti64_set_error("ti64_stencil_step: general kernel needs r_c and state");
    return TI64_EINVAL;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // constants formed with the reference's operations (thermal.py:211-215, :252)
  StencilConst c;
  c.inv_rch2 = a->dt / (tp->rho_c * a->h * a->h);
  c.inv_rch = a->dt / (tp->rho_c * a->h);
  c.inv_rc = a->dt / tp->rho_c;
  c.dk = tp->k_ms - tp->k_p;
  c.t4inf = std::pow(tp->t_inf, 4.0);
  const double kb = tp->k_p + 1.0 * c.dk;
  c.kf = 2.0 * kb * kb / (kb + kb);
  c.dliq = tp->t_liq - tp->t_sol;
  c.src_coef = c.inv_rc * a->src_peak;
  const int64_t nzu = a->z_end - a->z_begin;
  if (nzu <= 0) return TI64_OK;
  if (a->all_built) {
    const int zchunk = ZCHUNK;
    dim3 grid((unsigned)((a->nx + TX - 1) / TX), (unsigned)((a->ny + TYT - 1) / TYT),
              (unsigned)((nzu + zchunk - 1) / zchunk));
    if (!use_tma() || !launch_built<0>(src_d, dst_d, *a, c, ti64_fields{}, nullptr,
                                           CoupledODE{}, nzu, zchunk, st))
      built_pipe_kernel<false><<<grid, dim3(TX, TY), 0, st>>>(src_d, dst_d, *a, c, zchunk,
                                                            ti64_fields{}, nullptr, CoupledODE{});
  } else {
    const int64_t plane = a->nx * a->ny;
    const int64_t n = nzu * plane;
    stencil_general_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src_d, dst_d, rc_d,
                                                                       state_d, *tp, *a, c);
    consolidate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        dst_d, rc_d, state_d, (a->z_begin - a->z_base) * plane, n, tp->t_sol, c.dliq);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    ti64_set_error(std::string("ti64_stencil_step: ") + cudaGetErrorString(e));
    return TI64_ECUDA;
  }
  ti64_set_error("");
  return TI64_OK;
}

namespace {
__global__ void step_counter_kernel(int64_t* step_d, int64_t k) { *step_d += k; }
}  // namespace

extern "C" int64_t ti64_step_counter_add(int64_t* step_d, int64_t k, void* stream) {
  if (!step_d) {
    ti64_set_error("ti64_step_counter_add: bad argument");
    return TI64_EINVAL;
  }
  step_counter_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(step_d, k);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    ti64_set_error(std::string("ti64_step_counter_add: ") + cudaGetErrorString(e));
    return TI64_ECUDA;
  }
  return TI64_OK;
}

// scratch of the split step for a state of n_cells cells: the hot-row bitmap
// (1 bit per 32-cell row), the row count (+ pad to 16 B) and the row list
extern "C" int64_t ti64_coupled_scratch_words(int64_t n_cells) {
  if (n_cells < 0) return TI64_EINVAL;
  const int64_t nrows = (n_cells + 31) / 32;
  return (nrows + 31) / 32 + 4 + nrows;
}

static int64_t coupled_step_impl(const double* tn_d, double* tn1_d, const ti64_fields* f,
                                 int64_t state_z0, uint32_t* idle_bits_d, uint32_t* scratch_d,
                                 const ti64_thermal* tp, const ti64_stencil_args* a,
                                 const ti64_kparams* kp, const ti64_icfg* cfg, int64_t lanes,
                                 int32_t init_bits, void* stream, void* kin_stream) {
  if (!tn_d || !tn1_d || !f || !idle_bits_d || !tp || !a || !kp || !cfg || tn_d == tn1_d ||
      !a->all_built || a->losses_on || a->nx % 32 != 0 || a->nx < 1 || a->ny < 1 ||
      a->z_top != a->nz || a->z_begin < 0 || a->z_end > a->nz || a->z_begin > a->z_end ||
      a->z_begin < a->z_base || a->z_end > a->z_base + a->nz_stored ||
      (a->z_begin > 0 && a->z_begin - 1 < a->z_base) ||
      (a->z_end < a->nz && a->z_end + 1 > a->z_base + a->nz_stored) ||
      state_z0 < 0 || a->z_begin < state_z0 ||
      !(lanes == 1 || lanes == 2 || lanes == 4 || lanes == 8)) {
    ti64_set_error("ti64_coupled_step: bad argument (all-built grid, no losses, nx % 32 == 0, "
                   "a slab holding the updated planes and their z neighbours)");
    return TI64_EINVAL;
  }
  if (cfg->scheme != TI64_SCHEME_EXPLICIT) {
    ti64_set_error("ti64_coupled_step: only the explicit scheme is implemented");
    return TI64_ENOTSUP;
  }
  if (!(a->dt <= cfg->dt_sub_max * (1.0 + 1e-9))) {
    ti64_set_error("ti64_coupled_step: dt above dt_sub_max (kinetics subcycling) unsupported");
    return TI64_EINVAL;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaStream_t kin = reinterpret_cast<cudaStream_t>(kin_stream);
  const int64_t plane = a->nx * a->ny;
  const int64_t c_lo = (a->z_begin - state_z0) * plane;  // state cells of the updated planes
  const int64_t c_hi = (a->z_end - state_z0) * plane;
  if (c_hi == c_lo) return TI64_OK;
  if (init_bits) {
    idle_bits_init_kernel<<<(unsigned)(((c_hi - c_lo) / 32 + 255) / 256), 256, 0, st>>>(
        *f, idle_bits_d, c_lo, c_hi);
    if (kin != st) {  // the kinetics stream reads the map
      cudaEvent_t ev;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      cudaEventRecord(ev, st);
      cudaStreamWaitEvent(kin, ev, 0);
      cudaEventDestroy(ev);
    }
  }
  StencilConst c;
  c.inv_rch2 = a->dt / (tp->rho_c * a->h * a->h);
  c.inv_rch = a->dt / (tp->rho_c * a->h);
  c.inv_rc = a->dt / tp->rho_c;
  c.dk = tp->k_ms - tp->k_p;
  c.t4inf = std::pow(tp->t_inf, 4.0);
  const double kb = tp->k_p + 1.0 * c.dk;
  c.kf = 2.0 * kb * kb / (kb + kb);
  c.dliq = tp->t_liq - tp->t_sol;
  c.src_coef = c.inv_rc * a->src_peak;
  CoupledODE o;
  o.kp = *kp;
  o.dv = make_derived(*kp);
  o.cfg = *cfg;
  o.dt = a->dt;
  o.L = (int)lanes;
  o.rest_ok = kp->t_as_end <= kp->t_sol && kp->t_as_end <= kp->t_as_start && cfg->stuck_tol < 0.5;
  o.hot = nullptr;
  o.sz0 = state_z0;
  o.toff = (state_z0 - a->z_base) * plane;
  const int zchunk = ZCHUNK;
  const int64_t nzu = a->z_end - a->z_begin;
  // split step: rows are whole (nx % 32 == 0) and the row range starts on a
  // hot-word boundary (c_lo % 1024 == 0)
  if (use_tma() && o.rest_ok && scratch_d && c_lo % 1024 == 0) {
    const int64_t row_lo = c_lo / 32, row_hi = c_hi / 32;
    const int64_t nrows_state = row_hi;  // bitmap words cover rows [0, row_hi)
    uint32_t* hot = scratch_d;
    unsigned int* count = reinterpret_cast<unsigned int*>(scratch_d + (nrows_state + 31) / 32);
    uint32_t* list = scratch_d + (nrows_state + 31) / 32 + 4;
    o.hot = hot;
    if (launch_built<2>(tn_d, tn1_d, *a, c, *f, idle_bits_d, o, nzu, zchunk, st)) {
      static int sms = 0;
      if (sms == 0) {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        sms = v;
      }
      if (kin != st) {  // the row kinetics follow the stencil on their own stream
        cudaEvent_t ev;
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        cudaEventRecord(ev, st);
        cudaStreamWaitEvent(kin, ev, 0);
        cudaEventDestroy(ev);
      }
      cudaMemsetAsync(count, 0, sizeof(unsigned int), kin);
      const int64_t thr = (row_hi - row_lo + 3) / 4;
      rows_scan_kernel<<<(unsigned)((thr + 255) / 256), 256, 0, kin>>>(idle_bits_d, hot, row_lo,
                                                                       row_hi, list, count);
      rows_kinetics_kernel<<<(unsigned)(sms * 8), 128, 0, kin>>>(tn_d, tn1_d, *f, idle_bits_d, o,
                                                                 list, count);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        ti64_set_error(std::string("ti64_coupled_step: ") + cudaGetErrorString(e));
        return TI64_ECUDA;
      }
      ti64_set_error("");
      return TI64_OK;
    }
    o.hot = nullptr;  // grid TMA cannot map: the fused cp.async kernel below
  }
  dim3 grid((unsigned)(a->nx / TX), (unsigned)((a->ny + TYT - 1) / TYT),
            (unsigned)((nzu + zchunk - 1) / zchunk));
  if (!use_tma() || !launch_built<1>(tn_d, tn1_d, *a, c, *f, idle_bits_d, o, nzu, zchunk, st))
    built_pipe_kernel<true><<<grid, dim3(TX, TY), 0, st>>>(tn_d, tn1_d, *a, c, zchunk, *f,
                                                          idle_bits_d, o);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    ti64_set_error(std::string("ti64_coupled_step: ") + cudaGetErrorString(e));
    return TI64_ECUDA;
  }
  ti64_set_error("");
  return TI64_OK;
}

extern "C" int64_t ti64_coupled_step(const double* tn_d, double* tn1_d, const ti64_fields* f,
                                     int64_t state_z0, uint32_t* idle_bits_d,
                                     uint32_t* scratch_d, const ti64_thermal* tp,
                                     const ti64_stencil_args* a, const ti64_kparams* kp,
                                     const ti64_icfg* cfg, int64_t lanes, int32_t init_bits,
                                     void* stream) {
  return coupled_step_impl(tn_d, tn1_d, f, state_z0, idle_bits_d, scratch_d, tp, a, kp, cfg, lanes,
                           init_bits, stream, stream);
}

extern "C" int64_t ti64_coupled_step_streams(const double* tn_d, double* tn1_d,
                                             const ti64_fields* f, int64_t state_z0,
                                             uint32_t* idle_bits_d, uint32_t* scratch_d,
                                             const ti64_thermal* tp, const ti64_stencil_args* a,
                                             const ti64_kparams* kp, const ti64_icfg* cfg,
                                             int64_t lanes, int32_t init_bits, void* stream,
                                             void* kin_stream) {
  return coupled_step_impl(tn_d, tn1_d, f, state_z0, idle_bits_d, scratch_d, tp, a, kp, cfg, lanes,
                           init_bits, stream, kin_stream);
}

// _thermal_substeps (thermal.py:290-318): nsub stencil steps from src into
// dst, intermediate results alternating through buf_a / buf_b, src left
// untouched — one C call per macro step instead of one host round trip per
// substep (the build's cool-down steps take up to ~1500 substeps each).
extern "C" int64_t ti64_thermal_substeps(const double* src_d, double* dst_d, double* buf_a_d,
                                         double* buf_b_d, double* rc_d, const uint8_t* state_d,
                                         const ti64_thermal* tp, const ti64_stencil_args* a,
                                         int64_t nsub, void* stream) {
  if (nsub < 1 || (nsub > 1 && (!buf_a_d || (nsub > 2 && !buf_b_d)))) {
    ti64_set_error("ti64_thermal_substeps: bad argument (nsub >= 1, scratch buffers)");
    return TI64_EINVAL;
  }
  const double* cur = src_d;
  for (int64_t s = 0; s < nsub; ++s) {
    double* out = (s == nsub - 1) ? dst_d : ((s % 2 == 0) ? buf_a_d : buf_b_d);
    const int64_t rc = ti64_stencil_step(cur, out, rc_d, state_d, tp, a, stream);
    if (rc != TI64_OK) return rc;
    cur = out;
  }
  return TI64_OK;
}
