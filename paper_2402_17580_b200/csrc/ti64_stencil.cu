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
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "../../include/ti64_b200.h"
#include "ti64_fastmath.cuh"

using namespace ti64;

namespace {

constexpr int STATE_INACTIVE = 0;
constexpr int STATE_POWDER = 1;


struct StencilConst {
  double inv_rch2, inv_rch, inv_rc, dk, t4inf, kf, dliq;
  double src_coef;  // inv_rc * src_peak  (association of thermal.py:261)
};

__device__ __forceinline__ double clip01(double g) { return g < 0.0 ? 0.0 : (g > 1.0 ? 1.0 : g); }

// top-layer Gaussian source term (thermal.py:255-261)
__device__ __forceinline__ double add_source(double t_new, int64_t x, int64_t y,
                                             const ti64_stencil_args& a,
                                             const StencilConst& c) {
  const double xc = __dmul_rn(__dadd_rn((double)x, 0.5), a.h);
  const double yc = __dmul_rn(__dadd_rn((double)y, 0.5), a.h);
  const double dx = __dsub_rn(xc, a.beam_x), dy = __dsub_rn(yc, a.beam_y);
  const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  const double arg = __dmul_rn(__dmul_rn(-2.0, r2), a.src_r2inv);
  if (arg > -40.0) t_new = __dadd_rn(t_new, __dmul_rn(c.src_coef, fast_exp(arg)));
  return t_new;
}

constexpr int TX = 32, TY = 8;

// Arrays hold global planes [z_base, z_base + nz_stored); the block updates
// global planes [z0, z1) of its z-chunk.  z-1 / z / z+1 ride in registers, the
// current plane (+ x/y halo) is staged in shared memory.
__global__ void __launch_bounds__(TX* TY) stencil_built_kernel(const double* __restrict__ src,
                                                             double* __restrict__ dst,
                                                             ti64_stencil_args a,
                                                             StencilConst c, int zchunk) {
  __shared__ double pl[TY + 2][TX + 2];
  const int64_t nx = a.nx, ny = a.ny, nz = a.nz;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t x = (int64_t)blockIdx.x * TX + tx;
  const int64_t y = (int64_t)blockIdx.y * TY + ty;
  const int64_t z0 = a.z_begin + (int64_t)blockIdx.z * zchunk;
  int64_t z1 = z0 + zchunk;
  if (z1 > a.z_end) z1 = a.z_end;
  const bool in = x < nx && y < ny;
  const int64_t plane = nx * ny;
  const int64_t col = y * nx + x;
  const double* sp = src + (-a.z_base) * plane + col;  // sp[z*plane] = T(z, y, x)
  double* dp = dst + (-a.z_base) * plane + col;
  const double kf = c.kf;
  double tm = 0.0, t0 = 0.0, tp = 0.0;
  if (in && z0 < z1) {
    t0 = sp[z0 * plane];
    if (z0 > 0) tm = sp[(z0 - 1) * plane];
  }
  for (int64_t z = z0; z < z1; ++z) {
    if (in && z + 1 < nz) tp = sp[(z + 1) * plane];
    __syncthreads();
    if (in) pl[ty + 1][tx + 1] = t0;
    if (tx == 0 && x > 0 && y < ny) pl[ty + 1][0] = sp[z * plane - 1];
    if (tx == TX - 1 && x + 1 < nx && y < ny) pl[ty + 1][TX + 1] = sp[z * plane + 1];
    if (ty == 0 && y > 0 && x < nx) pl[0][tx + 1] = sp[z * plane - nx];
    if (ty == TY - 1 && y + 1 < ny && x < nx) pl[TY + 1][tx + 1] = sp[z * plane + nx];
    __syncthreads();
    if (in) {
      double flux = 0.0;
      if (x > 0) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(pl[ty + 1][tx], t0)));
      if (x + 1 < nx) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(pl[ty + 1][tx + 2], t0)));
      if (y > 0) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(pl[ty][tx + 1], t0)));
      if (y + 1 < ny) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(pl[ty + 2][tx + 1], t0)));
      if (z > 0) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(tm, t0)));
      if (z + 1 < nz) flux = __dadd_rn(flux, __dmul_rn(kf, __dsub_rn(tp, t0)));
      double t_new = __dadd_rn(t0, __dmul_rn(c.inv_rch2, flux));
      if (a.source_on != 0 && z == a.z_top - 1) t_new = add_source(t_new, x, y, a, c);
      if (a.bc_bottom_on != 0 && z == 0) t_new = a.bc_bottom;  // thermal.py:274-278
      dp[z * plane] = t_new;
    }
    tm = t0;
    t0 = tp;
  }
}

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
  if (a.source_on != 0 && z == a.z_top - 1) t_new = add_source(t_new, x, y, a, c);
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

}  // namespace

void ti64_set_error(const std::string& msg);  // ti64_kernels.cu

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
    const int zchunk = 16;
    dim3 grid((unsigned)((a->nx + TX - 1) / TX), (unsigned)((a->ny + TY - 1) / TY),
              (unsigned)((nzu + zchunk - 1) / zchunk));
    stencil_built_kernel<<<grid, dim3(TX, TY), 0, st>>>(src_d, dst_d, *a, c, zchunk);
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
