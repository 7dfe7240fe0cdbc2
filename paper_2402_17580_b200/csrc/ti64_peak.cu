// ti64_peak.cu — roofline denominators measured on the box:
//  * a dependent-free DFMA stream (FP64 peak; MEASURED_PEAKS.json carries no
//    FP64 figure): 8 independent FMA chains per thread, full occupancy;
//  * a DAXPY stream update y += a x (24 B per element), the GPU form of the
//    reference's bandwidth baseline (bench.py:83-108 measure_bandwidth).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/ti64_b200.h"

void ti64_set_error(const std::string& msg);

namespace {
__global__ void __launch_bounds__(256) dfma_kernel(double* out, int64_t iters, double b,
                                                  double c) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-3, a2 = a0 + 2e-3, a3 = a0 + 3e-3;
  double a4 = a0 + 4e-3, a5 = a0 + 5e-3, a6 = a0 + 6e-3, a7 = a0 + 7e-3;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 = __fma_rn(a0, b, c); a1 = __fma_rn(a1, b, c); a2 = __fma_rn(a2, b, c);
      a3 = __fma_rn(a3, b, c); a4 = __fma_rn(a4, b, c); a5 = __fma_rn(a5, b, c);
      a6 = __fma_rn(a6, b, c); a7 = __fma_rn(a7, b, c);
    }
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}
// y[i] += a * x[i] with 2 elements per thread (16-byte accesses); no FMA
// contraction (--fmad=false), as the reference's numba loop
__global__ void __launch_bounds__(256) daxpy_kernel(double* __restrict__ y,
                                                   const double* __restrict__ x, double a,
                                                   int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * i < n; i += stride) {
    if (2 * i + 1 < n) {
      const double2 xv = reinterpret_cast<const double2*>(x)[i];
      double2 yv = reinterpret_cast<double2*>(y)[i];
      yv.x = yv.x + a * xv.x;
      yv.y = yv.y + a * xv.y;
      reinterpret_cast<double2*>(y)[i] = yv;
    } else {
      y[2 * i] = y[2 * i] + a * x[2 * i];
    }
  }
}
}  // namespace

extern "C" int64_t ti64_bench_daxpy(double* y_d, const double* x_d, double a, int64_t n,
                                    void* stream) {
  if (!y_d || !x_d || n < 0 || ((reinterpret_cast<uintptr_t>(y_d) |
                                 reinterpret_cast<uintptr_t>(x_d)) & 15)) {
    ti64_set_error("ti64_bench_daxpy: bad argument (16-byte aligned device arrays)");
    return TI64_EINVAL;
  }
  if (n == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n / 2 + 255) / 256;
  const int blocks = (int)(want < (int64_t)sms * 8 ? want : (int64_t)sms * 8);
  daxpy_kernel<<<blocks < 1 ? 1 : blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      y_d, x_d, a, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    ti64_set_error(std::string("ti64_bench_daxpy: ") + cudaGetErrorString(e));
    return TI64_ECUDA;
  }
  return 24 * n;  // bytes moved (2 loads + 1 store of 8 B)
}

extern "C" int64_t ti64_bench_dfma(double* scratch_d, int64_t iters, int32_t blocks,
                                   void* stream) {
  if (!scratch_d || iters < 1 || blocks < 1) {
    ti64_set_error("ti64_bench_dfma: bad argument");
    return TI64_EINVAL;
  }
  dfma_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      scratch_d, iters, 0.9999999999, 1e-12);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    ti64_set_error(std::string("ti64_bench_dfma: ") + cudaGetErrorString(e));
    return TI64_ECUDA;
  }
  // flops per launch: blocks * 256 threads * iters * 4 * 8 FMAs * 2
  return (int64_t)blocks * 256 * iters * 64;
}
