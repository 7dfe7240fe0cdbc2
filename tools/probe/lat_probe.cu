// Dependent-chain latency probe (one warp): cycles per dependent op for
// DFMA, DADD, DMUL, DSETP+select, MUFU.RCP64H, __ddiv_rn, __dsqrt_rn, a
// warp vote, and fast_exp / ln cores.  nvcc -arch=sm_100a -O3 --fmad=false
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2402_17580_b200/csrc/ti64_fastmath.cuh"
using namespace ti64;

template <int OP>
__global__ void chain(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = __fma_rn(x, y, 1e-7);
    if (OP == 1) x = __dadd_rn(x, 1e-7);
    if (OP == 2) x = __dmul_rn(x, y);
    if (OP == 3) x = x > 0.5 ? __dadd_rn(x, 1e-9) : __dsub_rn(x, 1e-9);
    if (OP == 4) x = __ddiv_rn(1.0, x);
    if (OP == 5) x = __dsqrt_rn(x);
    if (OP == 6) x = __dadd_rn(x, __all_sync(0xffffffffu, x > 0.0) ? 1e-9 : 2e-9);
    if (OP == 7) x = __dmul_rn(fast_exp(__dmul_rn(x, -1e-3)), 1.0000001);
    if (OP == 8) x = __dadd_rn(fast_ln(x), 1.5);
    if (OP == 9) x = pow_floored(x, 0.999);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { *cyc = t1 - t0; }
  out[threadIdx.x] = x;
}

int main() {
  double* d; long long* c; cudaMalloc(&d, 1024 * 8); cudaMalloc(&c, 8);
  const char* names[] = {"DFMA", "DADD", "DMUL", "DSETP+sel+DADD", "ddiv_rn", "dsqrt_rn",
                         "vote+sel+DADD", "fast_exp+DMUL", "fast_ln+DADD", "pow_floored"};
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
#define RUN(K) { chain<K><<<1, 32>>>(d, c, 0.75, n); long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); \
                 if (rep) printf("%-18s %7.1f cycles per op\n", names[K], (double)h / n); }
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9)
  }
  return 0;
}
