// SASS instruction counts of the bit-exact building blocks of one explicit
// point-update (for the FP64-ceiling argument in DESIGN.md §5.1):
//   nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -cubin \
//        -I include -o /tmp/sf.cubin tools/probe/sass_floor.cu
//   cuobjdump -sass /tmp/sf.cubin   (tools/probe/sass_floor.py counts by pipe)
#include "../../paper_2402_17580_b200/csrc/ti64_fastmath.cuh"
using namespace ti64;
extern "C" __global__ void k_pow_floored(const double* b, const double* x, double* o) {
  const int i = threadIdx.x;
  o[i] = pow_floored(b[i], x[i]);
}
extern "C" __global__ void k_exp_core(const double* b, double* o) {
  const int i = threadIdx.x;
  o[i] = exp_core(b[i]);
}
extern "C" __global__ void k_exp_sel(const double* b, double* o) {
  const int i = threadIdx.x;
  o[i] = exp_nn_sel(b[i]);
}
extern "C" __global__ void k_ln_core(const double* b, double* o) {
  const int i = threadIdx.x;
  o[i] = ln_core(b[i]);
}
extern "C" __global__ void k_ddiv(const double* a, const double* b, double* o) {
  const int i = threadIdx.x;
  o[i] = __ddiv_rn(a[i], b[i]);
}
extern "C" __global__ void k_load_store(const double* a, double* o) {
  const int i = threadIdx.x;
  o[i] = a[i];
}
