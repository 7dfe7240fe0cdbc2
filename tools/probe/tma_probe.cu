// Minimal TMA probe: 3D box load of doubles into smem, copy back.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
constexpr int BX = 36, BY = 18;

__global__ void k(const __grid_constant__ CUtensorMap tmap, double* out, int cx, int cy, int cz, int variant) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* box = reinterpret_cast<double*>(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 6144);
  const unsigned sbox = (unsigned)__cvta_generic_to_shared(box);
  const unsigned sbar = (unsigned)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sbar), "r"(1u));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sbar), "r"(BX * BY * 8) : "memory");
    if (variant == 0)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                   ::"r"(sbox), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(cx), "r"(cy), "r"(cz), "r"(sbar) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                   ::"r"(sbox), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(cx), "r"(cy), "r"(cz), "r"(sbar) : "memory");
  }
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(sbar), "r"(0u) : "memory");
  for (int i = threadIdx.x; i < BX * BY; i += blockDim.x) out[i] = box[i];
}

int main() {
  const int nx = 64, ny = 40, nz = 8;
  std::vector<double> h(nx * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, BX * BY * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  printf("entry %p q=%d\n", p, (int)q);
  EncodeTiledFn enc = (EncodeTiledFn)p;
  CUtensorMap m;
  memset(&m, 0, sizeof m);
  cuuint64_t dims[3] = {nx, ny, nz};
  cuuint64_t strides[2] = {nx * 8, nx * ny * 8};
  cuuint32_t box[3] = {BX, BY, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)r);
  for (int variant = 1; variant >= 0; --variant) {
    for (int t = 0; t < 2; ++t) {
      int cx = t == 0 ? 0 : -2, cy = t == 0 ? 0 : -1, cz = 2;
      k<<<1, 128, 6144 + 64>>>(m, o, cx, cy, cz, variant);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<double> got(BX * BY);
      cudaMemcpy(got.data(), o, BX * BY * 8, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int yy = 0; yy < BY; ++yy)
        for (int xx = 0; xx < BX; ++xx) {
          int gx = cx + xx, gy = cy + yy;
          double want = (gx >= 0 && gx < nx && gy >= 0 && gy < ny) ? h[(cz * ny + gy) * nx + gx] : 0.0;
          if (got[yy * BX + xx] != want) ++bad;
        }
      printf("variant %d start (%d,%d,%d): err=%s bad=%d\n", variant, cx, cy, cz, cudaGetErrorString(e), bad);
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
