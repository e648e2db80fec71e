// Probe: 3-D tiled TMA load with negative start coordinates (zero-filled padding)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m, float* out, int G, int c0, int bw) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar), d = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(G * bw * bw * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(d),
                 "l"(&m), "r"(c0), "r"(c0), "r"(0), "r"(b) : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(b) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * 1024; i += blockDim.x) out[i] = sm[i];
}
int main(int argc, char** argv) {
  const int c0 = atoi(argv[1]), bw = atoi(argv[2]);
  const int n = 3, G = 2;
  float h[n * 784];
  for (int i = 0; i < n * 784; ++i) h[i] = i + 1;
  float *x, *o;
  cudaMalloc(&x, sizeof(h)); cudaMalloc(&o, G * 1024 * 4);
  cudaMemcpy(x, h, sizeof(h), cudaMemcpyHostToDevice);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[3] = {28, 28, n}; cuuint64_t str[2] = {28 * 4, 784 * 4};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bw, (cuuint32_t)G}, es[3] = {1, 1, 1};
  CUresult r = ((Enc)p)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  k<<<1, 128, G * 4096 + 1024>>>(m, o, G, c0, bw);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  float ho[G * 1024];
  cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int g = 0; g < G; ++g)
    for (int r2 = 0; r2 < 32; ++r2)
      for (int c = 0; c < 32; ++c) {
        int ih = r2 - 2, iw = c - 2;
        float want = (ih >= 0 && ih < 28 && iw >= 0 && iw < 28) ? h[g * 784 + ih * 28 + iw] : 0.f;
        bad += ho[g * 1024 + r2 * 32 + c] != want;
      }
  printf("bad %d\n", bad);
}
