// Throughput probe: legacy warp-level mma.sync.m16n8k8 TF32 (fp32 accumulate) on sm_100a.
// Each warp issues independent MMA chains from register operands; reports TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(float* out, int iters) {
  unsigned a[4][4], b[4][2];
  float c[4][4][4];
  for (int i = 0; i < 4; ++i) {
    for (int j = 0; j < 4; ++j) a[i][j] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i + j);
    for (int j = 0; j < 2; ++j) b[i][j] = __float_as_uint(0.5f + threadIdx.x * 1e-3f + i - j);
    for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) c[i][j][k] = 0.f;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[i][j][0]), "+f"(c[i][j][1]), "+f"(c[i][j][2]), "+f"(c[i][j][3])
                     : "r"(a[i][0]), "r"(a[i][1]), "r"(a[i][2]), "r"(a[i][3]), "r"(b[j][0]), "r"(b[j][1]));
  }
  float s = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) s += c[i][j][k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    int blocks = 148 * 2;
    probe<<<blocks, warps * 32>>>(out, 16);
    cudaEvent_t s, e;
    cudaEventCreate(&s); cudaEventCreate(&e);
    cudaEventRecord(s);
    probe<<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    double flops = (double)blocks * warps * iters * 16 * (16.0 * 8 * 8 * 2);
    printf("warps/block %d x %d blocks: %.1f TFLOP/s (tf32 mma.sync m16n8k8)\n", warps, blocks, flops / ms / 1e9);
  }
  return 0;
}
