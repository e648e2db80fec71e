// tcgen05.mma (kind::tf32, cta_group::1, M = 128) issue/execute rate vs N, with A
// from TMEM (.kind::tf32 [d], [a_tmem], b_desc) or A from shared memory (SS).
// One CTA per SM, one warp issues `reps` MMAs back to back into one accumulator,
// commits, waits; cycles per MMA = elapsed / reps.  Values are garbage (rate only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

template <int N, bool TS>
__global__ void probe(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = __shfl_sync(0xffffffffu, slot, 0);
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t sb = smem_u32(smem);
    const uint64_t bd = sdesc(sb, 16, 1024, 2);
    const uint64_t ad = sdesc(sb + 32768, 16, 1024, 2);
    const uint32_t a_t = tm + 256;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (TS)
        asm volatile(
            "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
            " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n}\n" ::"r"(tm),
            "r"(a_t), "l"(bd), "r"(idesc));
      else
        asm volatile(
            "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
            " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n}\n" ::"r"(tm),
            "l"(ad), "l"(bd), "r"(idesc));
    }
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&bar))
        : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done)
                   : "r"(smem_u32(&bar))
                   : "memory");
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, bool TS>
void run(int reps) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<N, TS><<<148, 128, 64 * 1024>>>(reps, d);
  probe<N, TS><<<148, 128, 64 * 1024>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%s N=%3d: %.1f cycles per MMA (floor 128*N/256 = %d)  %s\n", TS ? "A=TMEM" : "A=SMEM", N, avg / reps,
         128 * N / 256, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  const int reps = 4096;
  run<16, true>(reps); run<32, true>(reps); run<64, true>(reps); run<128, true>(reps); run<256, true>(reps);
  run<16, false>(reps); run<32, false>(reps); run<64, false>(reps); run<128, false>(reps); run<256, false>(reps);
  return 0;
}
