// Fused AllReduce + elementwise update over peer memory (coll.h).
#include "coll.h"

#include <algorithm>
#include <cstdint>

namespace cg {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// spin until *p >= e; a peer that never arrives fails the launch (10 s watchdog)
__device__ __forceinline__ void wait_ge(const unsigned long long* p, unsigned long long e) {
  const uint64_t t0 = gtimer();
  while (ld_acquire_sys(p) < e)
    if (gtimer() - t0 > 10000000000ull) __trap();
}

// The update chain, op by op in fp32 with IEEE rounding (the generated kernels'
// semantics: no contraction; MAX2 / MIN2 propagate NaN).
__device__ __forceinline__ float apply_chain(const EpiProg& epi, float v, long long i, long long ncol) {
#pragma unroll 1
  for (int e = 0; e < epi.n; ++e) {
    if (epi.op[e] == EPI_RELU) {
      v = v > 0.f ? v : 0.f;
      continue;
    }
    const float x = epi.scalar[e] == 1 ? __ldg(epi.x[e]) : epi.scalar[e] == 2 ? __ldg(epi.x[e] + i) : __ldg(epi.x[e] + i % ncol);
    const float a = epi.swap[e] ? x : v, b = epi.swap[e] ? v : x;
    switch (epi.op[e]) {
      case EPI_ADD: v = __fadd_rn(a, b); break;
      case EPI_SUB: v = __fsub_rn(a, b); break;
      case EPI_MUL: v = __fmul_rn(a, b); break;
      case EPI_DIV: v = __fdiv_rn(a, b); break;
      case EPI_MAX: asm("max.NaN.f32 %0, %1, %2;" : "=f"(v) : "f"(a), "f"(b)); break;
      case EPI_MIN: asm("min.NaN.f32 %0, %1, %2;" : "=f"(v) : "f"(a), "f"(b)); break;
      case EPI_RGRAD: v = a > 0.f ? b : 0.f; break;
    }
  }
  return v;
}

__global__ void __launch_bounds__(256) fused_allreduce_kernel(const __grid_constant__ CollArgs a) {
  const int P = a.nranks;
  unsigned long long* my = a.flags[a.rank];
  unsigned long long e = 0;
  if (P > 1) {
    // arrival: this rank's gradients are final (stream order) -> tell every rank
    e = *reinterpret_cast<volatile unsigned long long*>(my + 128) + 1;
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < P) {
      __threadfence_system();
      st_release_sys(a.flags[threadIdx.x] + a.rank, e);
    }
    if (threadIdx.x == 0)
      for (int r = 0; r < P; ++r) wait_ge(my + r, e);
    __syncthreads();
  }
  const CollSeg& sg = a.segs[blockIdx.y];
  const float* g[kCollMaxRanks];
#pragma unroll
  for (int r = 0; r < kCollMaxRanks; ++r) g[r] = r < P ? a.base[r] + sg.goff : nullptr;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (sg.vec) {
    const long long n4 = sg.n >> 2;
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += stride) {
      float4 s = reinterpret_cast<const float4*>(g[0])[j];
#pragma unroll 1
      for (int r = 1; r < P; ++r) {  // rank order: identical on every rank
        const float4 t = reinterpret_cast<const float4*>(g[r])[j];
        s.x = __fadd_rn(s.x, t.x); s.y = __fadd_rn(s.y, t.y); s.z = __fadd_rn(s.z, t.z); s.w = __fadd_rn(s.w, t.w);
      }
      const long long i = j * 4;
      s.x = apply_chain(sg.epi, s.x, i, sg.ncol);
      s.y = apply_chain(sg.epi, s.y, i + 1, sg.ncol);
      s.z = apply_chain(sg.epi, s.z, i + 2, sg.ncol);
      s.w = apply_chain(sg.epi, s.w, i + 3, sg.ncol);
      reinterpret_cast<float4*>(sg.out)[j] = s;
    }
  } else {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < sg.n; i += stride) {
      float s = g[0][i];
#pragma unroll 1
      for (int r = 1; r < P; ++r) s = __fadd_rn(s, g[r][i]);
      sg.out[i] = apply_chain(sg.epi, s, i, sg.ncol);
    }
  }
  if (P > 1) {
    // departure: the last block to finish tells every rank that this rank has read
    // its gradients, and waits until every rank has read this rank's (so the next
    // iteration may overwrite them), then advances the epoch
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(my + 129, 1ull) == (unsigned long long)gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
    if (last) {
      if (threadIdx.x < P) st_release_sys(a.flags[threadIdx.x] + 64 + a.rank, e);
      if (threadIdx.x == 0) {
        for (int r = 0; r < P; ++r) wait_ge(my + 64 + r, e);
        my[129] = 0;
        *reinterpret_cast<volatile unsigned long long*>(my + 128) = e;
        __threadfence();
      }
    }
  }
}

}  // namespace

bool coll_seg_vec_ok(const CollSeg& s, const float* const* base, int nranks) {
  bool vec = (s.n & 3) == 0 && (reinterpret_cast<uintptr_t>(s.out) & 15) == 0 && (s.goff & 3) == 0;
  for (int r = 0; r < nranks; ++r) vec = vec && (reinterpret_cast<uintptr_t>(base[r]) & 15) == 0;
  for (int e = 0; e < s.epi.n; ++e)  // full-tensor operands are read per element (any alignment)
    (void)e;
  return vec;
}

cudaError_t launch_fused_allreduce(const CollArgs& a, int num_sms, cudaStream_t s) {
  if (a.nranks < 1 || a.nranks > kCollMaxRanks || a.rank < 0 || a.rank >= a.nranks || a.nseg < 1 || a.nseg > 65535)
    return cudaErrorInvalidValue;
  // blocks per segment: about two waves over all segments together
  const int gx = std::max(1, (2 * num_sms * 4 + a.nseg - 1) / a.nseg);
  fused_allreduce_kernel<<<dim3((unsigned)std::min(gx, 1024), (unsigned)a.nseg), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace cg
