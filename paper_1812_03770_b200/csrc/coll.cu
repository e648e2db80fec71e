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
  // this segment's descriptor and update chain, staged once per block (read per
  // element from the global table, the chain's fields were a chain of dependent
  // loads per op per element: C3's update 22.6 us for 7.4 MB of gradients)
  __shared__ CollSeg sseg;
  if (threadIdx.x == 0) sseg = a.segs[blockIdx.y];
  __syncthreads();
  const CollSeg& sg = sseg;
  const bool ncol32 = sg.ncol < (1ll << 31) && sg.n < (1ll << 31);
  const float* g[kCollMaxRanks];
#pragma unroll
  for (int r = 0; r < kCollMaxRanks; ++r) g[r] = r < P ? a.base[r] + sg.goff : nullptr;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (sg.vec) {
    // CU float4 vectors per thread per iteration (grid-stride, coalesced), every load
    // of a step issued before its arithmetic: the gradient vectors, then per chain op
    // its operand vectors (a full-tensor operand such as W in W - lr * g) -- one HBM
    // latency per step for all of them (one vector at a time was two serialised
    // latencies per vector: C3's update 13 -> ~4 us)
    constexpr int CU = 4;
    const long long n4 = sg.n >> 2;
    for (long long j0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; j0 < n4; j0 += CU * stride) {
      float v[CU][4];
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const long long j = j0 + u * stride;
        float4 t = j < n4 ? reinterpret_cast<const float4*>(g[0])[j] : make_float4(0.f, 0.f, 0.f, 0.f);
        v[u][0] = t.x; v[u][1] = t.y; v[u][2] = t.z; v[u][3] = t.w;
      }
#pragma unroll 1
      for (int r = 1; r < P; ++r) {  // rank order: identical on every rank
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const long long j = j0 + u * stride;
          if (j >= n4) continue;
          const float4 t = reinterpret_cast<const float4*>(g[r])[j];
          v[u][0] = __fadd_rn(v[u][0], t.x); v[u][1] = __fadd_rn(v[u][1], t.y);
          v[u][2] = __fadd_rn(v[u][2], t.z); v[u][3] = __fadd_rn(v[u][3], t.w);
        }
      }
#pragma unroll 1
      for (int e = 0; e < sg.epi.n; ++e) {
        const int op = sg.epi.op[e], sc = sg.epi.scalar[e], sw = sg.epi.swap[e];
        const float* x = sg.epi.x[e];
        float xe[CU][4];
#pragma unroll
        for (int u = 0; u < CU; ++u) {  // (vec: a float4 never straddles a row, coll_seg_vec_ok)
          const long long j = j0 + u * stride;
          const long long i = j * 4;
          if (op == EPI_RELU || j >= n4) {
            xe[u][0] = xe[u][1] = xe[u][2] = xe[u][3] = 0.f;
          } else if (sc == 1) {
            xe[u][0] = xe[u][1] = xe[u][2] = xe[u][3] = __ldg(x);
          } else {
            const long long off = sc == 2 ? i : ncol32 ? (long long)((unsigned)i % (unsigned)sg.ncol) : i % sg.ncol;
            const float4 t = __ldg(reinterpret_cast<const float4*>(x + off));
            xe[u][0] = t.x; xe[u][1] = t.y; xe[u][2] = t.z; xe[u][3] = t.w;
          }
        }
#pragma unroll
        for (int u = 0; u < CU; ++u) epi_apply<4>(v[u], op, sw, xe[u]);
      }
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const long long j = j0 + u * stride;
        if (j < n4) reinterpret_cast<float4*>(sg.out)[j] = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
      }
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
  for (int e = 0; e < s.epi.n; ++e) {  // vector operands: 16-byte loads; a column float4 within one row
    if (s.epi.op[e] == EPI_RELU || s.epi.scalar[e] == 1) continue;
    vec = vec && (reinterpret_cast<uintptr_t>(s.epi.x[e]) & 15) == 0;
    if (s.epi.scalar[e] == 0) vec = vec && (s.ncol & 3) == 0;
  }
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
