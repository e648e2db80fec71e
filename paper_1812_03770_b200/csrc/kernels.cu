// Precompiled sm_100a kernels: update-edge copy, copy, split-reduction finalize,
// SIMT dot, and the NHWC conv / pool / concat family.
//
// Definitions follow SURVEY §8(c) c1-defs (the oracle's op semantics):
//   CONV2D            y[n,ho,wo,co] = sum_{kh,kw,ci} x[n, ho*sh+kh-pt, wo*sw+kw-pl, ci] w[kh,kw,ci,co]
//   CONV2D_BWD_INPUT  dx[n,h,w,ci]  = sum dy[n,ho,wo,co] w[kh,kw,ci,co], h = ho*sh+kh-pt, w = wo*sw+kw-pl
//   CONV2D_BWD_KERNEL dw[kh,kw,ci,co] = sum_{n,ho,wo} x[n, ho*sh+kh-pt, wo*sw+kw-pl, ci] dy[n,ho,wo,co]
//   MAXPOOL2D_BWD     each window's dy goes to its FIRST maximal element (kh outer, kw inner)
//   AVGPOOL2D         mean over in-bounds window elements
// All accumulations are sequential per output in a fixed order; no atomics, so
// results are run-to-run bit-stable.
#include "kernels.h"

#include "dot_tc.h"  // EpiProg / epi_run (f2 pooling fusion)

#include <algorithm>
#include <climits>
#include <type_traits>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <set>
#include <tuple>

namespace cg {

cudaError_t smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({fn, dev, bytes})) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({fn, dev, bytes});
  return e;
}

namespace {

__global__ void update_copy_kernel(const CopyDesc* __restrict__ d) {
  const CopyDesc e = d[blockIdx.y];
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if ((e.n & 3) == 0) {
    const float4* s = reinterpret_cast<const float4*>(e.src);
    float4* o = reinterpret_cast<float4*>(e.dst);
    for (long long i = t; i < (e.n >> 2); i += stride) o[i] = s[i];
  } else {
    for (long long i = t; i < e.n; i += stride) e.dst[i] = e.src[i];
  }
}

__global__ void copy_kernel(const float* __restrict__ src, float* __restrict__ dst, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if ((n & 3) == 0) {
    const float4* s = reinterpret_cast<const float4*>(src);
    float4* o = reinterpret_cast<float4*>(dst);
    for (long long i = t; i < (n >> 2); i += stride) o[i] = s[i];
  } else {
    for (long long i = t; i < n; i += stride) dst[i] = src[i];
  }
}

__global__ void reduce_finalize_kernel(const float* __restrict__ ws, float* __restrict__ out, long long oi, long long S,
                                       int op) {
  long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= oi) return;
  float acc = ws[j];
  long long s = 1;
  for (; s + 4 <= S; s += 4) {  // four partials in flight, combined in s order
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ws[(s + u) * oi + j];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (op == 0) acc = __fadd_rn(acc, v[u]);
      else asm("max.NaN.f32 %0, %0, %1;" : "+f"(acc) : "f"(v[u]));  // NaN-propagating, as numpy max
    }
  }
  for (; s < S; ++s) {
    float v = ws[s * oi + j];
    if (op == 0) acc = __fadd_rn(acc, v);
    else asm("max.NaN.f32 %0, %0, %1;" : "+f"(acc) : "f"(v));
  }
  out[j] = acc;
}

// reduce_finalize_kernel on 4 consecutive outputs per thread (oi % 4 == 0).
__global__ void reduce_finalize4_kernel(const float4* __restrict__ ws, float4* __restrict__ out, long long oi4,
                                        long long S, int op) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= oi4) return;
  float4 acc = ws[j];
  auto comb = [&](float& a, float v) {
    if (op == 0) a = __fadd_rn(a, v);
    else asm("max.NaN.f32 %0, %0, %1;" : "+f"(a) : "f"(v));
  };
  long long s = 1;
  for (; s + 2 <= S; s += 2) {
    const float4 v0 = ws[s * oi4 + j], v1 = ws[(s + 1) * oi4 + j];
    comb(acc.x, v0.x), comb(acc.y, v0.y), comb(acc.z, v0.z), comb(acc.w, v0.w);
    comb(acc.x, v1.x), comb(acc.y, v1.y), comb(acc.z, v1.z), comb(acc.w, v1.w);
  }
  if (s < S) {
    const float4 v = ws[s * oi4 + j];
    comb(acc.x, v.x), comb(acc.y, v.y), comb(acc.z, v.z), comb(acc.w, v.w);
  }
  out[j] = acc;
}

// Few outputs, many partials: one block per output, each thread a strided
// sequential sum, then a fixed-order shared-memory tree (deterministic).
__global__ void __launch_bounds__(256) reduce_finalize_tree_kernel(const float* __restrict__ ws, float* __restrict__ out,
                                                                   long long oi, long long S, int op) {
  __shared__ float sm[256];
  const long long j = blockIdx.x;
  float acc = op == 0 ? 0.f : -__int_as_float(0x7f800000);
  for (long long s = threadIdx.x; s < S; s += 256) {
    const float v = ws[s * oi + j];
    if (op == 0) acc = __fadd_rn(acc, v);
    else asm("max.NaN.f32 %0, %0, %1;" : "+f"(acc) : "f"(v));
  }
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int h = 128; h >= 1; h /= 2) {
    if (threadIdx.x < h) {
      float a = sm[threadIdx.x], b = sm[threadIdx.x + h];
      if (op == 0) a = __fadd_rn(a, b);
      else asm("max.NaN.f32 %0, %0, %1;" : "+f"(a) : "f"(b));
      sm[threadIdx.x] = a;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = sm[0];
}

// One warp per output: lanes take strided partials, fixed-order shuffle tree.
__global__ void __launch_bounds__(256) reduce_finalize_warp_kernel(const float* __restrict__ ws, float* __restrict__ out,
                                                                   long long oi, long long S, int op) {
  const long long j = (long long)blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (j >= oi) return;
  float acc = op == 0 ? 0.f : -__int_as_float(0x7f800000);
  long long s = lane;
  for (; s + 96 < S; s += 128) {  // four strided partials in flight, combined in s order
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ws[(s + 32 * u) * oi + j];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (op == 0) acc = __fadd_rn(acc, v[u]);
      else asm("max.NaN.f32 %0, %0, %1;" : "+f"(acc) : "f"(v[u]));
    }
  }
  for (; s < S; s += 32) {
    const float v = ws[s * oi + j];
    if (op == 0) acc = __fadd_rn(acc, v);
    else asm("max.NaN.f32 %0, %0, %1;" : "+f"(acc) : "f"(v));
  }
#pragma unroll
  for (int o = 16; o >= 1; o /= 2) {
    const float v = __shfl_xor_sync(0xffffffffu, acc, o);
    if (op == 0) acc = __fadd_rn(acc, v);
    else asm("max.NaN.f32 %0, %0, %1;" : "+f"(acc) : "f"(v));
  }
  if (lane == 0) out[j] = acc;
}

// 64x64 output tile, 16-deep k slab, 256 threads x (4x4) outputs, fp32 FFMA
__global__ void __launch_bounds__(256) dot_simt_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                      float* __restrict__ C, int M, int N, int K, int ta, int tb) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tr = tid / 16, tc = tid % 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = tid; e < 64 * 16; e += 256) {
      int mm, kk;
      if (ta) { kk = e / 64; mm = e % 64; } else { mm = e / 16; kk = e % 16; }
      int gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < M && gk < K) v = ta ? A[(long long)gk * M + gm] : A[(long long)gm * K + gk];
      As[kk][mm] = v;
      int nn;
      if (tb) { nn = e / 16; kk = e % 16; } else { kk = e / 64; nn = e % 64; }
      int gn = n0 + nn;
      gk = k0 + kk;
      v = 0.f;
      if (gn < N && gk < K) v = tb ? B[(long long)gn * K + gk] : B[(long long)gk * N + gn];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tr * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tc * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gm = m0 + tr * 4 + i, gn = n0 + tc * 4 + j;
      if (gm < M && gn < N) C[(long long)gm * N + gn] = acc[i][j];
    }
}

template <typename I>
__global__ void conv_fwd_kernel(const float* __restrict__ x, const float* __restrict__ w, float* __restrict__ y, ConvGeom g,
                                I total) {
  for (I t = (I)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
    int co = (int)(t % g.co);
    I q = t / g.co;
    int wo = (int)(q % g.wo);
    q /= g.wo;
    int ho = (int)(q % g.ho);
    int n = (int)(q / g.ho);
    float acc = 0.f;
    for (int kh = 0; kh < g.kh; ++kh) {
      int hi = ho * g.sh + kh - g.pt;
      if (hi < 0 || hi >= g.h) continue;
      for (int kw = 0; kw < g.kw; ++kw) {
        int wi = wo * g.sw + kw - g.pl;
        if (wi < 0 || wi >= g.w) continue;
        const float* xp = x + (((long long)n * g.h + hi) * g.w + wi) * g.ci;
        const float* wp = w + ((long long)(kh * g.kw + kw) * g.ci) * g.co + co;
        for (int ci = 0; ci < g.ci; ++ci) acc = fmaf(xp[ci], wp[(long long)ci * g.co], acc);
      }
    }
    y[t] = acc;
  }
}

template <typename I>
__global__ void conv_bwd_input_kernel(const float* __restrict__ dy, const float* __restrict__ w, float* __restrict__ dx,
                                      ConvGeom g, I total) {
  for (I t = (I)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
    int ci = (int)(t % g.ci);
    I q = t / g.ci;
    int wi = (int)(q % g.w);
    q /= g.w;
    int hi = (int)(q % g.h);
    int n = (int)(q / g.h);
    float acc = 0.f;
    for (int kh = 0; kh < g.kh; ++kh) {
      int hs = hi + g.pt - kh;
      if (hs < 0 || hs % g.sh) continue;
      int ho = hs / g.sh;
      if (ho >= g.ho) continue;
      for (int kw = 0; kw < g.kw; ++kw) {
        int ws_ = wi + g.pl - kw;
        if (ws_ < 0 || ws_ % g.sw) continue;
        int wo = ws_ / g.sw;
        if (wo >= g.wo) continue;
        const float* dyp = dy + (((long long)n * g.ho + ho) * g.wo + wo) * g.co;
        const float* wp = w + ((long long)(kh * g.kw + kw) * g.ci + ci) * g.co;
        for (int co = 0; co < g.co; ++co) acc = fmaf(dyp[co], wp[co], acc);
      }
    }
    dx[t] = acc;
  }
}

// partial[s][kh,kw,ci,co] over positions p in [s*chunk, (s+1)*chunk) of (n, ho, wo)
__global__ void conv_bwd_kernel_kernel(const float* __restrict__ x, const float* __restrict__ dy, float* __restrict__ part,
                                       ConvGeom g, long long P, long long chunk, int outs) {
  int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= outs) return;
  int co = o % g.co;
  int r = o / g.co;
  int ci = r % g.ci;
  r /= g.ci;
  int kw = r % g.kw;
  int kh = r / g.kw;
  long long p0 = (long long)blockIdx.y * chunk, p1 = min(p0 + chunk, P);
  float acc = 0.f;
  for (long long p = p0; p < p1; ++p) {
    int wo = (int)(p % g.wo);
    long long q = p / g.wo;
    int ho = (int)(q % g.ho);
    int n = (int)(q / g.ho);
    int hi = ho * g.sh + kh - g.pt, wi = wo * g.sw + kw - g.pl;
    if (hi < 0 || hi >= g.h || wi < 0 || wi >= g.w) continue;
    acc = fmaf(x[(((long long)n * g.h + hi) * g.w + wi) * g.ci + ci], dy[p * g.co + co], acc);
  }
  part[(long long)blockIdx.y * outs + o] = acc;
}

template <typename I>
__global__ void maxpool_kernel(const float* __restrict__ x, float* __restrict__ y, ConvGeom g, I total) {
  for (I t = (I)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
    int c = (int)(t % g.co);
    I q = t / g.co;
    int wo = (int)(q % g.wo);
    q /= g.wo;
    int ho = (int)(q % g.ho);
    int n = (int)(q / g.ho);
    float m = -__int_as_float(0x7f800000);
    for (int kh = 0; kh < g.kh; ++kh) {
      int hi = ho * g.sh + kh - g.pt;
      if (hi < 0 || hi >= g.h) continue;
      for (int kw = 0; kw < g.kw; ++kw) {
        int wi = wo * g.sw + kw - g.pl;
        if (wi < 0 || wi >= g.w) continue;
        asm("max.NaN.f32 %0, %0, %1;" : "+f"(m) : "f"(x[(((long long)n * g.h + hi) * g.w + wi) * g.co + c]));
      }
    }
    y[t] = m;
  }
}

template <typename I>
__global__ void maxpool_bwd_kernel(const float* __restrict__ x, const float* __restrict__ dy, float* __restrict__ dx,
                                   ConvGeom g, I total) {
  for (I t = (I)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
    int c = (int)(t % g.co);
    I q = t / g.co;
    int wi0 = (int)(q % g.w);
    q /= g.w;
    int hi0 = (int)(q % g.h);
    int n = (int)(q / g.h);
    float acc = 0.f;
    // windows containing (hi0, wi0), in ascending (ho, wo) order
    int ho_lo = max(0, (hi0 + g.pt - g.kh + g.sh) / g.sh), ho_hi = min(g.ho - 1, (hi0 + g.pt) / g.sh);
    int wo_lo = max(0, (wi0 + g.pl - g.kw + g.sw) / g.sw), wo_hi = min(g.wo - 1, (wi0 + g.pl) / g.sw);
    if (hi0 + g.pt - g.kh + g.sh < 0) ho_lo = 0;
    if (wi0 + g.pl - g.kw + g.sw < 0) wo_lo = 0;
    for (int ho = ho_lo; ho <= ho_hi; ++ho)
      for (int wo = wo_lo; wo <= wo_hi; ++wo) {
        // first maximal element of window (ho, wo)
        float m = -__int_as_float(0x7f800000);
        int bh = -1, bw = -1;
        for (int kh = 0; kh < g.kh; ++kh) {
          int hi = ho * g.sh + kh - g.pt;
          if (hi < 0 || hi >= g.h) continue;
          for (int kw = 0; kw < g.kw; ++kw) {
            int wi = wo * g.sw + kw - g.pl;
            if (wi < 0 || wi >= g.w) continue;
            float v = x[(((long long)n * g.h + hi) * g.w + wi) * g.co + c];
            if (v > m || bh < 0) { m = v; bh = hi; bw = wi; }
          }
        }
        if (bh == hi0 && bw == wi0) acc = __fadd_rn(acc, dy[(((long long)n * g.ho + ho) * g.wo + wo) * g.co + c]);
      }
    dx[t] = acc;
  }
}

// Non-overlapping windows that tile the input exactly (kh == sh, kw == sw, no
// padding, h == ho*sh, w == wo*sw): one thread per window routes dy to the first
// maximal element (kh outer, kw inner) and writes zeros elsewhere — a scatter
// without conflicts, each element written exactly once.
template <typename I>
__global__ void maxpool_bwd_tiled_kernel(const float* __restrict__ x, const float* __restrict__ dy, float* __restrict__ dx,
                                         ConvGeom g, I total) {
  for (I t = (I)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
    int c = (int)(t % g.co);
    I q = t / g.co;
    int wo = (int)(q % g.wo);
    q /= g.wo;
    int ho = (int)(q % g.ho);
    int n = (int)(q / g.ho);
    const long long base = ((long long)n * g.h + ho * g.sh) * g.w + wo * g.sw;
    float m = -__int_as_float(0x7f800000);
    int best = -1;
    for (int kh = 0; kh < g.kh; ++kh)
      for (int kw = 0; kw < g.kw; ++kw) {
        const float v = x[(base + (long long)kh * g.w + kw) * g.co + c];
        if (v > m || best < 0) { m = v; best = kh * g.kw + kw; }
      }
    const float d = dy[t];
    for (int kh = 0; kh < g.kh; ++kh)
      for (int kw = 0; kw < g.kw; ++kw)
        dx[(base + (long long)kh * g.w + kw) * g.co + c] = (kh * g.kw + kw == best) ? d : 0.f;
  }
}

// 2 x 2 stride-2 VALID max pool with few channels (C4: C = 6, 16).  Thread =
// (output pixel, V channels) so neighbouring lanes read neighbouring 8- / 16-byte
// pieces of the same window rows.  Same combine order as maxpool_kernel (bit-identical).
// With pro.n > 0 (f2 pooling fusion, even H and W) the window values are first
// computed from x by the producer's elementwise chain and stored to xo (every
// element of xo lies in exactly one window), then pooled.  xo may alias x (an
// in-place chain): each element is read and written by the same thread, in order.
// codes != NULL: also record, per (output pixel, channel), the window position the
// backward pass routes the gradient to (maxpool2_bwd_kernel's rule on the same
// values), so the backward reads one byte instead of the four window values.
template <int C, int V>
__global__ void maxpool2_fwd_kernel(const float* x, float* __restrict__ y, ConvGeom g, int total, float* xo,
                                    const __grid_constant__ EpiProg pro, unsigned char* __restrict__ codes) {
  using VT = typename std::conditional<V == 4, float4, float2>::type;
  constexpr int Q = C / V;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int p = t / Q, c = (t - p * Q) * V;
    const int wo = p % g.wo, q = p / g.wo, ho = q % g.ho, n = q / g.ho;
    const size_t o0 = (((size_t)n * g.h + 2 * ho) * g.w + 2 * wo) * C + c, o1 = o0 + (size_t)g.w * C;
    VT w4[4];
    w4[0] = *reinterpret_cast<const VT*>(x + o0);
    w4[1] = *reinterpret_cast<const VT*>(x + o0 + C);
    w4[2] = *reinterpret_cast<const VT*>(x + o1);
    w4[3] = *reinterpret_cast<const VT*>(x + o1 + C);
    if (pro.n) {
      const size_t off[4] = {o0, o0 + C, o1, o1 + C};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float v[V];
#pragma unroll
        for (int e = 0; e < V; ++e) v[e] = reinterpret_cast<const float*>(&w4[k])[e];
        epi_run<V>(pro, v, (long long)off[k], c);
#pragma unroll
        for (int e = 0; e < V; ++e) reinterpret_cast<float*>(&w4[k])[e] = v[e];
        if (xo) *reinterpret_cast<VT*>(xo + off[k]) = w4[k];  // (NULL: no reader needs the values)
      }
    }
    const float* wf = reinterpret_cast<const float*>(w4);
    VT o;
    float* of = reinterpret_cast<float*>(&o);
#pragma unroll
    for (int e = 0; e < V; ++e) {
      float m = -__int_as_float(0x7f800000);
#pragma unroll
      for (int k = 0; k < 4; ++k) asm("max.NaN.f32 %0, %0, %1;" : "+f"(m) : "f"(wf[k * V + e]));
      of[e] = m;
    }
    *reinterpret_cast<VT*>(y + (size_t)p * C + c) = o;
    if (codes) {
      unsigned packed = 0;
#pragma unroll
      for (int e = 0; e < V; ++e) {
        float m = -__int_as_float(0x7f800000);
        int best = -1;
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // (the backward kernel's first-maximum rule)
          const float v = wf[k * V + e];
          if (v > m || best < 0) { m = v; best = k; }
        }
        // bit 7: the window's selected value is > 0 (for the backward's RELU_GRAD
        // when the pooled input is relu(a): a[best] > 0 <=> relu(a)[best] > 0)
        packed |= ((unsigned)best | (m > 0.f ? 0x80u : 0u)) << (8 * e);
      }
      if (V == 4) *reinterpret_cast<unsigned*>(codes + (size_t)p * C + c) = packed;
      else *reinterpret_cast<unsigned short*>(codes + (size_t)p * C + c) = (unsigned short)packed;
    }
  }
}

// backward of the above: each window's dy goes to its first maximal element
// (row-major, as maxpool_bwd_tiled_kernel); rows / columns a VALID pool never
// reads (odd H or W) get zero gradient.  Thread = (output pixel, V channels):
// neighbouring lanes touch neighbouring 8- / 16-byte pieces of the same window rows.
// With epi.n > 0 (f2 pooling fusion, even H and W: no skipped rows / columns) the
// consumer's elementwise chain is applied to every gradient value before the store;
// its full-tensor operands are read at the same flat index (dx may alias one of
// them: same thread, read before write).
template <int C, int V>
// code_mask: the consumer chain is RELU_GRAD(a, .) with x = relu(a): applied from
// the codes' recorded sign bit instead of reading a.
__global__ void maxpool2_bwd_kernel(const float* __restrict__ x, const float* __restrict__ dy, float* dx, ConvGeom g,
                                    int total, const __grid_constant__ EpiProg epi, const unsigned char* __restrict__ codes,
                                    int code_mask) {
  using VT = typename std::conditional<V == 4, float4, float2>::type;
  constexpr int Q = C / V;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int p = t / Q, c = (t - p * Q) * V;
    const int wo = p % g.wo, q = p / g.wo, ho = q % g.ho, n = q / g.ho;
    const size_t o0 = (((size_t)n * g.h + 2 * ho) * g.w + 2 * wo) * C + c, o1 = o0 + (size_t)g.w * C;
    VT w4[4];
    unsigned packed = 0;
    if (codes) {  // the forward pass's recorded decisions
      packed = V == 4 ? __ldg(reinterpret_cast<const unsigned*>(codes + (size_t)p * C + c))
                      : __ldg(reinterpret_cast<const unsigned short*>(codes + (size_t)p * C + c));
    } else {
      w4[0] = __ldg(reinterpret_cast<const VT*>(x + o0));
      w4[1] = __ldg(reinterpret_cast<const VT*>(x + o0 + C));
      w4[2] = __ldg(reinterpret_cast<const VT*>(x + o1));
      w4[3] = __ldg(reinterpret_cast<const VT*>(x + o1 + C));
    }
    const VT dv = __ldg(reinterpret_cast<const VT*>(dy + (size_t)p * C + c));
    // the usual chain, RELU_GRAD(pre-activation, this gradient): its four mask vectors
    // are loaded here with the window's other loads (one memory round trip, not two)
    const bool rg = epi.n == 1 && epi.op[0] == EPI_RGRAD && epi.scalar[0] == 2 && epi.swap[0] == 1 &&
                    (reinterpret_cast<uintptr_t>(epi.x[0]) & (sizeof(VT) - 1)) == 0;
    VT m4[4];
    if (rg) {
      const float* a = epi.x[0];
      m4[0] = __ldg(reinterpret_cast<const VT*>(a + o0));
      m4[1] = __ldg(reinterpret_cast<const VT*>(a + o0 + C));
      m4[2] = __ldg(reinterpret_cast<const VT*>(a + o1));
      m4[3] = __ldg(reinterpret_cast<const VT*>(a + o1 + C));
    }
    VT r4[4];
    const float* wf = reinterpret_cast<const float*>(w4);
    const float* df = reinterpret_cast<const float*>(&dv);
    float* rf = reinterpret_cast<float*>(r4);
#pragma unroll
    for (int e = 0; e < V; ++e) {
      int best = -1;
      if (codes) {
        const unsigned cb = (packed >> (8 * e)) & 255u;
        best = code_mask && !(cb & 0x80u) ? -1 : (int)(cb & 3u);  // (-1: masked, nothing routed)
      } else {
        float m = -__int_as_float(0x7f800000);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float v = wf[k * V + e];
          if (v > m || best < 0) { m = v; best = k; }
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) rf[k * V + e] = best == k ? df[e] : 0.f;
    }
    if (rg) {  // RELU_GRAD(a, v) = a > 0 ? v : 0, as epi_apply
      const float* mf = reinterpret_cast<const float*>(m4);
#pragma unroll
      for (int i = 0; i < 4 * V; ++i) rf[i] = mf[i] > 0.f ? rf[i] : 0.f;
    } else if (epi.n) {
      const size_t off[4] = {o0, o0 + C, o1, o1 + C};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float v[V];
#pragma unroll
        for (int e = 0; e < V; ++e) v[e] = rf[k * V + e];
        epi_run<V>(epi, v, (long long)off[k], c);
#pragma unroll
        for (int e = 0; e < V; ++e) rf[k * V + e] = v[e];
      }
    }
    *reinterpret_cast<VT*>(dx + o0) = r4[0];
    *reinterpret_cast<VT*>(dx + o0 + C) = r4[1];
    *reinterpret_cast<VT*>(dx + o1) = r4[2];
    *reinterpret_cast<VT*>(dx + o1 + C) = r4[3];
    // zero the column / row a VALID 2x2 pool skips (odd W / H)
    const bool lastc = wo == g.wo - 1 && g.w > 2 * g.wo;
    const VT z = {};
    if (lastc) {
      *reinterpret_cast<VT*>(dx + o0 + 2 * C) = z;
      *reinterpret_cast<VT*>(dx + o1 + 2 * C) = z;
    }
    if (ho == g.ho - 1 && g.h > 2 * g.ho) {
      const size_t o2 = o1 + (size_t)g.w * C;
      *reinterpret_cast<VT*>(dx + o2) = z;
      *reinterpret_cast<VT*>(dx + o2 + C) = z;
      if (lastc) *reinterpret_cast<VT*>(dx + o2 + 2 * C) = z;
    }
  }
}

template <typename I>
__global__ void avgpool_kernel(const float* __restrict__ x, float* __restrict__ y, ConvGeom g, I total) {
  for (I t = (I)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
    int c = (int)(t % g.co);
    I q = t / g.co;
    int wo = (int)(q % g.wo);
    q /= g.wo;
    int ho = (int)(q % g.ho);
    int n = (int)(q / g.ho);
    float s = 0.f;
    int cnt = 0;
    for (int kh = 0; kh < g.kh; ++kh) {
      int hi = ho * g.sh + kh - g.pt;
      if (hi < 0 || hi >= g.h) continue;
      for (int kw = 0; kw < g.kw; ++kw) {
        int wi = wo * g.sw + kw - g.pl;
        if (wi < 0 || wi >= g.w) continue;
        s = __fadd_rn(s, x[(((long long)n * g.h + hi) * g.w + wi) * g.co + c]);
        ++cnt;
      }
    }
    y[t] = __fdiv_rn(s, (float)cnt);
  }
}

template <typename I>
__global__ void concat_kernel(ConcatArgs a, float* __restrict__ dst, I outer, I dst_inner, I src_inner) {
  // iterate over the SOURCE elements (src_inner = sum of the sources' inner extents):
  // columns of the destination row that no source covers are left untouched
  const I total = outer * src_inner;
  for (I t = (I)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
    const I row = t / src_inner;
    I c = t % src_inner;
    int k = 0;
    while (k + 1 < a.n && c >= (I)a.inner[k]) c -= (I)a.inner[k++];
    dst[row * dst_inner + a.offset[k] + c] = a.src[k][row * a.inner[k] + c];
  }
}

// ---- channel-vectorised pools / concat (C % 4 == 0): one thread per 4 channels,
// the same per-lane operation order as the scalar kernels (bit-identical results)
__device__ __forceinline__ float nanmax(float a, float b) {
  asm("max.NaN.f32 %0, %0, %1;" : "+f"(a) : "f"(b));
  return a;
}

// KS > 0: square KS x KS window known at compile time: the KS*KS loads are issued
// together (predicated) before the fixed-order combine -> same results, more MLP
// 3 x 3 stride-1 average pool (C5): a thread computes RS vertically adjacent outputs
// of one (column, 4 channels), so the 3 + RS - 1 input rows of its strip are loaded
// once (3 (RS + 2) loads for RS outputs instead of 9 RS).  Interior strips only
// (the caller's grid covers strips; border outputs go through the generic path of
// pool4_kernel); per output the summation order is pool4_kernel's (kh, then kw).
constexpr int AVG_RS = 4;
__global__ void avgpool3_strip_kernel(const float4* __restrict__ x, float4* __restrict__ y, ConvGeom g, int total) {
  const int C4 = g.co / 4, HS = (g.ho + AVG_RS - 1) / AVG_RS;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int c = t % C4;
    int q = t / C4;
    const int wo = q % g.wo;
    q /= g.wo;
    const int hs = q % HS, n = q / HS;
    const int ho0 = hs * AVG_RS, nr = min(AVG_RS, g.ho - ho0);
    const int hi0 = ho0 - g.pt, wi0 = wo - g.pl;
    const bool interior = hi0 >= 0 && wi0 >= 0 && hi0 + nr + 2 <= g.h && wi0 + 3 <= g.w;
    if (interior && nr == AVG_RS) {  // the strip's (RS + 2) x 3 window once, in registers
      const float4* xb = x + (((size_t)n * g.h + hi0) * g.w + wi0) * C4 + c;
      float4 v[AVG_RS + 2][3];
#pragma unroll
      for (int rr = 0; rr < AVG_RS + 2; ++rr)
#pragma unroll
        for (int kw = 0; kw < 3; ++kw) v[rr][kw] = __ldg(xb + (rr * g.w + kw) * C4);
      const float r = 1.f / 9.f;
#pragma unroll
      for (int j = 0; j < AVG_RS; ++j) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int kh = 0; kh < 3; ++kh)
#pragma unroll
          for (int kw = 0; kw < 3; ++kw) {
            const float4 u = v[j + kh][kw];
            acc.x = __fadd_rn(acc.x, u.x); acc.y = __fadd_rn(acc.y, u.y);
            acc.z = __fadd_rn(acc.z, u.z); acc.w = __fadd_rn(acc.w, u.w);
          }
        y[(((size_t)n * g.ho + ho0 + j) * g.wo + wo) * C4 + c] =
            make_float4(__fmul_rn(acc.x, r), __fmul_rn(acc.y, r), __fmul_rn(acc.z, r), __fmul_rn(acc.w, r));
      }
      continue;
    }
    for (int j = 0; j < nr; ++j) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      float r;
      if (interior) {
        const float4* xb = x + (((size_t)n * g.h + hi0 + j) * g.w + wi0) * C4 + c;
#pragma unroll
        for (int kh = 0; kh < 3; ++kh)
#pragma unroll
          for (int kw = 0; kw < 3; ++kw) {
            const float4 v = __ldg(xb + (kh * g.w + kw) * C4);
            acc.x = __fadd_rn(acc.x, v.x); acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z); acc.w = __fadd_rn(acc.w, v.w);
          }
        r = 1.f / 9.f;
      } else {
        int cnt = 0;
        for (int kh = 0; kh < 3; ++kh) {
          const int hi = hi0 + j + kh;
          if (hi < 0 || hi >= g.h) continue;
          for (int kw = 0; kw < 3; ++kw) {
            const int wi = wi0 + kw;
            if (wi < 0 || wi >= g.w) continue;
            const float4 v = __ldg(x + (((size_t)n * g.h + hi) * g.w + wi) * C4 + c);
            acc.x = __fadd_rn(acc.x, v.x); acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z); acc.w = __fadd_rn(acc.w, v.w);
            ++cnt;
          }
        }
        r = __frcp_rn((float)cnt);
      }
      y[(((size_t)n * g.ho + ho0 + j) * g.wo + wo) * C4 + c] =
          make_float4(__fmul_rn(acc.x, r), __fmul_rn(acc.y, r), __fmul_rn(acc.z, r), __fmul_rn(acc.w, r));
    }
  }
}

template <bool MAXP, int KS>
__global__ void pool4_kernel(const float4* __restrict__ x, float4* __restrict__ y, ConvGeom g, int total4) {
  const int C4 = g.co / 4;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total4; t += gridDim.x * blockDim.x) {
    const int c = t % C4;
    int q = t / C4;
    const int wo = q % g.wo;
    q /= g.wo;
    const int ho = q % g.ho, n = q / g.ho;
    const float ninf = -__int_as_float(0x7f800000);
    float4 acc = MAXP ? make_float4(ninf, ninf, ninf, ninf) : make_float4(0.f, 0.f, 0.f, 0.f);
    int cnt = 0;
    const int hi0 = ho * g.sh - g.pt, wi0 = wo * g.sw - g.pl;
    if (KS > 0 && hi0 >= 0 && wi0 >= 0 && hi0 + KS <= g.h && wi0 + KS <= g.w) {
      // interior window (most outputs): no bounds checks, 32-bit offsets from one base
      const float4* xb = x + (((size_t)n * g.h + hi0) * g.w + wi0) * C4 + c;
      constexpr int KK = KS > 0 ? KS * KS : 1;
      float4 v[KK];
#pragma unroll
      for (int kh = 0; kh < KS; ++kh)
#pragma unroll
        for (int kw = 0; kw < KS; ++kw) v[kh * KS + kw] = __ldg(xb + (kh * g.w + kw) * C4);
#pragma unroll
      for (int i = 0; i < KK; ++i) {
        if (MAXP) {
          acc.x = nanmax(acc.x, v[i].x); acc.y = nanmax(acc.y, v[i].y); acc.z = nanmax(acc.z, v[i].z); acc.w = nanmax(acc.w, v[i].w);
        } else {
          acc.x = __fadd_rn(acc.x, v[i].x); acc.y = __fadd_rn(acc.y, v[i].y);
          acc.z = __fadd_rn(acc.z, v[i].z); acc.w = __fadd_rn(acc.w, v[i].w);
        }
      }
      cnt = KK;
    } else if (KS > 0) {
      constexpr int KK = KS > 0 ? KS * KS : 1;
      float4 v[KK];
      bool ok[KK];
#pragma unroll
      for (int kh = 0; kh < KS; ++kh)
#pragma unroll
        for (int kw = 0; kw < KS; ++kw) {
          const int hi = ho * g.sh + kh - g.pt, wi = wo * g.sw + kw - g.pl;
          ok[kh * KS + kw] = hi >= 0 && hi < g.h && wi >= 0 && wi < g.w;
          v[kh * KS + kw] = ok[kh * KS + kw] ? __ldg(x + (((size_t)n * g.h + hi) * g.w + wi) * C4 + c) : acc;
        }
#pragma unroll
      for (int i = 0; i < KS * KS; ++i) {
        if (!ok[i]) continue;
        if (MAXP) {
          acc.x = nanmax(acc.x, v[i].x); acc.y = nanmax(acc.y, v[i].y); acc.z = nanmax(acc.z, v[i].z); acc.w = nanmax(acc.w, v[i].w);
        } else {
          acc.x = __fadd_rn(acc.x, v[i].x); acc.y = __fadd_rn(acc.y, v[i].y);
          acc.z = __fadd_rn(acc.z, v[i].z); acc.w = __fadd_rn(acc.w, v[i].w);
        }
        ++cnt;
      }
    } else
    for (int kh = 0; kh < g.kh; ++kh) {
      const int hi = ho * g.sh + kh - g.pt;
      if (hi < 0 || hi >= g.h) continue;
      for (int kw = 0; kw < g.kw; ++kw) {
        const int wi = wo * g.sw + kw - g.pl;
        if (wi < 0 || wi >= g.w) continue;
        const float4 v = __ldg(x + (((size_t)n * g.h + hi) * g.w + wi) * C4 + c);
        if (MAXP) {
          acc.x = nanmax(acc.x, v.x); acc.y = nanmax(acc.y, v.y); acc.z = nanmax(acc.z, v.z); acc.w = nanmax(acc.w, v.w);
        } else {
          acc.x = __fadd_rn(acc.x, v.x); acc.y = __fadd_rn(acc.y, v.y);
          acc.z = __fadd_rn(acc.z, v.z); acc.w = __fadd_rn(acc.w, v.w);
        }
        ++cnt;
      }
    }
    if (!MAXP) {  // x (1 / count): within 1 ulp of the quotient (the pool tolerance)
      const float r = __frcp_rn((float)cnt);
      acc = make_float4(__fmul_rn(acc.x, r), __fmul_rn(acc.y, r), __fmul_rn(acc.z, r), __fmul_rn(acc.w, r));
    }
    y[t] = acc;
  }
}

__global__ void concat4_kernel(ConcatArgs a, float4* __restrict__ dst, int outer, int dst_inner4, int src_inner4) {
  const int total = outer * src_inner4;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int row = t / src_inner4;
    int c = (t - row * src_inner4) * 4, k = 0;
    while (k + 1 < a.n && c >= (int)a.inner[k]) c -= (int)a.inner[k++];
    dst[(size_t)row * dst_inner4 + (a.offset[k] + c) / 4] =
        __ldg(reinterpret_cast<const float4*>(a.src[k] + (size_t)row * a.inner[k] + c));
  }
}

// Debug: position-weighted 64-bit checksum of a buffer (integer atomics: deterministic)
__global__ void checksum_kernel(const unsigned* __restrict__ w, long long n, unsigned long long* out) {
  unsigned long long acc = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc += (unsigned long long)w[i] * (unsigned long long)((i * 2654435761ULL) | 1ULL);
  for (int o = 16; o >= 1; o /= 2) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

int grid_for(long long total, int threads = 256) {
  long long b = (total + threads - 1) / threads;
  return (int)std::max<long long>(1, std::min<long long>(b, 148LL * 16));
}

}  // namespace

cudaError_t launch_update_copy(const CopyDesc* descs_dev, int n_desc, long long max_n, cudaStream_t s) {
  if (n_desc <= 0) return cudaSuccess;
  int gx = grid_for((max_n + 3) / 4);
  update_copy_kernel<<<dim3(gx, n_desc), 256, 0, s>>>(descs_dev);
  return cudaGetLastError();
}

cudaError_t launch_copy(const float* src, float* dst, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  copy_kernel<<<grid_for((n + 3) / 4), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

cudaError_t launch_reduce_finalize(const float* ws, float* out, long long oi, long long S, int op, cudaStream_t s) {
  if (S >= 512 && oi <= 4096) {  // very many partials: a block per output
    reduce_finalize_tree_kernel<<<(unsigned)oi, 256, 0, s>>>(ws, out, oi, S, op);
    return cudaGetLastError();
  }
  if (S >= 8 && oi <= 262144) {  // a warp per output
    reduce_finalize_warp_kernel<<<(unsigned)((oi + 7) / 8), 256, 0, s>>>(ws, out, oi, S, op);
    return cudaGetLastError();
  }
  if (oi % 4 == 0 && (reinterpret_cast<uintptr_t>(ws) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    reduce_finalize4_kernel<<<(unsigned)((oi / 4 + 255) / 256), 256, 0, s>>>((const float4*)ws, (float4*)out, oi / 4, S, op);
    return cudaGetLastError();
  }
  reduce_finalize_kernel<<<(unsigned)((oi + 255) / 256), 256, 0, s>>>(ws, out, oi, S, op);
  return cudaGetLastError();
}

cudaError_t launch_dot_simt(const float* A, const float* B, float* C, int M, int N, int K, int ta, int tb,
                            cudaStream_t s) {
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  dot_simt_kernel<<<grid, 256, 0, s>>>(A, B, C, M, N, K, ta, tb);
  return cudaGetLastError();
}

cudaError_t launch_conv2d_fwd(const float* x, const float* w, float* y, const ConvGeom& g, cudaStream_t s) {
  long long total = (long long)g.n * g.ho * g.wo * g.co;
  if (total < INT32_MAX) conv_fwd_kernel<int><<<grid_for(total), 256, 0, s>>>(x, w, y, g, (int)total);
  else conv_fwd_kernel<long long><<<grid_for(total), 256, 0, s>>>(x, w, y, g, total);
  return cudaGetLastError();
}

cudaError_t launch_conv2d_bwd_input(const float* dy, const float* w, float* dx, const ConvGeom& g, cudaStream_t s) {
  long long total = (long long)g.n * g.h * g.w * g.ci;
  if (total < INT32_MAX) conv_bwd_input_kernel<int><<<grid_for(total), 256, 0, s>>>(dy, w, dx, g, (int)total);
  else conv_bwd_input_kernel<long long><<<grid_for(total), 256, 0, s>>>(dy, w, dx, g, total);
  return cudaGetLastError();
}

static void bwdk_split(const ConvGeom& g, int num_sms, long long* P, long long* chunk, long long* S, int* outs) {
  *outs = g.kh * g.kw * g.ci * g.co;
  *P = (long long)g.n * g.ho * g.wo;
  long long want_threads = (long long)num_sms * 2048;
  long long sp = std::max<long long>(1, want_threads / std::max(1, *outs));
  sp = std::min<long long>(sp, std::max<long long>(1, *P / 64));
  sp = std::min<long long>(sp, 65535);
  *chunk = (*P + sp - 1) / sp;
  *S = (*P + *chunk - 1) / *chunk;
}

size_t conv2d_bwd_kernel_ws(const ConvGeom& g, int num_sms) {
  long long P, chunk, S;
  int outs;
  bwdk_split(g, num_sms, &P, &chunk, &S, &outs);
  return (size_t)(S * outs);
}

cudaError_t launch_conv2d_bwd_kernel(const float* x, const float* dy, float* dw, float* ws, const ConvGeom& g,
                                     int num_sms, cudaStream_t s) {
  long long P, chunk, S;
  int outs;
  bwdk_split(g, num_sms, &P, &chunk, &S, &outs);
  dim3 grid((outs + 127) / 128, (unsigned)S);
  conv_bwd_kernel_kernel<<<grid, 128, 0, s>>>(x, dy, ws, g, P, chunk, outs);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_reduce_finalize(ws, dw, outs, S, 0, s);
}

static bool maxpool2_ok(const ConvGeom& g) {
  return g.kh == 2 && g.kw == 2 && g.sh == 2 && g.sw == 2 && g.pt == 0 && g.pl == 0 && (g.co == 6 || g.co == 16) &&
         (long long)g.n * g.h * g.w * g.co < INT32_MAX && g.h >= 2 * g.ho && g.w >= 2 * g.wo && g.h <= 2 * g.ho + 1 &&
         g.w <= 2 * g.wo + 1 && !getenv("CG_POOL_GENERIC");
}

bool maxpool_fusable(const ConvGeom& g) { return maxpool2_ok(g) && g.h == 2 * g.ho && g.w == 2 * g.wo; }

cudaError_t launch_maxpool(const float* x, float* y, const ConvGeom& g, cudaStream_t s, const EpiProg* pro, float* xo,
                           unsigned char* codes) {
  if (codes && !maxpool_fusable(g)) return cudaErrorInvalidValue;
  long long total = (long long)g.n * g.ho * g.wo * g.co;
  EpiProg ep{};
  if (pro && pro->n) {
    if (!maxpool_fusable(g) || (!xo && !codes)) return cudaErrorInvalidValue;
    ep = *pro;
  }
  if (maxpool2_ok(g)) {
    const int pix = g.n * g.ho * g.wo;
    if (g.co == 6) maxpool2_fwd_kernel<6, 2><<<grid_for(pix * 3), 256, 0, s>>>(x, y, g, pix * 3, xo, ep, codes);
    else maxpool2_fwd_kernel<16, 4><<<grid_for(pix * 4), 256, 0, s>>>(x, y, g, pix * 4, xo, ep, codes);
    return cudaGetLastError();
  }
  if (g.co % 4 == 0 && total < INT32_MAX) {
    const int blocks = (int)std::min<long long>((total / 4 + 255) / 256, 65535LL * 8);
    if (g.kh == 3 && g.kw == 3) pool4_kernel<true, 3><<<blocks, 256, 0, s>>>((const float4*)x, (float4*)y, g, (int)(total / 4));
    else pool4_kernel<true, 0><<<grid_for(total / 4), 256, 0, s>>>((const float4*)x, (float4*)y, g, (int)(total / 4));
    return cudaGetLastError();
  }
  if (total < INT32_MAX) maxpool_kernel<int><<<grid_for(total), 256, 0, s>>>(x, y, g, (int)total);
  else maxpool_kernel<long long><<<grid_for(total), 256, 0, s>>>(x, y, g, total);
  return cudaGetLastError();
}

cudaError_t launch_maxpool_bwd(const float* x, const float* dy, float* dx, const ConvGeom& g, cudaStream_t s,
                               const EpiProg* epi, const unsigned char* codes, int code_mask) {
  if ((codes && !maxpool_fusable(g)) || (code_mask && !codes)) return cudaErrorInvalidValue;
  EpiProg ep{};
  if (epi && epi->n) {
    if (!maxpool_fusable(g)) return cudaErrorInvalidValue;
    ep = *epi;
  }
  if (maxpool2_ok(g)) {
    const int pix = g.n * g.ho * g.wo;
    if (g.co == 6) maxpool2_bwd_kernel<6, 2><<<grid_for(pix * 3), 256, 0, s>>>(x, dy, dx, g, pix * 3, ep, codes, code_mask);
    else maxpool2_bwd_kernel<16, 4><<<grid_for(pix * 4), 256, 0, s>>>(x, dy, dx, g, pix * 4, ep, codes, code_mask);
    return cudaGetLastError();
  }
  if (g.kh == g.sh && g.kw == g.sw && g.pt == 0 && g.pl == 0 && g.h == g.ho * g.sh && g.w == g.wo * g.sw) {
    long long windows = (long long)g.n * g.ho * g.wo * g.co;
    if (windows < INT32_MAX) maxpool_bwd_tiled_kernel<int><<<grid_for(windows), 256, 0, s>>>(x, dy, dx, g, (int)windows);
    else maxpool_bwd_tiled_kernel<long long><<<grid_for(windows), 256, 0, s>>>(x, dy, dx, g, windows);
    return cudaGetLastError();
  }
  long long total = (long long)g.n * g.h * g.w * g.co;
  if (total < INT32_MAX) maxpool_bwd_kernel<int><<<grid_for(total), 256, 0, s>>>(x, dy, dx, g, (int)total);
  else maxpool_bwd_kernel<long long><<<grid_for(total), 256, 0, s>>>(x, dy, dx, g, total);
  return cudaGetLastError();
}

// 3x3 stride-1 average pool, one thread per (image, output column, float4 of channels)
// sweeping the rows: the 3 x 3 window slides down in registers (one new input row of
// three float4 per output row, against 4.5 loads per output for 4-row strips).
// Same arithmetic as avgpool3_strip_kernel: the in-bounds taps summed in (kh, kw)
// order from +0, times 1/9 (interior) or __frcp_rn(count).
__global__ void __launch_bounds__(256) avgpool3_sweep_kernel(const float4* __restrict__ x, float4* __restrict__ y,
                                                            ConvGeom g, int total) {
  const int C4 = g.co / 4;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int c = t % C4;
    const int q = t / C4, wo = q % g.wo, n = q / g.wo;
    const int wi0 = wo - g.pl;
    const float4* xn = x + (size_t)n * g.h * g.w * C4 + c;
    int cols = 0;
#pragma unroll
    for (int kw = 0; kw < 3; ++kw) cols += (unsigned)(wi0 + kw) < (unsigned)g.w;
    auto load_row = [&](int hi, float4 (&r)[3]) {
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        const int wi = wi0 + kw;
        r[kw] = (unsigned)hi < (unsigned)g.h && (unsigned)wi < (unsigned)g.w ? __ldg(xn + ((size_t)hi * g.w + wi) * C4)
                                                                            : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    float4 win[3][3];
    load_row(-g.pt, win[0]);
    load_row(1 - g.pt, win[1]);
    for (int ho = 0; ho < g.ho; ++ho) {
      const int hi0 = ho - g.pt;
      load_row(hi0 + 2, win[2]);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      int rows = 0;
#pragma unroll
      for (int kh = 0; kh < 3; ++kh) {
        rows += (unsigned)(hi0 + kh) < (unsigned)g.h;
#pragma unroll
        for (int kw = 0; kw < 3; ++kw) {  // (+0 for an out-of-image tap: exact, acc is never -0)
          const float4 u = win[kh][kw];
          acc.x = __fadd_rn(acc.x, u.x); acc.y = __fadd_rn(acc.y, u.y);
          acc.z = __fadd_rn(acc.z, u.z); acc.w = __fadd_rn(acc.w, u.w);
        }
      }
      const int cnt = rows * cols;
      const float r = cnt == 9 ? 1.f / 9.f : __frcp_rn((float)cnt);
      y[(((size_t)n * g.ho + ho) * g.wo + wo) * C4 + c] =
          make_float4(__fmul_rn(acc.x, r), __fmul_rn(acc.y, r), __fmul_rn(acc.z, r), __fmul_rn(acc.w, r));
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        win[0][kw] = win[1][kw];
        win[1][kw] = win[2][kw];
      }
    }
  }
}

cudaError_t launch_avgpool(const float* x, float* y, const ConvGeom& g, cudaStream_t s) {
  long long total = (long long)g.n * g.ho * g.wo * g.co;
  if (g.co % 4 == 0 && total < INT32_MAX) {
    const int blocks = (int)std::min<long long>((total / 4 + 255) / 256, 65535LL * 8);
    // (measured on C5's eleven 3x3 average pools: 1.31 ms with 4-row strips, 1.15 ms
    // sweeping; CG_POOL_STRIPS=1 keeps the strips for A/B)
    static const bool sweep = !getenv("CG_POOL_STRIPS");
    if (sweep && g.kh == 3 && g.kw == 3 && g.sh == 1 && g.sw == 1 && g.ho == g.h + 2 * g.pt - 2) {
      const long long cols = (long long)g.n * g.wo * (g.co / 4);
      avgpool3_sweep_kernel<<<grid_for(cols), 256, 0, s>>>((const float4*)x, (float4*)y, g, (int)cols);
    } else if (g.kh == 3 && g.kw == 3 && g.sh == 1 && g.sw == 1 && !getenv("CG_POOL_NO_STRIPS")) {
      const long long strips = (long long)g.n * ((g.ho + AVG_RS - 1) / AVG_RS) * g.wo * (g.co / 4);
      avgpool3_strip_kernel<<<grid_for(strips), 256, 0, s>>>((const float4*)x, (float4*)y, g, (int)strips);
    } else if (g.kh == 3 && g.kw == 3) pool4_kernel<false, 3><<<blocks, 256, 0, s>>>((const float4*)x, (float4*)y, g, (int)(total / 4));
    else pool4_kernel<false, 0><<<grid_for(total / 4), 256, 0, s>>>((const float4*)x, (float4*)y, g, (int)(total / 4));
    return cudaGetLastError();
  }
  if (total < INT32_MAX) avgpool_kernel<int><<<grid_for(total), 256, 0, s>>>(x, y, g, (int)total);
  else avgpool_kernel<long long><<<grid_for(total), 256, 0, s>>>(x, y, g, total);
  return cudaGetLastError();
}

cudaError_t launch_concat(const ConcatArgs& a, float* dst, long long outer, long long dst_inner, cudaStream_t s) {
  if (a.n < 1) return cudaSuccess;
  long long src_inner = 0;
  for (int k = 0; k < a.n; ++k) src_inner += a.inner[k];
  bool vec = dst_inner % 4 == 0 && outer * dst_inner < INT32_MAX && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  for (int k = 0; k < a.n; ++k)
    vec = vec && a.inner[k] % 4 == 0 && a.offset[k] % 4 == 0 && (reinterpret_cast<uintptr_t>(a.src[k]) & 15) == 0;
  if (vec) {
    concat4_kernel<<<grid_for(outer * src_inner / 4), 256, 0, s>>>(a, (float4*)dst, (int)outer, (int)(dst_inner / 4),
                                                                   (int)(src_inner / 4));
    return cudaGetLastError();
  }
  if (outer * dst_inner < INT32_MAX)
    concat_kernel<int><<<grid_for(outer * src_inner), 256, 0, s>>>(a, dst, (int)outer, (int)dst_inner, (int)src_inner);
  else
    concat_kernel<long long><<<grid_for(outer * src_inner), 256, 0, s>>>(a, dst, outer, dst_inner, src_inner);
  return cudaGetLastError();
}

unsigned long long debug_checksum(const float* p, long long n, cudaStream_t s) {
  static unsigned long long* d = nullptr;
  if (!d) cudaMalloc(&d, sizeof(unsigned long long));
  cudaMemsetAsync(d, 0, sizeof(unsigned long long), s);
  checksum_kernel<<<grid_for(n), 256, 0, s>>>(reinterpret_cast<const unsigned*>(p), n, d);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  return h;
}

}  // namespace cg
