// CONV2D family for small images and few channels (LeNet-shaped graphs, C4):
// each thread block keeps whole images in shared memory, so every input,
// output and gradient element crosses HBM exactly once; the arithmetic is
// fp32 FFMA in a fixed order per output (deterministic, no atomics).
//
//   fwd      y[n,ho,wo,co]   = sum_{kh,kw,ci} x[n,ho*sh+kh-pt,wo*sw+kw-pl,ci] w[kh,kw,ci,co]
//            one thread per output pixel, all Co in registers (CO template)
//   bwd-in   dx[n,h,w,ci]    = sum_{kh,kw,co} dy[n,(h+pt-kh)/sh,(w+pl-kw)/sw,co] w[kh,kw,ci,co]
//            one thread per input pixel, all Ci in registers (CI template)
//   bwd-k    dw[kh,kw,ci,co] = sum_{n,ho,wo} x[n,ho*sh+kh-pt,wo*sw+kw-pl,ci] dy[n,ho,wo,co]
//            thread = (tap, 4 output channels, pixel phase); per-block partials
//            over a chunk of images, then a fixed-order reduction.
// (definitions: SURVEY §8(c) c1-defs, the oracle's conv2d_f64 family)
#include <cuda_runtime.h>

#include <algorithm>

#include "conv_small.h"
#include "kernels.h"

namespace cg {

namespace {

constexpr int SMEM_LIMIT = 96 * 1024;

// zero-padded image n of x [N,H,W,C] into s, channel-planar [C][Hp][Wp] so that
// threads on adjacent pixels read adjacent words (no bank conflicts)
__device__ __forceinline__ void load_padded(float* s, const float* __restrict__ x, int n, int H, int W, int C, int Hp,
                                            int Wp, int pt, int pl) {
  const int tot = Hp * Wp * C;
  const float* xi = x + (size_t)n * H * W * C;
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {  // e walks the NHWC source order (coalesced)
    const int c = e % C, q = e / C, wp = q % Wp, hp = q / Wp;
    const int h = hp - pt, w = wp - pl;
    s[(c * Hp + hp) * Wp + wp] = (h >= 0 && h < H && w >= 0 && w < W) ? __ldg(xi + ((size_t)h * W + w) * C + c) : 0.f;
  }
}

template <int CO, int KS>  // KS > 0: square KS x KS kernel known at compile time (unrolled taps)
__global__ void __launch_bounds__(256) conv_fwd_img(const float* __restrict__ x, const float* __restrict__ w,
                                                    float* __restrict__ y, ConvGeom g, int Hp, int Wp) {
  extern __shared__ float sm[];
  const int KT = g.kh * g.kw * g.ci;
  float* ws = sm;                    // [KT][CO] (co padded with zeros)
  float* xs = sm + KT * CO;          // padded image
  for (int e = threadIdx.x; e < KT * CO; e += blockDim.x) {
    const int co = e % CO, k = e / CO;
    ws[e] = co < g.co ? w[(size_t)k * g.co + co] : 0.f;
  }
  const int P = g.ho * g.wo;
  for (int n = blockIdx.x; n < g.n; n += gridDim.x) {
    __syncthreads();
    load_padded(xs, x, n, g.h, g.w, g.ci, Hp, Wp, g.pt, g.pl);
    __syncthreads();
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      const int ho = p / g.wo, wo = p % g.wo;
      float acc[CO];
#pragma unroll
      for (int c = 0; c < CO; ++c) acc[c] = 0.f;
      const int KH = KS ? KS : g.kh, KW = KS ? KS : g.kw;
#pragma unroll
      for (int kh = 0; kh < KH; ++kh)
#pragma unroll
        for (int kw = 0; kw < KW; ++kw) {
          const float* xp = xs + (ho * g.sh + kh) * Wp + wo * g.sw + kw;
          const float* wp = ws + ((kh * KW + kw) * g.ci) * CO;
          for (int ci = 0; ci < g.ci; ++ci) {
            const float a = xp[ci * Hp * Wp];
#pragma unroll
            for (int c = 0; c < CO; c += 4) {
              const float4 b = *reinterpret_cast<const float4*>(wp + ci * CO + c);
              acc[c] = fmaf(a, b.x, acc[c]);
              acc[c + 1] = fmaf(a, b.y, acc[c + 1]);
              acc[c + 2] = fmaf(a, b.z, acc[c + 2]);
              acc[c + 3] = fmaf(a, b.w, acc[c + 3]);
            }
          }
        }
      float* yp = y + ((size_t)n * P + p) * g.co;
#pragma unroll
      for (int c = 0; c < CO; ++c)
        if (c < g.co) yp[c] = acc[c];
    }
  }
}

template <int CI, int KS>
__global__ void __launch_bounds__(256) conv_bwdin_img(const float* __restrict__ dy, const float* __restrict__ w,
                                                      float* __restrict__ dx, ConvGeom g) {
  extern __shared__ float sm[];
  const int taps = g.kh * g.kw;
  float* wt = sm;                            // [tap][co][CI] (ci padded)
  float* ds = sm + taps * g.co * CI;         // dy image, channel-planar [co][ho*wo]
  for (int e = threadIdx.x; e < taps * g.co * CI; e += blockDim.x) {
    const int ci = e % CI, q = e / CI, co = q % g.co, t = q / g.co;
    wt[e] = ci < g.ci ? w[((size_t)t * g.ci + ci) * g.co + co] : 0.f;
  }
  const int P = g.h * g.w, PO = g.ho * g.wo * g.co, PP = g.ho * g.wo;
  for (int n = blockIdx.x; n < g.n; n += gridDim.x) {
    __syncthreads();
    const float* dyi = dy + (size_t)n * PO;
    for (int e = threadIdx.x; e < PO; e += blockDim.x) ds[(e % g.co) * PP + e / g.co] = __ldg(dyi + e);
    __syncthreads();
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      const int hi = p / g.w, wi = p % g.w;
      float acc[CI];
#pragma unroll
      for (int c = 0; c < CI; ++c) acc[c] = 0.f;
      const int KH = KS ? KS : g.kh, KW = KS ? KS : g.kw;
#pragma unroll
      for (int kh = 0; kh < KH; ++kh) {
        const int hs = hi + g.pt - kh;
        if (hs < 0 || hs % g.sh) continue;
        const int ho = hs / g.sh;
        if (ho >= g.ho) continue;
#pragma unroll
        for (int kw = 0; kw < KW; ++kw) {
          const int wsn = wi + g.pl - kw;
          if (wsn < 0 || wsn % g.sw) continue;
          const int wo = wsn / g.sw;
          if (wo >= g.wo) continue;
          const float* dp = ds + ho * g.wo + wo;
          const float* wp = wt + (kh * KW + kw) * g.co * CI;
          for (int co = 0; co < g.co; ++co) {
            const float d = dp[co * PP];
#pragma unroll
            for (int c = 0; c < CI; c += 4) {
              const float4 b = *reinterpret_cast<const float4*>(wp + co * CI + c);
              acc[c] = fmaf(d, b.x, acc[c]);
              acc[c + 1] = fmaf(d, b.y, acc[c + 1]);
              acc[c + 2] = fmaf(d, b.z, acc[c + 2]);
              acc[c + 3] = fmaf(d, b.w, acc[c + 3]);
            }
          }
        }
      }
      float* xp = dx + ((size_t)n * P + p) * g.ci;
#pragma unroll
      for (int c = 0; c < CI; ++c)
        if (c < g.ci) xp[c] = acc[c];
    }
  }
}

// bwd-kernel: thread = (tap t, co quad q, pixel phase ph); images [blockIdx.x*chunk, +chunk)
template <int CI>
__global__ void __launch_bounds__(256) conv_bwdk_img(const float* __restrict__ x, const float* __restrict__ dy,
                                                     float* __restrict__ part, ConvGeom g, int Hp, int Wp, int PH,
                                                     int chunk) {
  extern __shared__ float sm[];
  const int taps = g.kh * g.kw, CQ = (g.co + 3) / 4;
  const int units = taps * CQ;
  float* xs = sm;                       // padded image
  float* ds = sm + (Hp * Wp * g.ci + 3) / 4 * 4;  // dy image [ho][wo][co4] (16-byte aligned, co padded to 4)
  const int co4 = CQ * 4;
  const int t = threadIdx.x % units, ph = threadIdx.x / units;
  const bool active = ph < PH;
  const int tap = t / CQ, q = t % CQ;
  const int kh = tap / g.kw, kw = tap % g.kw;
  float acc[CI][4];
#pragma unroll
  for (int c = 0; c < CI; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.f;
  const int P = g.ho * g.wo;
  const int n0 = blockIdx.x * chunk, n1 = min(g.n, n0 + chunk);
  for (int n = n0; n < n1; ++n) {
    __syncthreads();
    load_padded(xs, x, n, g.h, g.w, g.ci, Hp, Wp, g.pt, g.pl);
    const float* dyi = dy + (size_t)n * P * g.co;
    for (int e = threadIdx.x; e < P * co4; e += blockDim.x) {
      const int c = e % co4, p = e / co4;
      ds[e] = c < g.co ? __ldg(dyi + (size_t)p * g.co + c) : 0.f;
    }
    __syncthreads();
    if (active) {
      int ho = ph / g.wo, wo = ph % g.wo;  // (ho, wo) of pixel p, advanced incrementally
      for (int p = ph; p < P; p += PH) {
        if (p != ph) {
          wo += PH;
          while (wo >= g.wo) { wo -= g.wo; ++ho; }
        }
        const float4 d = *reinterpret_cast<const float4*>(ds + p * co4 + q * 4);
        const float* xp = xs + (ho * g.sh + kh) * Wp + wo * g.sw + kw;
#pragma unroll
        for (int c = 0; c < CI; ++c) {
          if (c < g.ci) {
            const float a = xp[c * Hp * Wp];
            acc[c][0] = fmaf(a, d.x, acc[c][0]);
            acc[c][1] = fmaf(a, d.y, acc[c][1]);
            acc[c][2] = fmaf(a, d.z, acc[c][2]);
            acc[c][3] = fmaf(a, d.w, acc[c][3]);
          }
        }
      }
    }
  }
  // fixed-order reduction over the PH pixel phases, then one partial per block
  __syncthreads();
  float* red = sm;  // [PH][taps*ci*co4]
  const int O = taps * g.ci * co4;
  if (active) {
#pragma unroll
    for (int c = 0; c < CI; ++c)
      if (c < g.ci)
        for (int j = 0; j < 4; ++j) red[ph * O + (tap * g.ci + c) * co4 + q * 4 + j] = acc[c][j];
  }
  __syncthreads();
  const int OO = taps * g.ci * g.co;
  for (int o = threadIdx.x; o < OO; o += blockDim.x) {
    const int co = o % g.co, r = o / g.co;  // r = tap*ci + ci
    float s = red[r * co4 + co];
    for (int h = 1; h < PH; ++h) s = __fadd_rn(s, red[h * O + r * co4 + co]);
    part[(size_t)blockIdx.x * OO + o] = s;
  }
}

struct Pads {
  int Hp, Wp;
};
Pads pads(const ConvGeom& g) {
  return {(g.ho - 1) * g.sh + g.kh, (g.wo - 1) * g.sw + g.kw};
}

int co_pad(int c) { return c <= 8 ? 8 : c <= 16 ? 16 : c <= 32 ? 32 : 0; }

size_t fwd_smem(const ConvGeom& g) {
  Pads p = pads(g);
  int CO = co_pad(g.co);
  return ((size_t)g.kh * g.kw * g.ci * CO + (size_t)std::max(p.Hp, g.h + g.pt) * std::max(p.Wp, g.w + g.pl) * g.ci) * 4;
}
size_t bwdin_smem(const ConvGeom& g) {
  int CI = co_pad(g.ci);
  return ((size_t)g.kh * g.kw * g.co * CI + (size_t)g.ho * g.wo * g.co) * 4;
}
void bwdk_geom(const ConvGeom& g, int* PH, int* units) {
  *units = g.kh * g.kw * ((g.co + 3) / 4);
  *PH = std::max(1, 256 / *units);
}
size_t bwdk_smem(const ConvGeom& g) {
  Pads p = pads(g);
  int PH, units;
  bwdk_geom(g, &PH, &units);
  const int co4 = (g.co + 3) / 4 * 4;
  size_t img = ((size_t)std::max(p.Hp, g.h + g.pt) * std::max(p.Wp, g.w + g.pl) * g.ci + 3) / 4 * 4 +
               (size_t)g.ho * g.wo * co4;
  size_t red = (size_t)PH * g.kh * g.kw * g.ci * co4;
  return std::max(img, red) * 4;
}
int bwdk_blocks(const ConvGeom& g, int num_sms) { return std::min(g.n, num_sms * 8); }

template <typename F>
void set_smem(F f) {
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT);
}

}  // namespace

bool conv_small_fwd_ok(const ConvGeom& g) { return co_pad(g.co) && fwd_smem(g) <= SMEM_LIMIT; }
bool conv_small_bwdin_ok(const ConvGeom& g) { return co_pad(g.ci) && bwdin_smem(g) <= SMEM_LIMIT; }
bool conv_small_bwdk_ok(const ConvGeom& g) {
  int PH, units;
  bwdk_geom(g, &PH, &units);
  return g.ci <= 8 && units <= 256 && bwdk_smem(g) <= SMEM_LIMIT;
}
size_t conv_small_bwdk_ws(const ConvGeom& g, int num_sms) {
  return (size_t)bwdk_blocks(g, num_sms) * g.kh * g.kw * g.ci * g.co;
}

cudaError_t launch_conv_small_fwd(const float* x, const float* w, float* y, const ConvGeom& g, int num_sms,
                                  cudaStream_t s) {
  Pads p = pads(g);
  const int Hp = std::max(p.Hp, g.h + g.pt), Wp = std::max(p.Wp, g.w + g.pl);
  const size_t smem = fwd_smem(g);
  const int grid = std::min(g.n, num_sms * 8);
  const bool k5 = g.kh == 5 && g.kw == 5;
#define CG_FWD(CO, KS) \
  set_smem(conv_fwd_img<CO, KS>);  \
  conv_fwd_img<CO, KS><<<grid, 256, smem, s>>>(x, w, y, g, Hp, Wp)
  switch (co_pad(g.co)) {
    case 8: if (k5) { CG_FWD(8, 5); } else { CG_FWD(8, 0); } break;
    case 16: if (k5) { CG_FWD(16, 5); } else { CG_FWD(16, 0); } break;
    default: if (k5) { CG_FWD(32, 5); } else { CG_FWD(32, 0); } break;
  }
#undef CG_FWD
  return cudaGetLastError();
}

cudaError_t launch_conv_small_bwdin(const float* dy, const float* w, float* dx, const ConvGeom& g, int num_sms,
                                    cudaStream_t s) {
  const size_t smem = bwdin_smem(g);
  const int grid = std::min(g.n, num_sms * 8);
  const bool k5 = g.kh == 5 && g.kw == 5;
#define CG_BIN(CI, KS) \
  set_smem(conv_bwdin_img<CI, KS>);  \
  conv_bwdin_img<CI, KS><<<grid, 256, smem, s>>>(dy, w, dx, g)
  switch (co_pad(g.ci)) {
    case 8: if (k5) { CG_BIN(8, 5); } else { CG_BIN(8, 0); } break;
    case 16: if (k5) { CG_BIN(16, 5); } else { CG_BIN(16, 0); } break;
    default: if (k5) { CG_BIN(32, 5); } else { CG_BIN(32, 0); } break;
  }
#undef CG_BIN
  return cudaGetLastError();
}

cudaError_t launch_conv_small_bwdk(const float* x, const float* dy, float* dw, float* ws, const ConvGeom& g,
                                   int num_sms, cudaStream_t s) {
  Pads p = pads(g);
  const int Hp = std::max(p.Hp, g.h + g.pt), Wp = std::max(p.Wp, g.w + g.pl);
  int PH, units;
  bwdk_geom(g, &PH, &units);
  const int blocks = bwdk_blocks(g, num_sms);
  const int chunk = (g.n + blocks - 1) / blocks;
  const int nb = (g.n + chunk - 1) / chunk;
  const size_t smem = bwdk_smem(g);
  if (g.ci <= 1) {
    set_smem(conv_bwdk_img<1>);
    conv_bwdk_img<1><<<nb, 256, smem, s>>>(x, dy, ws, g, Hp, Wp, PH, chunk);
  } else {
    set_smem(conv_bwdk_img<8>);
    conv_bwdk_img<8><<<nb, 256, smem, s>>>(x, dy, ws, g, Hp, Wp, PH, chunk);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_reduce_finalize(ws, dw, (long long)g.kh * g.kw * g.ci * g.co, nb, 0, s);
}

}  // namespace cg
