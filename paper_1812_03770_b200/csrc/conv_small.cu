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
#include <cstdlib>

#include "conv_small.h"
#include "kernels.h"

namespace cg {

namespace {

constexpr int SMEM_LIMIT = 96 * 1024;

// a / d (0 <= a < 2^20, d >= 1) from a precomputed fp32 1/d: (a + 0.5) is exact and
// at least 0.5 from a multiple of d, while the two roundings perturb the quotient by
// < 2^-23 relative, i.e. < 0.5 / d for a < 2^22 -- so the floor is exact (also
// checked exhaustively for d <= 256).  The loaders' runtime integer divisions were
// the instruction count of the few-channel kernels.
__device__ __forceinline__ int fdivs(int a, float inv) {
  return __float2int_rd(__fmul_rn(__fadd_rn(__int2float_rn(a), 0.5f), inv));
}

// zero-padded image n of x [N,H,W,C] into s, channel-planar [C][Hp][Wp] so that
// threads on adjacent pixels read adjacent words (no bank conflicts)
template <int U = 8>  // loads in flight per thread
__device__ __forceinline__ void load_padded(float* s, const float* __restrict__ x, int n, int H, int W, int C, int Hp,
                                            int Wp, int pt, int pl) {
  const int tot = Hp * Wp * C;
  const float* xi = x + (size_t)n * H * W * C;
  const float invC = 1.f / (float)C, invWp = 1.f / (float)Wp;
  // e walks the NHWC source order (coalesced); U loads in flight per thread
  for (int e0 = threadIdx.x; e0 < tot; e0 += U * blockDim.x) {
    float v[U];
    int dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * blockDim.x;
      const int q = fdivs(e, invC), c = e - q * C, hp = fdivs(q, invWp), wp = q - hp * Wp;
      const int h = hp - pt, w = wp - pl;
      dst[u] = e < tot ? (c * Hp + hp) * Wp + wp : -1;
      v[u] = (e < tot && h >= 0 && h < H && w >= 0 && w < W) ? __ldg(xi + ((size_t)h * W + w) * C + c) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u] >= 0) s[dst[u]] = v[u];
  }
}

// dy image [P][C] -> shared [P][C4] (channels zero-padded to C4), 8 loads in flight
__device__ __forceinline__ void load_dy_padded(float* ds, const float* __restrict__ dyi, int P, int C, int C4) {
  const int tot = P * C4;
  const float invC4 = 1.f / (float)C4;
  for (int e0 = threadIdx.x; e0 < tot; e0 += 8 * blockDim.x) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      const int p = fdivs(e, invC4), c = e - p * C4;
      v[u] = (e < tot && c < C) ? __ldg(dyi + (size_t)p * C + c) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < tot) ds[e] = v[u];
    }
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
    load_padded<1>(xs, x, n, g.h, g.w, g.ci, Hp, Wp, g.pt, g.pl);
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
    load_dy_padded(ds, dy + (size_t)n * P * g.co, P, g.co, co4);
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

// ---------------------------------------------------------------- register-tiled, stride 1
// Forward correlation of a zero-padded, channel-planar image with a KS x KS
// kernel; each thread computes PX horizontally adjacent output pixels x all
// (padded) output channels, sliding a window of PX+KS-1 input values along the
// row so every shared-memory load feeds PX*COP FMAs.  FLIP = 1 runs the
// backward-input pass as this same correlation: input = dy (channels Co),
// weights flipped in both taps and transposed (ci <-> co), padding KS-1-p.
// Accumulation order per output: ci, kh, kw ascending (deterministic).
struct RtGeom {
  int n, hin, win, cin;     // image fed to the correlation (x, or dy for FLIP)
  int hout, wout, cout;     // result (y, or dx for FLIP)
  int pt, pl;               // zero padding in front
  int wcin, wcout;          // weight tensor [KS][KS][wcin][wcout] as stored (HWIO)
  int Hp, Wp;               // padded image dims in shared memory
};

template <int COP, int KS, int PX, bool FLIP>
__global__ void __launch_bounds__(256) conv_rt_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                                      float* __restrict__ y, RtGeom g, int IMG) {
  extern __shared__ float sm[];
  float* ws = sm;                                  // [KS*KS*cin][COP]
  float* xs = sm + KS * KS * g.cin * COP;          // IMG x [cin][Hp][Wp]
  const int IS = g.cin * g.Hp * g.Wp;
  for (int e = threadIdx.x; e < KS * KS * g.cin * COP; e += blockDim.x) {
    const int co = e % COP, r = e / COP, ci = r % g.cin, tap = r / g.cin;
    float v = 0.f;
    if (co < g.cout) {
      if (!FLIP) {
        v = w[((size_t)tap * g.cin + ci) * g.cout + co];
      } else {  // wf[kh][kw][ci'=co_orig][co'=ci_orig] = w[KS-1-kh][KS-1-kw][ci_orig][co_orig]
        const int kh = tap / KS, kw = tap % KS;
        const int ftap = (KS - 1 - kh) * KS + (KS - 1 - kw);
        v = w[((size_t)ftap * g.wcin + co) * g.wcout + ci];
      }
    }
    ws[e] = v;
  }
  // the padding of every image buffer stays zero: only interiors are rewritten per batch
  for (int e = threadIdx.x; e < IMG * IS; e += blockDim.x) xs[e] = 0.f;
  const int per = g.hout * ((g.wout + PX - 1) / PX);
  const int isz = g.hin * g.win * g.cin;
  const float invC = 1.f / (float)g.cin, invW = 1.f / (float)g.win, invH = 1.f / (float)g.hin;
  for (int n0 = blockIdx.x * IMG; n0 < g.n; n0 += gridDim.x * IMG) {
    const int nimg = min(IMG, g.n - n0);
    __syncthreads();
    // interiors of nimg consecutive images: one contiguous NHWC run, 8 loads in flight
    const float* src = x + (size_t)n0 * isz;
    const int tot = nimg * isz;
    for (int e0 = threadIdx.x; e0 < tot; e0 += 8 * 256) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * 256;
        v[u] = e < tot ? __ldg(src + e) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * 256;
        if (e < tot) {
          int c, ww, h, im;
          if (tot < (1 << 20)) {  // fp32-reciprocal divisions (exact in this range)
            const int q = fdivs(e, invC), q2 = fdivs(q, invW);
            c = e - q * g.cin, ww = q - q2 * g.win, im = fdivs(q2, invH), h = q2 - im * g.hin;
          } else {
            const int q = e / g.cin, q2 = q / g.win;
            c = e - q * g.cin, ww = q - q2 * g.win, im = q2 / g.hin, h = q2 - im * g.hin;
          }
          xs[im * IS + (c * g.Hp + h + g.pt) * g.Wp + ww + g.pl] = v[u];
        }
      }
    }
    __syncthreads();
    // item order: output row fastest, then image, then pixel quad, so a warp's
    // sliding windows start Wp (odd) words apart: conflict-free shared loads
    for (int it = threadIdx.x; it < nimg * per; it += blockDim.x) {
      const int ho = it % g.hout, r2 = it / g.hout, im = r2 % nimg, wo0 = (r2 / nimg) * PX;
      const float* xi = xs + im * IS;
      float acc[PX][COP];
#pragma unroll
      for (int p = 0; p < PX; ++p)
#pragma unroll
        for (int c = 0; c < COP; ++c) acc[p][c] = 0.f;
      for (int ci = 0; ci < g.cin; ++ci) {
#pragma unroll
        for (int kh = 0; kh < KS; ++kh) {
          const float* xr = xi + ((size_t)ci * g.Hp + ho + kh) * g.Wp + wo0;
          float xv[PX + KS - 1];
#pragma unroll
          for (int q = 0; q < PX + KS - 1; ++q) xv[q] = xr[q];
#pragma unroll
          for (int kw = 0; kw < KS; ++kw) {
            const float* wp = ws + ((kh * KS + kw) * g.cin + ci) * COP;
#pragma unroll
            for (int c = 0; c < COP; c += 4) {
              const float4 b = *reinterpret_cast<const float4*>(wp + c);
#pragma unroll
              for (int p = 0; p < PX; ++p) {
                const float a = xv[p + kw];
                acc[p][c] = fmaf(a, b.x, acc[p][c]);
                acc[p][c + 1] = fmaf(a, b.y, acc[p][c + 1]);
                acc[p][c + 2] = fmaf(a, b.z, acc[p][c + 2]);
                acc[p][c + 3] = fmaf(a, b.w, acc[p][c + 3]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int p = 0; p < PX; ++p) {
        if (wo0 + p >= g.wout) break;
        float* yp = y + (((size_t)(n0 + im) * g.hout + ho) * g.wout + wo0 + p) * g.cout;
#pragma unroll
        for (int c = 0; c < COP; ++c)
          if (c < g.cout) yp[c] = acc[p][c];
      }
    }
  }
}

// bwd-kernel, stride 1: thread = (kh, ci, co quad, row phase); the KS kw taps of
// one (kh, ci) slide along a row (one new x value per pixel) -> 4*KS FMAs per
// dy float4; per-block partials over a chunk of images, fixed-order reductions.
template <int KS>
__global__ void __launch_bounds__(256) conv_bwdk_rt_kernel(const float* __restrict__ x, const float* __restrict__ dy,
                                                           float* __restrict__ part, ConvGeom g, int Hp, int Wp, int PH,
                                                           int chunk) {
  extern __shared__ float sm[];
  const int CQ = (g.co + 3) / 4, co4 = CQ * 4;
  const int units = KS * g.ci * CQ;
  float* xs = sm;                                   // [ci][Hp][Wp]
  float* ds = sm + (g.ci * Hp * Wp + 3) / 4 * 4;    // [P][co4]
  const int t = threadIdx.x % units, ph = threadIdx.x / units;
  const bool active = ph < PH;
  const int q = t % CQ, r = t / CQ, ci = r % g.ci, kh = r / g.ci;
  float acc[KS][4];
#pragma unroll
  for (int kw = 0; kw < KS; ++kw) acc[kw][0] = acc[kw][1] = acc[kw][2] = acc[kw][3] = 0.f;
  const int P = g.ho * g.wo;
  const int n0 = blockIdx.x * chunk, n1 = min(g.n, n0 + chunk);
  for (int n = n0; n < n1; ++n) {
    __syncthreads();
    load_padded(xs, x, n, g.h, g.w, g.ci, Hp, Wp, g.pt, g.pl);
    load_dy_padded(ds, dy + (size_t)n * P * g.co, P, g.co, co4);
    __syncthreads();
    if (active) {
      for (int ho = ph; ho < g.ho; ho += PH) {
        const float* xr = xs + ((size_t)ci * Hp + ho + kh) * Wp;
        float xv[KS];
#pragma unroll
        for (int kw = 0; kw < KS - 1; ++kw) xv[kw + 1] = xr[kw];
        for (int wo = 0; wo < g.wo; ++wo) {
#pragma unroll
          for (int kw = 0; kw < KS - 1; ++kw) xv[kw] = xv[kw + 1];
          xv[KS - 1] = xr[wo + KS - 1];
          const float4 d = *reinterpret_cast<const float4*>(ds + (ho * g.wo + wo) * co4 + q * 4);
#pragma unroll
          for (int kw = 0; kw < KS; ++kw) {
            acc[kw][0] = fmaf(xv[kw], d.x, acc[kw][0]);
            acc[kw][1] = fmaf(xv[kw], d.y, acc[kw][1]);
            acc[kw][2] = fmaf(xv[kw], d.z, acc[kw][2]);
            acc[kw][3] = fmaf(xv[kw], d.w, acc[kw][3]);
          }
        }
      }
    }
  }
  __syncthreads();
  float* red = sm;  // [PH][KS*KS*ci*co4]
  const int O = KS * KS * g.ci * co4;
  if (active) {
#pragma unroll
    for (int kw = 0; kw < KS; ++kw)
      for (int j = 0; j < 4; ++j) red[ph * O + ((kh * KS + kw) * g.ci + ci) * co4 + q * 4 + j] = acc[kw][j];
  }
  __syncthreads();
  const int OO = KS * KS * g.ci * g.co;
  for (int o = threadIdx.x; o < OO; o += blockDim.x) {
    const int co = o % g.co, rr = o / g.co;
    float s_ = red[rr * co4 + co];
    for (int h = 1; h < PH; ++h) s_ = __fadd_rn(s_, red[h * O + rr * co4 + co]);
    part[(size_t)blockIdx.x * OO + o] = s_;
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
  smem_attr((const void*)f, SMEM_LIMIT);
}

constexpr int RT_PX = 4;

RtGeom rt_geom_fwd(const ConvGeom& g, int px = RT_PX) {
  RtGeom r{};
  r.n = g.n; r.hin = g.h; r.win = g.w; r.cin = g.ci;
  r.hout = g.ho; r.wout = g.wo; r.cout = g.co;
  r.pt = g.pt; r.pl = g.pl; r.wcin = g.ci; r.wcout = g.co;
  r.Hp = g.ho + g.kh - 1;
  r.Wp = ((g.wo + px - 1) / px * px + g.kw - 1) | 1;  // odd row pitch (bank spread)
  return r;
}
RtGeom rt_geom_bwdin(const ConvGeom& g, int px = RT_PX) {
  RtGeom r{};
  r.n = g.n; r.hin = g.ho; r.win = g.wo; r.cin = g.co;
  r.hout = g.h; r.wout = g.w; r.cout = g.ci;
  r.pt = g.kh - 1 - g.pt; r.pl = g.kw - 1 - g.pl; r.wcin = g.ci; r.wcout = g.co;
  r.Hp = g.h + g.kh - 1;
  r.Wp = ((g.w + px - 1) / px * px + g.kw - 1) | 1;
  return r;
}
bool rt_ok(const ConvGeom& g) {  // stride 1, square 5x5 or 3x3 taps
  return g.sh == 1 && g.sw == 1 && g.kh == g.kw && (g.kh == 5 || g.kh == 3);
}

// images per block iteration: enough work items for the block (>= 2 per thread)
// within the shared-memory budget
constexpr size_t RT_SMEM = 110 * 1024;
int rt_img(const RtGeom& r, int cop, int ks, int px = RT_PX) {
  const size_t wbytes = (size_t)ks * ks * r.cin * cop * 4, ibytes = (size_t)r.cin * r.Hp * r.Wp * 4;
  if (wbytes + ibytes > RT_SMEM) return 0;
  const int per = r.hout * ((r.wout + px - 1) / px);
  const int want = std::max(1, (256 + per - 1) / per);  // one item per thread; several blocks per SM
  return (int)std::max<size_t>(1, std::min<size_t>(want, (RT_SMEM - wbytes) / ibytes));
}

template <int COP, bool FLIP, int PX = RT_PX>
cudaError_t launch_rt(const float* x, const float* w, float* y, const RtGeom& r, int ks, int num_sms, cudaStream_t s) {
  const int IMG = rt_img(r, COP, ks, PX);
  const size_t smem = ((size_t)ks * ks * r.cin * COP + (size_t)IMG * r.cin * r.Hp * r.Wp) * 4;
  const int bps = std::max(1, std::min(4, (int)((224 * 1024) / (smem + 1024))));
  const int grid = std::max(1, std::min((r.n + IMG - 1) / IMG, num_sms * bps));
  if (ks == 5) {
    smem_attr((const void*)conv_rt_kernel<COP, 5, PX, FLIP>, (int)RT_SMEM);
    conv_rt_kernel<COP, 5, PX, FLIP><<<grid, 256, smem, s>>>(x, w, y, r, IMG);
  } else {
    smem_attr((const void*)conv_rt_kernel<COP, 3, PX, FLIP>, (int)RT_SMEM);
    conv_rt_kernel<COP, 3, PX, FLIP><<<grid, 256, smem, s>>>(x, w, y, r, IMG);
  }
  return cudaGetLastError();
}

void bwdk_rt_geom(const ConvGeom& g, int* PH, int* units) {
  *units = g.kh * g.ci * ((g.co + 3) / 4);
  *PH = std::max(1, std::min(g.ho, 256 / std::max(1, *units)));
}
size_t bwdk_rt_smem(const ConvGeom& g) {
  int PH, units;
  bwdk_rt_geom(g, &PH, &units);
  const int co4 = (g.co + 3) / 4 * 4;
  const int Hp = g.ho + g.kh - 1, Wp = g.wo + g.kw - 1;
  size_t img = ((size_t)g.ci * Hp * Wp + 3) / 4 * 4 + (size_t)g.ho * g.wo * co4;
  size_t red = (size_t)PH * g.kh * g.kw * g.ci * co4;
  return std::max(img, red) * 4;
}
bool bwdk_rt_ok(const ConvGeom& g) {
  int PH, units;
  bwdk_rt_geom(g, &PH, &units);
  return rt_ok(g) && units <= 256 && bwdk_rt_smem(g) <= SMEM_LIMIT;
}

}  // namespace

bool conv_small_fwd_ok(const ConvGeom& g) { return co_pad(g.co) && fwd_smem(g) <= SMEM_LIMIT; }
bool conv_small_bwdin_ok(const ConvGeom& g) { return co_pad(g.ci) && bwdin_smem(g) <= SMEM_LIMIT; }
bool conv_small_bwdk_ok(const ConvGeom& g) {
  if (bwdk_rt_ok(g)) return true;
  int PH, units;
  bwdk_geom(g, &PH, &units);
  return g.ci <= 8 && units <= 256 && bwdk_smem(g) <= SMEM_LIMIT;
}
size_t conv_small_bwdk_ws(const ConvGeom& g, int num_sms) {
  return (size_t)bwdk_blocks(g, num_sms) * g.kh * g.kw * g.ci * g.co;
}

cudaError_t launch_conv_small_fwd(const float* x, const float* w, float* y, const ConvGeom& g, int num_sms,
                                  cudaStream_t s) {
  // register tiling over 4 pixels x all (padded) output channels, several images per block
  if (rt_ok(g) && !getenv("CG_CONV_NO_RT")) {
    const RtGeom r = rt_geom_fwd(g);
    // (<= 8 channels only: at 16 the 128 registers per thread cost more occupancy than the
    // tiling saves -- C4 conv2: 320 us vs 291 us for conv_fwd_img)
    static const int px8 = getenv("CG_RT_PX8") ? atoi(getenv("CG_RT_PX8")) : 2;  // (C4 conv1: 2 best of 2 / 4 / 8)
    if (co_pad(g.co) == 8) {
      const RtGeom r8 = rt_geom_fwd(g, px8);
      if (px8 == 8 && rt_img(r8, 8, g.kh, 8)) return launch_rt<8, false, 8>(x, w, y, r8, g.kh, num_sms, s);
      if (px8 == 2 && rt_img(r8, 8, g.kh, 2)) return launch_rt<8, false, 2>(x, w, y, r8, g.kh, num_sms, s);
      if (rt_img(r, 8, g.kh)) return launch_rt<8, false>(x, w, y, r, g.kh, num_sms, s);
    }
    if (co_pad(g.co) == 16) {  // 2 pixels x 16 channels per thread (C4 conv2: 247 vs 293 us for conv_fwd_img)
      const RtGeom r2 = rt_geom_fwd(g, 2);
      if (rt_img(r2, 16, g.kh, 2)) return launch_rt<16, false, 2>(x, w, y, r2, g.kh, num_sms, s);
    }
  }
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
  // register-tiled transposed correlation (several images per block): C4's
  // 16 -> 6-channel backward-input 366 us vs 427 us for conv_bwdin_img
  if (rt_ok(g) && co_pad(g.ci) == 8 && g.co <= 16 && !getenv("CG_CONV_NO_RT")) {
    static const int pxf = getenv("CG_RT_PXF") ? atoi(getenv("CG_RT_PXF")) : 4;  // (measurement switch)
    const RtGeom r = rt_geom_bwdin(g, pxf);
    if (pxf == 8 && rt_img(r, 8, g.kh, 8)) return launch_rt<8, true, 8>(dy, w, dx, r, g.kh, num_sms, s);
    if (pxf == 2 && rt_img(r, 8, g.kh, 2)) return launch_rt<8, true, 2>(dy, w, dx, r, g.kh, num_sms, s);
    if (pxf == 4 && rt_img(r, 8, g.kh)) return launch_rt<8, true>(dy, w, dx, r, g.kh, num_sms, s);
  }
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
  if (bwdk_rt_ok(g)) {
    int PH, units;
    bwdk_rt_geom(g, &PH, &units);
    const int blocks = bwdk_blocks(g, num_sms);
    const int chunk = (g.n + blocks - 1) / blocks;
    const int nb = (g.n + chunk - 1) / chunk;
    const size_t smem = bwdk_rt_smem(g);
    const int Hp = g.ho + g.kh - 1, Wp = g.wo + g.kw - 1;
    if (g.kh == 5) {
      set_smem(conv_bwdk_rt_kernel<5>);
      conv_bwdk_rt_kernel<5><<<nb, 256, smem, s>>>(x, dy, ws, g, Hp, Wp, PH, chunk);
    } else {
      set_smem(conv_bwdk_rt_kernel<3>);
      conv_bwdk_rt_kernel<3><<<nb, 256, smem, s>>>(x, dy, ws, g, Hp, Wp, PH, chunk);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_reduce_finalize(ws, dw, (long long)g.kh * g.kw * g.ci * g.co, nb, 0, s);
  }
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
