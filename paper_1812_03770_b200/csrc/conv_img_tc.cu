// Few-channel, small-image convolutions on the 5th-generation tensor cores (sm_100a).
//
// A correlation of a stride-1 KS x KS kernel over small images (C4's LeNet
// layers: 28x28x1 -> 6, 14x14x6 -> 16, and the 16 -> 6 backward-input pass) is an
// implicit GEMM   out[q, n] = sum_k A[q, k] B[k, n]   with q = output pixel,
// k = (c, kh, kw) and n = output channel (<= 16).  The im2col operand A is never
// materialised: whole images are staged in shared memory (channel-planar, so
// adjacent pixels are adjacent words) and builder warps form each 128-pixel x
// 32-k slab from them with compile-time offsets (the geometry is a template),
// split it into TF32 hi/lo and write it to TENSOR MEMORY; the MMAs
// (tcgen05.mma.kind::tf32, M = 128, N = 16) take A from TMEM and B (the weights,
// split once per CTA) from shared memory.  3xTF32: hi.hi + hi.lo + lo.hi as in
// dot_tc.cu.
//
// Accuracy: the tensor core's fp32 accumulation truncates, so a 400-deep chain
// in one accumulator loses ~K/8 ulps (measured 1.6e-6 .. 2.5e-5 normwise on the
// DOT kernel).  Here each 32-deep k-block goes to a fresh TMEM accumulator and
// the epilogue warps add it into a register sum with round-to-nearest, so the
// truncation applies to 32-deep partials only (fp32-GEMM accuracy).  N <= 16
// makes that cheap: 16 registers per thread, one 8 KiB TMEM read per k-block.
//
// Work: persistent CTAs over units of G whole images (G*P pixels = T tiles of
// 128).  Warps: 0-3 image loaders (global NHWC -> planar smem, double-buffered),
// 4-7 and 8-11 two builder groups taking alternate k-blocks, 12-15 epilogue,
// 16 TMEM allocator + MMA issuer.  Deterministic: fixed summation order.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "conv_img_tc.h"

namespace cg {

namespace {

#include "tc_prims.cuh"

constexpr int CI_THREADS = 544;   // 17 warps
constexpr int CI_L = 6;           // A stages in TMEM (64 columns each: 32 hi + 32 lo)
constexpr int CI_ACOL = 32;       // TMEM columns 0..31: two 16-column accumulators

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT, bool FLIP>
struct CiGeo {
  static constexpr int K = CIN * KS * KS;
  static constexpr int NKB = (K + 31) / 32;
  static constexpr int P = OH * OW;            // output pixels per image
  // zero-padded planes: the window of every output pixel is in bounds (no masks)
  static constexpr int HP = OH + KS - 1, WP = OW + KS - 1;
  static constexpr int PLANE = HP * WP;
  static constexpr int IMGF = CIN * PLANE;     // floats per staged (padded) image
  static constexpr int SRCF = CIN * IH * IW;   // floats per source image
  static constexpr int B_BYTES = NKB * 4096;   // per k-block: hi tile 2 KiB + lo tile 2 KiB
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]),
      "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT, bool FLIP>
__global__ void __launch_bounds__(CI_THREADS, 1)
    conv_img_tc_kernel(const float* __restrict__ in, const float* __restrict__ w, float* __restrict__ out, int nimgs,
                       int G, int T) {
  using Geo = CiGeo<CIN, KS, IH, IW, OH, OW, PT, PL, COUT, FLIP>;
  constexpr int K = Geo::K, NKB = Geo::NKB, P = Geo::P, PLANE = Geo::PLANE, IMGF = Geo::IMGF, WP = Geo::WP;
  constexpr int SRCF = Geo::SRCF;
  extern __shared__ uint8_t smem_raw[];
  // align to 1024 B by pointer arithmetic on the __shared__ array (keeps the shared
  // address space visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  float* imgs = reinterpret_cast<float*>(smem + Geo::B_BYTES);   // 2 buffers x G images
  const int buf_floats = G * IMGF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Geo::B_BYTES + 2 * (size_t)buf_floats * 4);
  const uint32_t bar0 = smem_u32(bars);
  auto imgfull = [&](int b) { return bar0 + 8u * b; };
  auto imgfree = [&](int b) { return bar0 + 8u * (2 + b); };
  auto conv = [&](int l) { return bar0 + 8u * (4 + l); };
  auto lofree = [&](int l) { return bar0 + 8u * (4 + CI_L + l); };
  auto tfull = [&](int b) { return bar0 + 8u * (4 + 2 * CI_L + b); };
  auto tempty = [&](int b) { return bar0 + 8u * (6 + 2 * CI_L + b); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * CI_L);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int units = (nimgs + G - 1) / G;

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(imgfull(b), 128);  // every loader thread
      mbar_init(imgfree(b), 8);    // every builder warp
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), 4);     // the epilogue warps
    }
    for (int l = 0; l < CI_L; ++l) {
      mbar_init(conv(l), 4);       // the builder warps of one group
      mbar_init(lofree(l), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // B (weights) for every k-block, split once: K-major SWIZZLE_128B tiles of 16 rows
  // (n) x 32 k; 16-byte chunk c of row n at chunk c ^ (n & 7).  k = (c, kh, kw).
  for (int e = threadIdx.x; e < NKB * 16 * 32; e += blockDim.x) {
    const int kb = e / 512, rem = e % 512, n = rem / 32, kl = rem % 32, k = kb * 32 + kl;
    float v = 0.f;
    if (k < K && n < COUT) {
      const int c = k / (KS * KS), t = k % (KS * KS), kh = t / KS, kw = t % KS;
      if (!FLIP) {  // w [KS][KS][CIN][COUT]
        v = __ldg(w + ((size_t)(kh * KS + kw) * CIN + c) * COUT + n);
      } else {      // w [KS][KS][COUT (= ci of the forward)][CIN (= co)], flipped taps
        v = __ldg(w + ((size_t)((KS - 1 - kh) * KS + (KS - 1 - kw)) * COUT + n) * CIN + c);
      }
    }
    const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    const float lo = __fsub_rn(v, hi);
    const int off = n * 128 + (((kl >> 2) ^ (n & 7)) << 4) + (kl & 3) * 4;
    *reinterpret_cast<float*>(smem + kb * 4096 + off) = hi;
    *reinterpret_cast<float*>(smem + kb * 4096 + 2048 + off) = lo;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core
  // the padding of both image buffers stays zero: the loaders only rewrite interiors
  for (int e = threadIdx.x; e < 2 * buf_floats; e += blockDim.x) imgs[e] = 0.f;
  if (warp == 16) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ---------------- loaders: G images, global NHWC (contiguous) -> planar [c][h][w]
    int j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int b = j & 1;
      const int n0 = u * G, nimg = min(G, nimgs - n0);
      mbar_wait(imgfree(b), ((j >> 1) & 1) ^ 1);
      float* dst = imgs + b * buf_floats;
      const float* src = in + (size_t)n0 * SRCF;
      const int tot = nimg * SRCF;
      for (int e0 = threadIdx.x; e0 < tot; e0 += 8 * 128) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = e0 + q * 128;
          v[q] = e < tot ? __ldg(src + e) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = e0 + q * 128;
          if (e < tot) {
            const int im = e / SRCF, r = e - im * SRCF;        // r = (h * IW + w) * CIN + c
            const int pix = r / CIN, c = r - pix * CIN, h = pix / IW, ww = pix - h * IW;
            dst[im * IMGF + c * PLANE + (h + PT) * WP + ww + PL] = v[q];
          }
        }
      }
      mbar_arrive(imgfull(b));
    }
  } else if (warp < 12) {
    // ---------------- builders: A slab (128 pixels x 32 k) -> TMEM hi / lo columns
    const int grp = warp < 8 ? 0 : 1;
    const int wq = warp % 4, rr = wq * 32 + lane;  // TMEM lane quadrant / tile row
    int it = 0, j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int b = j & 1;
      const int n0 = u * G, nimg = min(G, nimgs - n0);
      mbar_wait(imgfull(b), (j >> 1) & 1);
      const float* img = imgs + b * buf_floats;
      for (int t = 0; t < T; ++t, it += NKB) {
        // this row's output pixel: image g, (oh, ow); its window starts at (oh, ow) of the
        // padded planes (rows past the unit read image 0: their outputs are not stored)
        const int q = t * 128 + rr;
        const int g = q / P, p = q - g * P, oh = p / OW, ow = p - oh * OW;
        const float* base = img + (g < nimg ? g * IMGF + oh * WP + ow : 0);
#pragma unroll
        for (int kb = 0; kb < NKB; ++kb) {
          const int step = it + kb;
          if ((step & 1) != grp) continue;
          const int l = step % CI_L;
          mbar_wait(lofree(l), ((step / CI_L) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          uint32_t hv[32], lv[32];
#pragma unroll
          for (int kl = 0; kl < 32; ++kl) {
            const int k = kb * 32 + kl;
            float v = 0.f;
            if (k < K) {
              const int c = k / (KS * KS), tt = k % (KS * KS), kh = tt / KS, kw = tt % KS;
              v = base[c * PLANE + kh * WP + kw];
            }
            const uint32_t h = __float_as_uint(v) & 0xFFFFE000u;
            hv[kl] = h;
            lv[kl] = __float_as_uint(__fsub_rn(v, __uint_as_float(h)));
          }
          const uint32_t ta = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(CI_ACOL + l * 64);
          tmem_st32(ta, hv);
          tmem_st32(ta + 32, lv);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(conv(l));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(imgfree(b));  // this warp has read the images of unit j
    }
  } else if (warp < 16) {
    // ---------------- epilogue: each k-block's accumulator -> round-to-nearest register sum
    const int wq = warp % 4, rr = wq * 32 + lane;
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int n0 = u * G, nimg = min(G, nimgs - n0);
      for (int t = 0; t < T; ++t) {
        float sum[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) sum[i] = 0.f;
        for (int kb = 0; kb < NKB; ++kb, ++it) {
          const int b = it & 1;
          mbar_wait(tfull(b), (it >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          float v[16];
          tmem_ld16(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(b * 16), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) sum[i] = __fadd_rn(sum[i], v[i]);
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty(b));
        }
        const int q = t * 128 + rr;
        if (q < nimg * P) {
          float* o = out + ((size_t)n0 * P + q) * COUT;
          if (COUT % 4 == 0) {
#pragma unroll
            for (int i = 0; i < COUT; i += 4)
              *reinterpret_cast<float4*>(o + i) = make_float4(sum[i], sum[i + 1], sum[i + 2], sum[i + 3]);
          } else if (COUT % 2 == 0) {
#pragma unroll
            for (int i = 0; i < COUT; i += 2) *reinterpret_cast<float2*>(o + i) = make_float2(sum[i], sum[i + 1]);
          } else {
#pragma unroll
            for (int i = 0; i < COUT; ++i) o[i] = sum[i];
          }
        }
      }
    }
  } else {
    // ---------------- warp 16: MMA issuer (whole warp walks the loop; one elected lane issues)
    // instruction descriptor: D f32, A / B tf32, A (TMEM) and B K-major, N = 16, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x)
      for (int t = 0; t < T; ++t)
        for (int kb = 0; kb < NKB; ++kb, ++it) {
          const int l = it % CI_L, b = it & 1;
          mbar_wait_warp(tempty(b), ((it >> 1) & 1) ^ 1);  // the epilogue has read this accumulator
          mbar_wait_warp(conv(l), (it / CI_L) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t d = tm + (uint32_t)(b * 16);
          const uint32_t ahi = tm + (uint32_t)(CI_ACOL + l * 64), alo = ahi + 32;
          const uint32_t bt = sbase + (uint32_t)(kb * 4096);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t dhi = sdesc(bt + kk * 32, 16, 1024, 2), dlo = sdesc(bt + 2048 + kk * 32, 16, 1024, 2);
            // small terms first, then the leading hi.hi product; a fresh accumulator per k-block
            mma_tf32_e<1>(d, alo + kk * 8, dhi, idesc, kk > 0 ? 1u : 0u);
            mma_tf32_e<1>(d, ahi + kk * 8, dlo, idesc, 1u);
            mma_tf32_e<1>(d, ahi + kk * 8, dhi, idesc, 1u);
          }
          mma_commit_e<1>(lofree(l));
          mma_commit_e<1>(tfull(b));
        }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 16) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------- backward-input as GEMM + col2im
// dx[h,w,ci] = sum_{kh,kw,co} dy[h-kh+PT, w-kw+PL, co] w[kh,kw,ci,co]  (stride 1).
// Per image: C[q, j] = sum_co dy[q, co] w[j, co] with q = dy pixel and
// j = (kh, kw, ci) -- a K = CO GEMM on the tensor cores (A = the dy rows straight
// from global memory, no im2col) -- then dx[h, w, ci] = sum over the in-bounds
// taps (kh, kw ascending, fixed order: deterministic) of C[(h-kh+PT, w-kw+PL), (kh, kw, ci)]
// from a shared-memory copy of C.  One 128-row tile = one image (HO*WO <= 128).
// Warps 0-3 builders, 4-11 epilogue (TMEM -> smem, col2im sums), 12 MMA.
constexpr int BI_THREADS = 416;
constexpr int BI_L = 4;                 // A stages (32 TMEM columns: 16 hi + 16 lo)

template <int CO, int KS, int HO, int WO, int H, int W, int PT, int PL, int CI>
struct BiGeo {
  static constexpr int NJ = KS * KS * CI;                // GEMM N (real)
  static constexpr int NN = (NJ + 15) / 16 * 16;         // MMA N (multiple of 16)
  static constexpr int P = HO * WO;                      // dy pixels per image (<= 128)
  static constexpr int CP = NJ | 1;                      // odd row pitch of C in smem
  static constexpr int B_BYTES = NN * 128 * 2;           // hi + lo tiles, K-major SW128 (K padded to 32)
  static constexpr int C_FLOATS = 128 * CP;
  static constexpr int ACC = NN;                         // TMEM columns per accumulator
  static constexpr int ACOL = 2 * NN;                    // first A-stage column
  static_assert(P <= 128, "one image per tile");
  static_assert(CO == 16, "K = 16: two TF32 k-slices");
  static_assert(2 * NN + BI_L * 32 <= 512, "TMEM");
};

template <int CO, int KS, int HO, int WO, int H, int W, int PT, int PL, int CI>
__global__ void __launch_bounds__(BI_THREADS, 1)
    conv_bwdin_col2im_kernel(const float* __restrict__ dy, const float* __restrict__ w, float* __restrict__ dx,
                             int nimgs) {
  using Geo = BiGeo<CO, KS, HO, WO, H, W, PT, PL, CI>;
  constexpr int NJ = Geo::NJ, NN = Geo::NN, P = Geo::P, CP = Geo::CP;
  extern __shared__ uint8_t smem_raw[];
  // align to 1024 B by pointer arithmetic on the __shared__ array (keeps the shared
  // address space visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  float* Cs = reinterpret_cast<float*>(smem + Geo::B_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Geo::B_BYTES + (size_t)Geo::C_FLOATS * 4);
  const uint32_t bar0 = smem_u32(bars);
  auto conv = [&](int l) { return bar0 + 8u * l; };
  auto lofree = [&](int l) { return bar0 + 8u * (BI_L + l); };
  auto tfull = [&](int b) { return bar0 + 8u * (2 * BI_L + b); };
  auto tempty = [&](int b) { return bar0 + 8u * (2 * BI_L + 2 + b); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * BI_L + 4);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int l = 0; l < BI_L; ++l) {
      mbar_init(conv(l), 4);
      mbar_init(lofree(l), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), 8);  // the 8 epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // B[k = co][n = j]: K-major SWIZZLE_128B rows of 32 k (k >= 16 zero), row n at n * 128 B
  for (int e = threadIdx.x; e < NN * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;
    const float v = (n < NJ && k < CO) ? __ldg(w + (size_t)n * CO + k) : 0.f;  // w [kh][kw][ci][co]: row j = (kh,kw,ci)
    const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    const int off = n * 128 + (((k >> 2) ^ (n & 7)) << 4) + (k & 3) * 4;
    *reinterpret_cast<float*>(smem + off) = hi;
    *reinterpret_cast<float*>(smem + NN * 128 + off) = __fsub_rn(v, hi);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 12) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ---------------- builders: dy row q (16 channels, 64 B) -> TMEM hi / lo (next image prefetched)
    const int rr = warp * 32 + lane;
    int it = 0;
    float4 nx[4];
    auto fetch = [&](int n, float4 (&v)[4]) {
      if (n < nimgs && rr < P) {
        const float4* src = reinterpret_cast<const float4*>(dy + ((size_t)n * P + rr) * CO);
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = __ldg(src + i);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    fetch(blockIdx.x, nx);
    for (int n = blockIdx.x; n < nimgs; n += gridDim.x, ++it) {
      float4 cur[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) cur[i] = nx[i];
      fetch(n + gridDim.x, nx);
      const int l = it % BI_L;
      mbar_wait(lofree(l), ((it / BI_L) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t hv[16], lv[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float c4[4] = {cur[i].x, cur[i].y, cur[i].z, cur[i].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t h = __float_as_uint(c4[q]) & 0xFFFFE000u;
          hv[4 * i + q] = h;
          lv[4 * i + q] = __float_as_uint(__fsub_rn(c4[q], __uint_as_float(h)));
        }
      }
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(Geo::ACOL + l * 32);
      tmem_st16(ta, hv);
      tmem_st16(ta + 16, lv);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(conv(l));
    }
  } else if (warp < 12) {
    // ---------------- epilogue: C (TMEM) -> smem, then dx by fixed-order col2im sums
    const int wq = warp % 4, half = (warp - 4) / 4;   // TMEM lane quadrant; column half
    const int rr = wq * 32 + lane;
    const int et = threadIdx.x - 128;                  // 0..255
    int it = 0;
    for (int n = blockIdx.x; n < nimgs; n += gridDim.x, ++it) {
      const int b = it & 1;
      mbar_wait(tfull(b), (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("bar.sync 1, 256;" ::: "memory");  // the previous image's col2im reads of Cs are done
      constexpr int NCH = NN / 16, H0 = (NCH + 1) / 2;
      for (int ch = half ? H0 : 0; ch < (half ? NCH : H0); ++ch) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(b * Geo::ACC + ch * 16), v);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (ch * 16 + i < NJ) Cs[rr * CP + ch * 16 + i] = v[i];
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty(b));
      asm volatile("bar.sync 1, 256;" ::: "memory");  // Cs complete
      float* o = dx + (size_t)n * H * W * CI;
      for (int e = et; e < H * W * CI; e += 256) {
        const int pix = e / CI, ci = e - pix * CI, h = pix / W, ww = pix - h * W;
        float s = 0.f;
#pragma unroll
        for (int kh = 0; kh < KS; ++kh) {
          const int oh = h - kh + PT;
          if ((unsigned)oh >= (unsigned)HO) continue;
#pragma unroll
          for (int kw = 0; kw < KS; ++kw) {
            const int ow = ww - kw + PL;
            if ((unsigned)ow < (unsigned)WO) s = __fadd_rn(s, Cs[(oh * WO + ow) * CP + (kh * KS + kw) * CI + ci]);
          }
        }
        o[e] = s;
      }
    }
  } else {
    // ---------------- warp 12: MMA issuer.  D f32, A / B tf32, both K-major, N = NN, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    int it = 0;
    for (int n = blockIdx.x; n < nimgs; n += gridDim.x, ++it) {
      const int l = it % BI_L, b = it & 1;
      mbar_wait_warp(tempty(b), ((it >> 1) & 1) ^ 1);
      mbar_wait_warp(conv(l), (it / BI_L) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tm + (uint32_t)(b * Geo::ACC);
      const uint32_t ahi = tm + (uint32_t)(Geo::ACOL + l * 32), alo = ahi + 16;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint64_t dhi = sdesc(sbase + kk * 32, 16, 1024, 2), dlo = sdesc(sbase + NN * 128 + kk * 32, 16, 1024, 2);
        mma_tf32_e<1>(d, alo + kk * 8, dhi, idesc, kk > 0 ? 1u : 0u);
        mma_tf32_e<1>(d, ahi + kk * 8, dlo, idesc, 1u);
        mma_tf32_e<1>(d, ahi + kk * 8, dhi, idesc, 1u);
      }
      mma_commit_e<1>(lofree(l));
      mma_commit_e<1>(tfull(b));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 12) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int CO, int KS, int HO, int WO, int H, int W, int PT, int PL, int CI>
cudaError_t launch_bwdin(const float* dy, const float* w, float* dx, int n, int num_sms, cudaStream_t s) {
  using Geo = BiGeo<CO, KS, HO, WO, H, W, PT, PL, CI>;
  const size_t smem = 1024 + Geo::B_BYTES + (size_t)Geo::C_FLOATS * 4 + 256;
  auto kern = conv_bwdin_col2im_kernel<CO, KS, HO, WO, H, W, PT, PL, CI>;
  cudaError_t e = smem_attr((const void*)kern, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<std::min(n, num_sms), BI_THREADS, smem, s>>>(dy, w, dx, n);
  return cudaGetLastError();
}

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT, bool FLIP>
cudaError_t launch_geo(const float* in, const float* w, float* out, int n, int num_sms, cudaStream_t s) {
  using Geo = CiGeo<CIN, KS, IH, IW, OH, OW, PT, PL, COUT, FLIP>;
  // images per unit: the largest G (<= 32) whose double-buffered images fit, preferring
  // little padding in the last 128-pixel tile of a unit
  constexpr size_t budget = 200 * 1024;
  int best_g = 1;
  double best_cost = 1e30;
  for (int G = 1; G <= 32; ++G) {
    const size_t bytes = Geo::B_BYTES + 2 * (size_t)G * Geo::IMGF * 4;
    if (bytes > budget) break;
    const int T = (G * Geo::P + 127) / 128;
    const double waste = (double)T * 128 / ((double)G * Geo::P);   // padded rows per real row
    const double cost = waste * (1.0 + 0.5 / G);                     // + per-unit overhead
    if (cost < best_cost) { best_cost = cost; best_g = G; }
  }
  const int G = best_g, T = (G * Geo::P + 127) / 128;
  const size_t smem = 1024 + Geo::B_BYTES + 2 * (size_t)G * Geo::IMGF * 4 + 256;
  auto kern = conv_img_tc_kernel<CIN, KS, IH, IW, OH, OW, PT, PL, COUT, FLIP>;
  cudaError_t e = smem_attr((const void*)kern, (int)smem);
  if (e != cudaSuccess) return e;
  const int units = (n + G - 1) / G;
  kern<<<std::min(units, num_sms), CI_THREADS, smem, s>>>(in, w, out, n, G, T);
  return cudaGetLastError();
}

// compiled geometries: C4 (LeNet on 28 x 28 x 1)
enum CiKind { CI_NONE, CI_C4_CONV1, CI_C4_CONV2, CI_C4_CONV2_BWDIN };

CiKind kind_of(const ConvGeom& g, bool flip) {
  if (g.sh != 1 || g.sw != 1 || g.kh != 5 || g.kw != 5) return CI_NONE;
  if (!flip && g.h == 28 && g.w == 28 && g.ci == 1 && g.co == 6 && g.ho == 28 && g.wo == 28 && g.pt == 2 && g.pl == 2)
    return CI_C4_CONV1;
  if (!flip && g.h == 14 && g.w == 14 && g.ci == 6 && g.co == 16 && g.ho == 10 && g.wo == 10 && g.pt == 0 && g.pl == 0)
    return CI_C4_CONV2;
  if (flip && g.h == 14 && g.w == 14 && g.ci == 6 && g.co == 16 && g.ho == 10 && g.wo == 10 && g.pt == 0 && g.pl == 0)
    return CI_C4_CONV2_BWDIN;
  return CI_NONE;
}

}  // namespace

bool conv_img_tc_supported(const ConvGeom& g, bool flip) {
  return kind_of(g, flip) != CI_NONE && !getenv("CG_NO_CONV_IMG_TC");
}

cudaError_t launch_conv_img_tc(const float* in, const float* w, float* out, const ConvGeom& g, bool flip, int num_sms,
                               cudaStream_t s) {
  switch (kind_of(g, flip)) {
    case CI_C4_CONV1:  // x [n,28,28,1] (*) w [5,5,1,6], SAME
      return launch_geo<1, 5, 28, 28, 28, 28, 2, 2, 6, false>(in, w, out, g.n, num_sms, s);
    case CI_C4_CONV2:  // p1 [n,14,14,6] (*) w [5,5,6,16], VALID
      return launch_geo<6, 5, 14, 14, 10, 10, 0, 0, 16, false>(in, w, out, g.n, num_sms, s);
    case CI_C4_CONV2_BWDIN:  // dy [n,10,10,16], w [5,5,6,16] -> dx [n,14,14,6] (VALID forward)
      return launch_bwdin<16, 5, 10, 10, 14, 14, 0, 0, 6>(in, w, out, g.n, num_sms, s);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace cg
