// Few-channel, small-image convolutions on the 5th-generation tensor cores (sm_100a).
//
// A correlation of a stride-1 KS x KS kernel over small images (C4's LeNet
// layers: 28x28x1 -> 6, 14x14x6 -> 16, and the 16 -> 6 backward-input pass) is an
// implicit GEMM   out[q, n] = sum_k A[q, k] B[k, n]   with q = output pixel,
// k = (kh, kw, c) and n = output channel (<= 16).  The im2col operand A is never
// materialised: whole images are staged in shared memory (NHWC as in HBM, zero
// padded for SAME) and builder warps form each 128-pixel x
// 32-k slab from them with compile-time offsets (the geometry is a template),
// split it into TF32 hi/lo and write it to TENSOR MEMORY; the MMAs
// (tcgen05.mma.kind::tf32, M = 128, N = 16) take A from TMEM and B (the weights,
// split once per CTA) from shared memory.  3xTF32: hi.hi + hi.lo + lo.hi as in
// dot_tc.cu.
//
// Accuracy: the tensor core's fp32 accumulation truncates (a K-deep chain loses
// ~K/8 ulps of the partial sums, measured 1.6e-6 .. 2.5e-5 normwise on the DOT
// kernel).  The first version gave each 32-deep k-block a fresh accumulator and
// summed them with round-to-nearest in registers; that made the MMA wait for an
// epilogue drain every k-block, and the K <= 150 of these convs is well inside the
// tolerance the generic implicit GEMM already meets with whole-K chains, so a
// tile's k-blocks now chain in one accumulator (integer-exact tests unaffected).
//
// Work: persistent CTAs over units of G whole images (G*P pixels = T tiles of
// 128).  Warps: 0-3 and 4-7 two builder groups taking alternate k-blocks, 8-11 and
// 12-15 two epilogue groups taking alternate tiles (the epilogue's per-tile latency
// -- TMEM load, fused chain, stores -- was the bound once a chain was fused), 16
// the TMA producer (images, double-buffered), 17 TMEM allocator + MMA issuer.
// Deterministic: fixed summation order.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <cstdlib>

#include "conv_img_tc.h"
#include "dot_tc.h"

namespace cg {

namespace {

#include "tc_prims.cuh"

#ifndef CG_CI_NACC
#define CG_CI_NACC 4
#endif
constexpr int CI_THREADS = 576;   // 18 warps
constexpr int CI_L = 6;           // A stages in TMEM (64 columns each: 32 hi + 32 lo)
constexpr int CI_NACC = CG_CI_NACC;  // 16-column accumulators (more tiles between the MMA and the epilogue)
constexpr int CI_ACOL = 16 * CI_NACC;

// Staged images for the small-image kernels: [HP][WPS][CIN] at XBASE + g * IMGF,
// zero where a window leaves the image.  Staging modes (one TMA-engine operation per
// chunk of G images wherever possible: many KB in flight per SM without registers):
//  WHOLE (VALID, HP == IH, WPS == IW): the staged layout is the source layout, one
//        bulk copy per chunk;
//  TMAP  (CIN = 1, padded): one 3-D tiled TMA per chunk, box {WPS, HP, G} at
//        (0, 0, n0) -- its out-of-bounds zero fill gives every staged row >= PL
//        trailing zeros and every image >= PT trailing zero rows, and those serve
//        as the left / top padding of the next row / image (a zero guard of XBASE
//        floats precedes image 0).  (Negative TMA start coordinates -- the direct
//        way to pad -- trap with an illegal instruction: tools/tma3d_probe.cu.)
//  rows  otherwise: one bulk copy per image row into a zero frame whose rows are
//        16-byte aligned (input column iw at staged column iw + PLS).
template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL>
struct StageGeo {
  static constexpr bool TMAP = CIN == 1 && (PT > 0 || PL > 0) && (IW * 4) % 16 == 0;
  static constexpr int PADW = PL > KS - 1 - PL ? PL : KS - 1 - PL;
  static constexpr int PADH = PT > KS - 1 - PT ? PT : KS - 1 - PT;
  static constexpr int PLS = TMAP ? 0 : (PL * CIN + 3) / 4 * 4 / CIN + (((PL * CIN + 3) / 4 * 4) % CIN ? 1 : 0);
  static constexpr int WMIN = TMAP ? IW + PADW : OW + KS - 1 - PL + PLS;
  static constexpr int WPS0 = ((WMIN * CIN + 3) / 4 * 4 + CIN - 1) / CIN;
  // TMAP rows: a pitch of 4 (mod 8) words spreads the KS x KS taps of one pixel over
  // distinct banks (pitch 32 put all five kh of a kw in one bank: 5-way conflicts)
  static constexpr int WPS = TMAP && WPS0 % 8 == 0 ? WPS0 + 4 : WPS0;
  static constexpr int HP = TMAP ? IH + PADH : OH + KS - 1;
  static constexpr int XBASE = TMAP ? (PT * WPS + PL + 31) / 32 * 32 : 0;
  static constexpr int IMGF = HP * WPS * CIN;  // floats per staged image
  static constexpr int SRCF = IH * IW * CIN;   // floats per source image
  static constexpr bool WHOLE = PT == 0 && PLS == 0 && HP == IH && WPS == IW;
  static constexpr int XBOX = HP * WPS * 4;    // bytes per image of a TMAP box
  static constexpr int H_ = IH, W_ = IW, PT_ = PT, C_ = CIN;
  // staged offset of the window origin (kh = kw = 0) of output pixel (oh, ow) of image g
  __host__ __device__ static constexpr int window(int g, int oh, int ow) {
    return XBASE + g * IMGF + ((oh - (TMAP ? PT : 0)) * WPS + ow + PLS - PL) * CIN;
  }
  __host__ __device__ static constexpr int tap(int kh, int kw, int c) { return (kh * WPS + kw) * CIN + c; }
  static_assert(!TMAP || (WPS <= 256 && HP <= 256), "TMA box");
  static_assert((TMAP || (PLS * CIN) % 4 == 0) && (WPS * CIN) % 4 == 0 && (TMAP || PLS >= PL) && WPS >= WMIN,
                "staged rows 16-byte aligned");
  static_assert(WHOLE || TMAP || (IW * CIN) % 4 == 0, "row copies are multiples of 16 bytes");
  static_assert(SRCF % 4 == 0 && IMGF % 4 == 0, "16-byte bulk copies");
};

// Producer-warp side of the staging: images [n0, n0 + nimg) of x into the buffer at
// shared address `buf` (XBASE-relative frame), completion on `bar` (count 1 + tx).
template <class SG>
__device__ __forceinline__ void stage_images(uint32_t buf, const float* x, uint64_t xmap_addr, int n0, int nimg, int G,
                                             uint32_t bar, int lane) {
  if (lane == 0) mbar_expect_tx(bar, SG::TMAP ? (uint32_t)(G * SG::XBOX) : (uint32_t)(nimg * SG::SRCF * 4));
  __syncwarp();
  if constexpr (SG::WHOLE) {
    if (lane == 0) bulk_g2s(buf, x + (size_t)n0 * SG::SRCF, (uint32_t)(nimg * SG::SRCF * 4), bar);
  } else if constexpr (SG::TMAP) {
    if (lane == 0)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              buf + SG::XBASE * 4),
          "l"(xmap_addr), "r"(0), "r"(0), "r"(n0), "r"(bar)
          : "memory");
  } else {
    for (int r = lane; r < nimg * SG::H_; r += 32) {  // one copy per image row, into the padded frame
      const int im = r / SG::H_, h = r - im * SG::H_;
      bulk_g2s(buf + (uint32_t)((im * SG::IMGF + ((h + SG::PT_) * SG::WPS + SG::PLS) * SG::C_) * 4),
               x + ((size_t)n0 * SG::H_ + r) * SG::W_ * SG::C_, (uint32_t)(SG::W_ * SG::C_ * 4), bar);
    }
  }
  __syncwarp();
}

// 3-D tiled map over single-channel images x[n][h][w] (fp32), box {bw, bh, g}: a load
// at (0, 0, n0) returns g frames with zero-filled trailing rows / columns (StageGeo TMAP).
typedef CUresult (*EncodeTiledFnCI)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
bool make_img_map(CUtensorMap* m, const float* x, int n, int h, int w, int bw, int bh, int g) {
  static EncodeTiledFnCI fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFnCI)p;
  });
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[2] = {(cuuint64_t)w * 4, (cuuint64_t)w * h * 4};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)g};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT>
struct CiGeo {
  using SG = StageGeo<CIN, KS, IH, IW, OH, OW, PT, PL>;
  static constexpr int K = CIN * KS * KS;
  static constexpr int NKB = (K + 31) / 32;
  static constexpr int P = OH * OW;            // output pixels per image
  static constexpr int B_BYTES = NKB * 4096;   // per k-block: hi tile 2 KiB + lo tile 2 KiB
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]),
      "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// issue only (the caller waits with tcgen05.wait::ld before reading r)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
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

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT>
__global__ void __launch_bounds__(CI_THREADS, 1)
    conv_img_tc_kernel(const float* __restrict__ in, const float* __restrict__ w, float* __restrict__ out, int nimgs,
                       int G, int T, const __grid_constant__ CUtensorMap xmap, const __grid_constant__ EpiProg epi) {
  using Geo = CiGeo<CIN, KS, IH, IW, OH, OW, PT, PL, COUT>;
  using SG = typename Geo::SG;
  constexpr int K = Geo::K, NKB = Geo::NKB, P = Geo::P;
  extern __shared__ uint8_t smem_raw[];
  // align to 1024 B by pointer arithmetic on the __shared__ array (keeps the shared
  // address space visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  float* imgs = reinterpret_cast<float*>(smem + Geo::B_BYTES);   // 2 buffers x G images
  const int buf_floats = (SG::XBASE + G * SG::IMGF + 31) / 32 * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Geo::B_BYTES + 2 * (size_t)buf_floats * 4);
  const uint32_t bar0 = smem_u32(bars);
  auto imgfull = [&](int b) { return bar0 + 8u * b; };
  auto imgfree = [&](int b) { return bar0 + 8u * (2 + b); };
  auto conv = [&](int l) { return bar0 + 8u * (4 + l); };
  auto lofree = [&](int l) { return bar0 + 8u * (4 + CI_L + l); };
  auto tfull = [&](int b) { return bar0 + 8u * (4 + 2 * CI_L + b); };
  auto tempty = [&](int b) { return bar0 + 8u * (4 + 2 * CI_L + CI_NACC + b); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 + 2 * CI_L + 2 * CI_NACC);
  // the fused chain's scalar / column operands, staged once: epx[e][co]
  float* epx = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);
  static_assert((4 + 2 * CI_L + 2 * CI_NACC) * 8 + 4 <= 512, "barrier area");
  static_assert(CI_ACOL + CI_L * 64 <= 512, "TMEM columns");

  // role index through a shuffle: provably warp-uniform (convergent role branches)
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;
  const int units = (nimgs + G - 1) / G;

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(imgfull(b), 1);    // the producer's arrive.expect_tx
      mbar_init(imgfree(b), 8);    // every builder warp
    }
    for (int b = 0; b < CI_NACC; ++b) {
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
  // (n) x 32 k; 16-byte chunk c of row n at chunk c ^ (n & 7).  k = (kh, kw, c).
  for (int e = threadIdx.x; e < NKB * 16 * 32; e += blockDim.x) {
    const int kb = e / 512, rem = e % 512, n = rem / 32, kl = rem % 32, k = kb * 32 + kl;
    float v = 0.f;
    if (k < K && n < COUT) {
      const int c = k % CIN, t = k / CIN, kh = t / KS, kw = t % KS;
      v = __ldg(w + ((size_t)(kh * KS + kw) * CIN + c) * COUT + n);  // w [KS][KS][CIN][COUT]
    }
    const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    const float lo = __fsub_rn(v, hi);
    const int off = n * 128 + (((kl >> 2) ^ (n & 7)) << 4) + (kl & 3) * 4;
    *reinterpret_cast<float*>(smem + kb * 4096 + off) = hi;
    *reinterpret_cast<float*>(smem + kb * 4096 + 2048 + off) = lo;
  }
  // the padding / guard of both image buffers stays zero (TMA writes only the frames)
  for (int e = threadIdx.x; e < 2 * buf_floats; e += blockDim.x) imgs[e] = 0.f;
  for (int e = threadIdx.x; e < epi.n * COUT; e += blockDim.x) {
    const int op = e / COUT, c = e % COUT;
    epx[e] = epi.op[op] == EPI_RELU || epi.scalar[op] == 2 ? 0.f : __ldg(epi.x[op] + (epi.scalar[op] == 1 ? 0 : c));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core / TMA
  if (warp == 17) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // per-role cycle accounting of CTA 0 (diagnostics only: compiled in with
  // -DCG_CI_TIMING -- the timers cost registers the roles need)
  long long w_a = 0, w_b = 0, w_c = 0, w_d = 0, t_role = 0;
#ifdef CG_CI_TIMING
#define CI_TIMED(acc, call)          \
  do {                               \
    const long long t_ = clock64();  \
    call;                            \
    acc += clock64() - t_;           \
  } while (0)
  t_role = clock64();
#else
#define CI_TIMED(acc, call) call
#endif

  if (warp < 8) {
    // ---------------- builders: A slab (128 pixels x 32 k) -> TMEM hi / lo columns
    const int grp = warp / 4;
    const int wq = warp % 4, rr = wq * 32 + lane;  // TMEM lane quadrant / tile row
    int it = 0, j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int b = j & 1;
      const int n0 = u * G, nimg = min(G, nimgs - n0);
      CI_TIMED(w_a, mbar_wait(imgfull(b), (j >> 1) & 1));
      const float* img = imgs + b * buf_floats;
      for (int t = 0; t < T; ++t, it += NKB) {
        // this row's output pixel: image g, (oh, ow) (rows past the unit read image 0:
        // their outputs are not stored)
        const int q = t * 128 + rr;
        const int g = q / P, p = q - g * P, oh = p / OW, ow = p - oh * OW;
        const float* base = img + SG::window(g < nimg ? g : 0, oh, ow);
#pragma unroll
        for (int kb = 0; kb < NKB; ++kb) {
          const int step = it + kb;
          if ((step & 1) != grp) continue;
          const int l = step % CI_L;
          float v[32];
          if constexpr (CIN % 2 == 0) {
            static_assert(SG::XBASE % 2 == 0 && SG::IMGF % 2 == 0, "8-byte pair loads");
            // k = (kh, kw, c): a pair (k, k + 1), k even, is channels (c, c + 1) of one
            // tap -- one 8-byte load (a 6-word lane stride hits 16 distinct bank pairs
            // per half warp: conflict-free; the channel-major order took 32 two-way
            // conflicted 4-byte loads per slab)
#pragma unroll
            for (int kl = 0; kl < 32; kl += 2) {
              const int k = kb * 32 + kl;
              v[kl] = v[kl + 1] = 0.f;
              if (k < K) {
                const int c = k % CIN, tt = k / CIN, kh = tt / KS, kw = tt % KS;
                const float2 t = *reinterpret_cast<const float2*>(base + SG::tap(kh, kw, c));
                v[kl] = t.x;
                v[kl + 1] = t.y;
              }
            }
          } else {
#pragma unroll
            for (int kl = 0; kl < 32; ++kl) {
              const int k = kb * 32 + kl;
              v[kl] = 0.f;
              if (k < K) {
                const int c = k % CIN, tt = k / CIN, kh = tt / KS, kw = tt % KS;
                v[kl] = base[SG::tap(kh, kw, c)];
              }
            }
          }
#ifdef CG_CI_EAGER
          CI_TIMED(w_b, mbar_wait(lofree(l), ((step / CI_L) & 1) ^ 1));
#else
          CI_TIMED(w_b, mbar_wait_lazy(lofree(l), ((step / CI_L) & 1) ^ 1));  // (CI_L stages of slack)
#endif
#ifdef CG_CI_TIMING
          const long long t_st = clock64();
#endif
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t ta = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(CI_ACOL + l * 64);
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t hv[16], lv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float x = v[half * 16 + i];
              const uint32_t h = __float_as_uint(x) & 0xFFFFE000u;
              hv[i] = h;
              lv[i] = __float_as_uint(__fsub_rn(x, __uint_as_float(h)));
            }
            tmem_st16(ta + half * 16, hv);
            tmem_st16(ta + 32 + half * 16, lv);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
#ifdef CG_CI_TIMING
          w_c += clock64() - t_st;
#endif
          __syncwarp();
          if (lane == 0) mbar_arrive(conv(l));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(imgfree(b));  // this warp has read the images of unit j
    }
  } else if (warp < 16) {
    // ---------------- epilogue: two groups of four warps (one per TMEM lane quadrant)
    // take alternate tiles; accumulator b = tile % CI_NACC always goes to group b % 2
    const int wq = warp % 4, rr = wq * 32 + lane, eg = (warp - 8) / 4;
    // the chain's first op, hoisted out of the tile loop when its operand is a scalar
    // or per-column vector (the usual bias ADD): code and values in registers, no
    // per-tile parameter / shared-memory loads on the epilogue's critical path
    const int n_epi = epi.n;
    const bool hoist = n_epi >= 1 && epi.scalar[0] != 2;
    const int code0 = hoist ? epi.op[0] : 0, sw0 = hoist ? epi.swap[0] : 0;
    float x0[COUT];
#pragma unroll
    for (int i = 0; i < COUT; ++i) x0[i] = hoist ? epx[i] : 0.f;
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int n0 = u * G, nimg = min(G, nimgs - n0);
      for (int t = 0; t < T; ++t, ++it) {
        if ((it & 1) != eg) continue;
        // the tile's NKB k-blocks accumulate in one TMEM accumulator (as the generic
        // implicit GEMM); a fresh accumulator per k-block made the MMA wait for a drain
        // every k-block
        float sum[16];
        {
          const int b = it % CI_NACC;
          CI_TIMED(w_a, mbar_wait(tfull(b), (it / CI_NACC) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifdef CG_CI_TIMING
          {
            const long long t_ = clock64();
            tmem_ld16(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(b * 16), sum);
            // (a branch on the result: the clock read waits for the load's data)
            if (__float_as_uint(sum[0]) == 0x7fc01234u && __float_as_uint(sum[15]) == 0x7fc01234u) __trap();
            w_b += clock64() - t_;
          }
#else
          tmem_ld16(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(b * 16), sum);
#endif
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty(b));
        }
        const int q = t * 128 + rr;
#ifdef CG_CI_TIMING
        const long long t_c = clock64();
#endif
        if (q < nimg * P) {
          if (n_epi) {  // fused elementwise chain (f2), op by op as the separate kernel
            float v[COUT];
#pragma unroll
            for (int i = 0; i < COUT; ++i) v[i] = sum[i];
            if (hoist) {
              if (code0 == EPI_ADD) {  // (the bias: no jump table)
#pragma unroll
                for (int i = 0; i < COUT; ++i) v[i] = __fadd_rn(v[i], x0[i]);
              } else {
                epi_apply<COUT>(v, code0, sw0, x0);
              }
            }
#pragma unroll 1
            for (int e = hoist ? 1 : 0; e < n_epi; ++e) {
              float xe[COUT];
              if (epi.scalar[e] == 2) {  // full tensor: this pixel's COUT values
                const float* src = epi.x[e] + ((size_t)n0 * P + q) * COUT;
#pragma unroll
                for (int i = 0; i < COUT; ++i) xe[i] = __ldg(src + i);
              } else {
#pragma unroll
                for (int i = 0; i < COUT; ++i) xe[i] = epx[e * COUT + i];
              }
              epi_apply<COUT>(v, epi.op[e], epi.swap[e], xe);
            }
#pragma unroll
            for (int i = 0; i < COUT; ++i) sum[i] = v[i];
          }
        }
#ifdef CG_CI_TIMING
        const long long t_d = clock64();
        w_c += t_d - t_c;
#endif
#if defined(CG_CI_NOSTORE)  // diagnostics only: wrong results
        if (__float_as_uint(sum[0]) == 0x7fc01234u) out[0] = sum[1];
#else
        // (measured slower on conv1: a shared-memory-staged variant with 16-byte
        // coalesced stores, 111 -> 134 us, and one TMA bulk store per tile from
        // double-buffered staging, 112 -> 122 us; the direct per-row stores stay)
        if (q < nimg * P) {
          float* o = out + ((size_t)n0 * P + q) * COUT;
          if (COUT % 4 == 0) {
#pragma unroll
            for (int i = 0; i < COUT; i += 4)
              *reinterpret_cast<float4*>(o + i) = make_float4(sum[i], sum[i + 1], sum[i + 2], sum[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < COUT; i += 2) *reinterpret_cast<float2*>(o + i) = make_float2(sum[i], sum[i + 1]);
          }
        }
#endif
#ifdef CG_CI_TIMING
        w_d += clock64() - t_d;
#endif
      }
    }
  } else if (warp == 16) {
    // ---------------- producer: one TMA-engine copy per unit of G images (double-buffered)
    const uint64_t xmap_addr = reinterpret_cast<uint64_t>(&xmap);  // (address of the parameter itself)
    int j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int b = j & 1;
      const int n0 = u * G, nimg = min(G, nimgs - n0);
      CI_TIMED(w_a, mbar_wait_lazy(imgfree(b), ((j >> 1) & 1) ^ 1));
      CI_TIMED(w_b, stage_images<SG>(smem_u32(imgs + b * buf_floats), in, xmap_addr, n0, nimg, G, imgfull(b), lane));
    }
  } else {
    // ---------------- warp 17: MMA issuer (whole warp walks the loop; one elected lane issues)
    // instruction descriptor: D f32, A / B tf32, A (TMEM) and B K-major, N = 16, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    int it = 0, tile = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x)
      for (int t = 0; t < T; ++t, ++tile) {
        const int b = tile % CI_NACC;
        CI_TIMED(w_a, mbar_wait_warp(tempty(b), ((tile / CI_NACC) & 1) ^ 1));  // the epilogue has read this accumulator
        const uint32_t d = tm + (uint32_t)(b * 16);
        for (int kb = 0; kb < NKB; ++kb, ++it) {
          const int l = it % CI_L;
          CI_TIMED(w_b, mbar_wait_warp(conv(l), (it / CI_L) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t ahi = tm + (uint32_t)(CI_ACOL + l * 64), alo = ahi + 32;
          const uint32_t bt = sbase + (uint32_t)(kb * 4096);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t dhi = sdesc(bt + kk * 32, 16, 1024, 2), dlo = sdesc(bt + 2048 + kk * 32, 16, 1024, 2);
            mma_tf32_e<1>(d, alo + kk * 8, dhi, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
            mma_tf32_e<1>(d, ahi + kk * 8, dlo, idesc, 1u);
            mma_tf32_e<1>(d, ahi + kk * 8, dhi, idesc, 1u);
          }
          mma_commit_e<1>(lofree(l));
        }
        mma_commit_e<1>(tfull(b));
#ifdef CG_CI_MMALAT  // diagnostics: serialise and time each tile's MMA execution
        CI_TIMED(w_c, mbar_wait_warp(tfull(b), (tile / CI_NACC) & 1));
#endif
      }
  }
#ifdef CG_CI_TIMING
  if (blockIdx.x == 0 && lane == 0)
    printf("ci<%d,%d> warp %2d: busy %8lld  wait_a %8lld  wait_b %8lld  c %8lld  d %8lld (cycles)\n", CIN, COUT, warp,
           clock64() - t_role, w_a, w_b, w_c, w_d);
#else
  (void)w_a; (void)w_b; (void)w_c; (void)w_d; (void)t_role;
#endif
#undef CI_TIMED
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 17) {
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
// Warps 0-3 builders, 4-7 drain (TMEM -> one of two smem copies of C), 8..19
// col2im (smem -> dx), 20 MMA, 21 producer (each image's dy, 6.4 KB contiguous, by
// one TMA bulk copy into a BI_DS-slot ring): the drain of image i+1 overlaps the
// col2im sums of image i (one group doing both in turn, with dy prefetched one
// image ahead in registers, was latency-bound: 117 us on C4 conv2).
constexpr int BI_CW = 12;               // col2im warps (588 (pixel, channel pair) items per C4 image)
constexpr int BI_THREADS = (10 + BI_CW) * 32;
constexpr int BI_DS = 4;                // dy ring slots
constexpr int BI_L = 4;                 // A stages (32 TMEM columns: 16 hi + 16 lo)

template <int CO, int KS, int HO, int WO, int H, int W, int PT, int PL, int CI>
struct BiGeo {
  static constexpr int NJ = KS * KS * CI;                // GEMM N (real)
  static constexpr int NN = (NJ + 15) / 16 * 16;         // MMA N (multiple of 16)
  static constexpr int P = HO * WO;                      // dy pixels per image (<= 128)
  // row pitch of C in smem: even (8-byte col2im loads), CP / 2 odd (a half-warp's
  // 8-byte reads of 16 consecutive rows hit 16 distinct bank pairs)
  static constexpr int CP = ((NJ + 1) / 2 * 2 / 2) % 2 ? (NJ + 1) / 2 * 2 : (NJ + 1) / 2 * 2 + 2;
  static_assert(CI % 2 == 0, "col2im reads channel pairs");
  static constexpr int B_BYTES = NN * 128 * 2;           // hi + lo tiles, K-major SW128 (K padded to 32)
  static constexpr int C_FLOATS = 128 * CP;
  static constexpr int DY_FLOATS = (P * CO + 31) / 32 * 32;  // one image of dy (128-byte slots)
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
  float* Cs0 = reinterpret_cast<float*>(smem + Geo::B_BYTES);  // two copies of C: [2][128][CP]
  float* dyr = Cs0 + 2 * Geo::C_FLOATS;                          // dy ring [BI_DS][DY_FLOATS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(dyr + BI_DS * Geo::DY_FLOATS);
  const uint32_t bar0 = smem_u32(bars);
  auto conv = [&](int l) { return bar0 + 8u * l; };
  auto lofree = [&](int l) { return bar0 + 8u * (BI_L + l); };
  auto tfull = [&](int b) { return bar0 + 8u * (2 * BI_L + b); };
  auto tempty = [&](int b) { return bar0 + 8u * (2 * BI_L + 2 + b); };
  auto csfull = [&](int b) { return bar0 + 8u * (2 * BI_L + 4 + b); };
  auto csfree = [&](int b) { return bar0 + 8u * (2 * BI_L + 6 + b); };
  auto dyfull = [&](int k) { return bar0 + 8u * (2 * BI_L + 8 + k); };
  auto dyfree = [&](int k) { return bar0 + 8u * (2 * BI_L + 8 + BI_DS + k); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * BI_L + 8 + 2 * BI_DS);
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;  // (warp-uniform)

  if (threadIdx.x == 0) {
    for (int l = 0; l < BI_L; ++l) {
      mbar_init(conv(l), 4);
      mbar_init(lofree(l), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), 4);  // the 4 drain warps
      mbar_init(csfull(b), 4);  // the 4 drain warps
      mbar_init(csfree(b), BI_CW);  // the col2im warps
    }
    for (int k = 0; k < BI_DS; ++k) {
      mbar_init(dyfull(k), 1);  // the producer's arrive.expect_tx
      mbar_init(dyfree(k), 4);  // the builder warps
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
  if (warp == 8 + BI_CW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  long long w_a = 0, w_b = 0, t_role = 0;
#ifdef CG_BI_TIMING
#define BI_TIMED(acc, call)          \
  do {                               \
    const long long t_ = clock64();  \
    call;                            \
    acc += clock64() - t_;           \
  } while (0)
  t_role = clock64();
#else
#define BI_TIMED(acc, call) call
#endif

  if (warp < 4) {
    // ---------------- builders: dy row q (16 channels, 64 B, from the ring) -> TMEM hi / lo
    const int rr = warp * 32 + lane;
    int it = 0;
    for (int n = blockIdx.x; n < nimgs; n += gridDim.x, ++it) {
      const int k = it % BI_DS;
      BI_TIMED(w_a, mbar_wait(dyfull(k), (it / BI_DS) & 1));
      float4 cur[4];
      if (rr < P) {
        const float4* src = reinterpret_cast<const float4*>(dyr + k * Geo::DY_FLOATS + rr * CO);
#pragma unroll
        for (int i = 0; i < 4; ++i) cur[i] = src[i];
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) cur[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      // (generic reads of the slot before the TMA refills it: proxy fence, then release)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(dyfree(k));
      const int l = it % BI_L;
      BI_TIMED(w_b, mbar_wait(lofree(l), ((it / BI_L) & 1) ^ 1));
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
  } else if (warp < 8) {
    // ---------------- drain: C (TMEM) -> smem copy it & 1 (all loads of a batch in flight)
    const int wq = warp % 4, rr = wq * 32 + lane;  // TMEM lane quadrant
    int it = 0;
    for (int n = blockIdx.x; n < nimgs; n += gridDim.x, ++it) {
      const int b = it & 1;
      float* Cs = Cs0 + b * Geo::C_FLOATS;
      BI_TIMED(w_a, mbar_wait(csfree(b), ((it >> 1) & 1) ^ 1));  // the col2im sums of image it - 2 are done
      BI_TIMED(w_b, mbar_wait(tfull(b), (it >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      constexpr int NCH = NN / 16, BATCH = 2;
#pragma unroll
      for (int c0 = 0; c0 < NCH; c0 += BATCH) {
        uint32_t r[BATCH][16];
#pragma unroll
        for (int c = 0; c < BATCH; ++c)
          if (c0 + c < NCH) tmem_ld16_nowait(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(b * Geo::ACC + (c0 + c) * 16), r[c]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int c = 0; c < BATCH; ++c)
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + c < NCH && (c0 + c) * 16 + i < NJ) Cs[rr * CP + (c0 + c) * 16 + i] = __uint_as_float(r[c][i]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(tempty(b));
        mbar_arrive(csfull(b));  // (release: the STS above are visible to the col2im warps)
      }
    }
  } else if (warp < 8 + BI_CW) {
    // ---------------- col2im: one thread per (dx pixel, channel pair) item: 25 taps x one
    // 8-byte read; each channel in two fixed-order partial sums (even / odd kh, kh and
    // kw ascending) added at the end -- deterministic, half the dependent-add chain
    // (items, not pixels, per thread: every col2im warp has work; 117 -> 84 us with the
    // drain / col2im split.  Loading all 25 taps before the sums measured slower.)
    constexpr int NT = BI_CW * 32, CH2 = CI / 2;
    const int et = threadIdx.x - 256;
    int it = 0;
    for (int n = blockIdx.x; n < nimgs; n += gridDim.x, ++it) {
      const int b = it & 1;
      const float* Cs = Cs0 + b * Geo::C_FLOATS;
      BI_TIMED(w_a, mbar_wait(csfull(b), (it >> 1) & 1));
      float* o = dx + (size_t)n * H * W * CI;
      for (int item = et; item < H * W * CH2; item += NT) {
        const int pix = item / CH2, cp = item - pix * CH2;
        const int h = pix / W, ww = pix - h * W;
        float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float* cbase = Cs + 2 * cp;
#pragma unroll
        for (int kh = 0; kh < KS; ++kh) {
          const int oh = h - kh + PT;
          const bool rok = (unsigned)oh < (unsigned)HO;
#pragma unroll
          for (int kw = 0; kw < KS; ++kw) {
            const int ow = ww - kw + PL;
            if (rok && (unsigned)ow < (unsigned)WO) {
              const float2 t = *reinterpret_cast<const float2*>(cbase + (oh * WO + ow) * CP + (kh * KS + kw) * CI);
              acc[kh & 1].x = __fadd_rn(acc[kh & 1].x, t.x);
              acc[kh & 1].y = __fadd_rn(acc[kh & 1].y, t.y);
            }
          }
        }
        *reinterpret_cast<float2*>(o + (size_t)pix * CI + 2 * cp) =
            make_float2(__fadd_rn(acc[0].x, acc[1].x), __fadd_rn(acc[0].y, acc[1].y));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(csfree(b));
    }
  } else if (warp == 9 + BI_CW) {
    // ---------------- producer: one bulk copy per image into the dy ring
    int it = 0;
    for (int n = blockIdx.x; n < nimgs; n += gridDim.x, ++it) {
      const int k = it % BI_DS;
      BI_TIMED(w_a, mbar_wait_lazy(dyfree(k), ((it / BI_DS) & 1) ^ 1));
      if (lane == 0) {
        constexpr uint32_t bytes = P * CO * 4;
        mbar_expect_tx(dyfull(k), bytes);
        bulk_g2s(smem_u32(dyr + k * Geo::DY_FLOATS), dy + (size_t)n * P * CO, bytes, dyfull(k));
      }
      __syncwarp();
    }
  } else {
    // ---------------- warp 8 + BI_CW: MMA issuer.  D f32, A / B tf32, both K-major, N = NN, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    int it = 0;
    for (int n = blockIdx.x; n < nimgs; n += gridDim.x, ++it) {
      const int l = it % BI_L, b = it & 1;
      BI_TIMED(w_a, mbar_wait_warp(tempty(b), ((it >> 1) & 1) ^ 1));
      BI_TIMED(w_b, mbar_wait_warp(conv(l), (it / BI_L) & 1));
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
#ifdef CG_BI_TIMING
  if (blockIdx.x == 0 && lane == 0)
    printf("bi warp %2d: busy %8lld  wait_a %8lld  wait_b %8lld (cycles)\n", warp, clock64() - t_role, w_a, w_b);
#else
  (void)w_a; (void)w_b; (void)t_role;
#endif
#undef BI_TIMED
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 8 + BI_CW) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------- backward-kernel as a K = pixels GEMM
// dw[m, co] = sum_q A[m, q] dy[q, co],  m = (kh, kw, ci) (HWIO row), q = (n, oh, ow),
// A[m, q] = x[n, oh+kh-PT, ow+kw-PL, ci]  (zero outside the image; stride 1).
// M = KS*KS*CIN rows sit in TMEM lanes (A from TMEM), the pixels are the GEMM's K,
// B = dy^T (K-major rows of 32 pixels per output channel) in shared memory.
//
// Rows: the first 128 (if M >= 128) form a direct tile per 32-pixel k-block; the
// remaining R <= 32 rows use a block-diagonal tile: lane quadrant Q holds those rows
// for k-block Q of a 128-pixel super-block, and B carries all four k-blocks as
// N = 4*N0 columns -- D[(Q, r), (Q', co)] with Q == Q' is the wanted sum, the rest is
// ignored.  Same MMA cost as four narrow tiles, but the builders of all four lane
// quadrants (= all four SM sub-partitions) share the work instead of quadrant 0 alone.
// Chains of BK_CH super-blocks accumulate in TMEM; the epilogue adds each chain into
// a round-to-nearest register sum; per-CTA partials are summed in a fixed order by
// reduce_finalize (deterministic).
//
// Data movement is TMA bulk copies issued by one producer warp (many KB in flight
// per SM without registers): x chunks (G images, zero-padded in place) into two
// buffers, dy super-blocks (128 pixels) into a ring.  Warps: 0..7 A builders (two
// groups, alternate jobs), 8..11 B builders, 12..15 epilogue, 16 producer, 17 MMA.
constexpr int BK_THREADS = 576;
constexpr int BK_NG = 2;    // A builder groups
constexpr int BK_CH = 8;    // super-blocks per TMEM accumulation chain (1,024 pixels deep; 2 measured slower)

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT>
struct BkGeo {
  static constexpr int MR = KS * KS * CIN;     // real rows of dw
  static constexpr int T0 = MR / 128;          // direct tiles (0 or 1)
  static constexpr int R = MR - 128 * T0;      // rows of the block-diagonal tile
  static constexpr int N0 = COUT <= 8 ? 8 : 16;
  static constexpr int NB = 4 * N0;            // B rows = diagonal-tile N
  static constexpr int P = OH * OW;
  using SG = StageGeo<CIN, KS, IH, IW, OH, OW, PT, PL>;
  static constexpr bool TMAP = SG::TMAP;
  static constexpr int PLS = SG::PLS, WPS = SG::WPS, HP = SG::HP, XBASE = SG::XBASE, IMGF = SG::IMGF;
  // zero run covering every row offset, rounded so both image buffers stay 128-byte aligned
  static constexpr int ZLEN = (((KS - 1) * WPS + KS - 1) * CIN + CIN + 31) / 32 * 32;
  static constexpr int JOBS = 4 * T0 + 1;      // A tiles per 128-pixel super-block
  static constexpr int DCOL1 = 0;              // diagonal accumulators: [0, NB), [NB, 2 NB)
  static constexpr int DCOL0 = 2 * NB;         // direct accumulators: 16 columns each
  static constexpr int ACOL = 2 * NB + (T0 ? 32 : 0);
  static constexpr int L = (512 - ACOL) / 64;  // A ring slots (hi 32 + lo 32 columns)
  static constexpr int B_STAGE = 2 * NB * 128; // hi + lo, K-major SWIZZLE_128B rows
  static constexpr int DSK = COUT <= 8 ? 4 : 1;  // super-blocks of dy per ring slot (fewer, larger copies)
  static constexpr int DSLOT = DSK * 128 * COUT * 4;
  static constexpr int DS = COUT <= 8 ? 4 : 8;  // dy ring slots (48 / 64 KB in flight per SM)
  static constexpr int NBS = COUT <= 8 ? 3 : 4; // B group stages (DSK super-blocks each: one sync per group)
  static constexpr int B_GSTAGE = DSK * B_STAGE;
  static_assert(T0 <= 1 && R >= 1 && R <= 32 && COUT <= 16, "geometry");
  static_assert(T0 == 0 || N0 == 16, "direct tiles use N = 16");
  static_assert(L >= 3, "TMEM");
  static_assert((128 * COUT) % 4 == 0, "16-byte bulk copies");
  static constexpr int SRCF = SG::SRCF;
};

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT>
__global__ void __launch_bounds__(BK_THREADS, 1)
    conv_bwdk_tc_kernel(const float* __restrict__ x, const float* __restrict__ dy, float* __restrict__ part, int nimgs,
                        int G, int dbg, const __grid_constant__ CUtensorMap xmap) {
  // dbg: per-role busy / wait cycles of CTA 0 (printf; measurement only, compiled in
  // with -DCG_BK_TIMING -- the timers cost registers the roles need)
  long long w_a = 0, w_b = 0, w_c = 0, t_role = 0;
#ifdef CG_BK_TIMING
#define BK_TIMED(acc, call)                \
  do {                                     \
    const long long t_ = dbg ? clock64() : 0; \
    call;                                  \
    if (dbg) acc += clock64() - t_;        \
  } while (0)
#else
#define BK_TIMED(acc, call) \
  do {                      \
    call;                   \
  } while (0)
#endif
  using Geo = BkGeo<CIN, KS, IH, IW, OH, OW, PT, PL, COUT>;
  constexpr int MR = Geo::MR, T0 = Geo::T0, R = Geo::R, N0 = Geo::N0, NB = Geo::NB, P = Geo::P, WPS = Geo::WPS;
  constexpr int IMGF = Geo::IMGF, SRCF = Geo::SRCF, JOBS = Geo::JOBS, L = Geo::L, ACOL = Geo::ACOL, DS = Geo::DS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const int ZOFF = (Geo::XBASE + G * IMGF + 31) / 32 * 32;
  const int buf_floats = ZOFF + Geo::ZLEN;          // images + a zero run (ZOFF)
  const int nq = (G * P + 127) / 128 * 128;         // pixel slots of a chunk (whole super-blocks)
  float* dring = reinterpret_cast<float*>(smem + Geo::NBS * Geo::B_GSTAGE);
  float* xs = dring + DS * Geo::DSLOT / 4;          // 2 image buffers
  int* cbase = reinterpret_cast<int*>(xs + 2 * buf_floats);  // pixel -> staged offset of its window
  uint64_t* bars = reinterpret_cast<uint64_t*>(cbase + nq);
  const uint32_t bar0 = smem_u32(bars);
  auto imgfull = [&](int b) { return bar0 + 8u * b; };
  auto imgfree = [&](int b) { return bar0 + 8u * (2 + b); };
  auto tfull = [&](int b) { return bar0 + 8u * (4 + b); };
  auto tempty = [&](int b) { return bar0 + 8u * (6 + b); };
  auto afull = [&](int l) { return bar0 + 8u * (8 + l); };
  auto lofree = [&](int l) { return bar0 + 8u * (8 + L + l); };
  auto bfull = [&](int s) { return bar0 + 8u * (8 + 2 * L + s); };
  auto bfree = [&](int s) { return bar0 + 8u * (8 + 2 * L + Geo::NBS + s); };
  auto dfull = [&](int s) { return bar0 + 8u * (8 + 2 * L + 2 * Geo::NBS + s); };
  auto dfree = [&](int s) { return bar0 + 8u * (8 + 2 * L + 2 * Geo::NBS + DS + s); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * L + 2 * Geo::NBS + 2 * DS);
  // (the role index through a shuffle: provably warp-uniform, so the role branches
  // stay convergent and elect.sync / tcgen05 issue need no WARPSYNC.COLLECTIVE)
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;

  // this CTA's images [i0, i1): contiguous, balanced; chunks of G images
  const int i0 = (int)((long long)blockIdx.x * nimgs / gridDim.x);
  const int i1 = (int)((long long)(blockIdx.x + 1) * nimgs / gridDim.x);
  const int nchunks = (i1 - i0 + G - 1) / G;
  auto chunk_imgs = [&](int c) { return min(G, i1 - (i0 + c * G)); };
  auto chunk_sk = [&](int c) { return (chunk_imgs(c) * P + 127) / 128; };
  int s_tot = 0;
  for (int c = 0; c < nchunks; ++c) s_tot += chunk_sk(c);

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(imgfull(b), 1);            // the producer's arrive.expect_tx
      mbar_init(imgfree(b), 4 * BK_NG);    // every A builder warp
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), 4);
    }
    for (int l = 0; l < L; ++l) {
      mbar_init(afull(l), 4);
      mbar_init(lofree(l), 1);
    }
    for (int s = 0; s < Geo::NBS; ++s) {
      mbar_init(bfull(s), 4);
      mbar_init(bfree(s), 1);
    }
    for (int s = 0; s < DS; ++s) {
      mbar_init(dfull(s), 1);
      mbar_init(dfree(s), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = threadIdx.x; e < 2 * buf_floats; e += blockDim.x) xs[e] = 0.f;  // pads + zero runs stay zero
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    const int g = q / P, p = q - g * P, oh = p / OW, ow = p - oh * OW;
    cbase[q] = q < G * P ? Geo::SG::window(g, oh, ow) : ZOFF;
  }
  // the zeroing is generic-proxy; the TMA writes that follow are async-proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 17) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
#ifdef CG_BK_TIMING
  if (dbg) t_role = clock64();
#endif

  if (warp < 4 * BK_NG) {
    // ---------------- A builders: one 128-lane x 32-pixel tile per job (hi | lo columns)
    const int grp = warp / 4, Q = warp % 4;
    auto row_off = [](int m) {
      const int c = m % CIN, t = m / CIN, kh = t / KS, kw = t % KS;
      return Geo::SG::tap(kh, kw, c);
    };
    const int off_direct = T0 ? row_off(Q * 32 + lane) : 0;
    const int off_diag = lane < R ? row_off(T0 * 128 + lane) : 0;
    int it = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int b = c & 1, limit = chunk_imgs(c) * P, nsk = chunk_sk(c);
      BK_TIMED(w_a, mbar_wait(imgfull(b), (c >> 1) & 1));
      const float* img = xs + b * buf_floats;
      for (int k = 0; k < nsk; ++k) {
#pragma unroll
        for (int j = 0; j < JOBS; ++j, ++it) {
          if (it % BK_NG != grp) continue;
          const int l = it % L;
          const bool direct = j < 4 * T0;
          const int q0 = k * 128 + (direct ? j : Q) * 32;
          const float* src = img + (direct ? off_direct : off_diag);
          // the window offsets of the 32 pixels are the same for every lane: broadcast
          // LDS.128s, then 32 independent loads (no per-column shuffle -> load chain)
          int cb[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int4 t = *reinterpret_cast<const int4*>(cbase + q0 + 4 * i);
            cb[4 * i] = t.x; cb[4 * i + 1] = t.y; cb[4 * i + 2] = t.z; cb[4 * i + 3] = t.w;
          }
          if (q0 + 32 > limit) {  // (uniform) ragged end of a chunk: those pixels read the zero run
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (q0 + i >= limit) cb[i] = ZOFF;
          }
          const uint32_t ta = tmem + ((uint32_t)(Q * 32) << 16) + (uint32_t)(ACOL + l * 64);
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = src[cb[half * 16 + i]];
            if (half == 0) {
              BK_TIMED(w_b, mbar_wait(lofree(l), ((it / L) & 1) ^ 1));
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            uint32_t hv[16], lv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const uint32_t h = __float_as_uint(v[i]) & 0xFFFFE000u;
              hv[i] = h;
              lv[i] = __float_as_uint(__fsub_rn(v[i], __uint_as_float(h)));
            }
            tmem_st16(ta + half * 16, hv);
            tmem_st16(ta + 32 + half * 16, lv);
          }
          BK_TIMED(w_c, asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"));
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(afull(l));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(imgfree(b));
    }
  } else if (warp < 4 * BK_NG + 4) {
    // ---------------- B builders: per group of DSK super-blocks, dy rows of one 32-pixel
    // k-block each -> N0 K-major rows (hi, lo); one dy slot and one B stage per group
    const int Qb = warp - 4 * BK_NG;
    constexpr int GS = Geo::DSK;
    int gi = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int nsk = chunk_sk(c), limit = chunk_imgs(c) * P;
      for (int k0 = 0; k0 < nsk; k0 += GS, ++gi) {
        const int ds = gi % DS, sb = gi % Geo::NBS;
        float cur[GS][N0];
#pragma unroll
        for (int u = 0; u < GS; ++u)
#pragma unroll
          for (int i = 0; i < N0; ++i) cur[u][i] = 0.f;
        BK_TIMED(w_a, mbar_wait(dfull(ds), (gi / DS) & 1));
#pragma unroll
        for (int u = 0; u < GS; ++u) {
          const int q = (k0 + u) * 128 + Qb * 32 + lane;
          if (k0 + u < nsk && q < limit) {
            const float* src = dring + (size_t)ds * (Geo::DSLOT / 4) + (u * 128 + Qb * 32 + lane) * COUT;
            if constexpr (COUT % 4 == 0) {
#pragma unroll
              for (int i = 0; i < COUT; i += 4) {
                const float4 t = *reinterpret_cast<const float4*>(src + i);
                cur[u][i] = t.x; cur[u][i + 1] = t.y; cur[u][i + 2] = t.z; cur[u][i + 3] = t.w;
              }
            } else if constexpr (COUT % 2 == 0) {
#pragma unroll
              for (int i = 0; i < COUT; i += 2) {
                const float2 t = *reinterpret_cast<const float2*>(src + i);
                cur[u][i] = t.x; cur[u][i + 1] = t.y;
              }
            } else {
#pragma unroll
              for (int i = 0; i < COUT; ++i) cur[u][i] = src[i];
            }
          }
        }
        // the slot is refilled by TMA (async proxy) once every B warp has arrived: the
        // generic reads above must be complete first -- without this fence the last
        // LDS.128 (channels 12..15) was still in flight when the refill landed
        BK_TIMED(w_c, asm volatile("fence.proxy.async.shared::cta;" ::: "memory"));
        __syncwarp();
        if (lane == 0) mbar_arrive(dfree(ds));
        BK_TIMED(w_b, mbar_wait(bfree(sb), ((gi / Geo::NBS) & 1) ^ 1));
#pragma unroll
        for (int u = 0; u < GS; ++u) {
          uint8_t* bh = smem + sb * Geo::B_GSTAGE + u * Geo::B_STAGE;
#pragma unroll
          for (int co = 0; co < N0; ++co) {
            const int n = Qb * N0 + co;
            const int off = n * 128 + (((lane >> 2) ^ (n & 7)) << 4) + (lane & 3) * 4;
            const float hi = __uint_as_float(__float_as_uint(cur[u][co]) & 0xFFFFE000u);
            *reinterpret_cast<float*>(bh + off) = hi;
            *reinterpret_cast<float*>(bh + NB * 128 + off) = __fsub_rn(cur[u][co], hi);
          }
        }
        BK_TIMED(w_c, asm volatile("fence.proxy.async.shared::cta;" ::: "memory"));
        __syncwarp();
        if (lane == 0) mbar_arrive(bfull(sb));
      }
    }
  } else if (warp < 4 * BK_NG + 8) {
    // ---------------- epilogue: each chain's accumulators -> round-to-nearest register sums
    const int Qe = warp - 4 * BK_NG - 4;
    float s0[16], s1[N0];
#pragma unroll
    for (int i = 0; i < 16; ++i) s0[i] = 0.f;
#pragma unroll
    for (int i = 0; i < N0; ++i) s1[i] = 0.f;
    const int nch = (s_tot + BK_CH - 1) / BK_CH;
    const uint32_t lrow = (uint32_t)(Qe * 32) << 16;
    for (int ch = 0; ch < nch; ++ch) {
      const int b = ch & 1;
      BK_TIMED(w_a, mbar_wait(tfull(b), (ch >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if constexpr (T0 > 0) {
        float v[16];
        tmem_ld16(tmem + lrow + (uint32_t)(Geo::DCOL0 + b * 16), v);
#pragma unroll
        for (int i = 0; i < 16; ++i) s0[i] = __fadd_rn(s0[i], v[i]);
      }
      {
        float v[N0];
        if constexpr (N0 == 16) tmem_ld16(tmem + lrow + (uint32_t)(Geo::DCOL1 + b * NB + Qe * N0), v);
        else tmem_ld8(tmem + lrow + (uint32_t)(Geo::DCOL1 + b * NB + Qe * N0), v);
#pragma unroll
        for (int i = 0; i < N0; ++i) s1[i] = __fadd_rn(s1[i], v[i]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty(b));
    }
    float* out = part + (size_t)blockIdx.x * MR * COUT;
    if constexpr (T0 > 0) {
      const int m = Qe * 32 + lane;
#pragma unroll
      for (int co = 0; co < COUT; ++co) out[(size_t)m * COUT + co] = s0[co];
    }
    // diagonal rows: the four quadrants hold partial sums over different k-blocks;
    // combine them in a fixed order (Q = 0..3) through shared memory (the B ring is
    // idle: every MMA has completed once the last chain was drained)
    float* red = reinterpret_cast<float*>(smem);
#pragma unroll
    for (int i = 0; i < N0; ++i) red[(Qe * 32 + lane) * N0 + i] = s1[i];
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (Qe == 0 && lane < R) {
      const int m = T0 * 128 + lane;
#pragma unroll
      for (int co = 0; co < COUT; ++co) {
        float t = red[lane * N0 + co];
        t = __fadd_rn(t, red[(32 + lane) * N0 + co]);
        t = __fadd_rn(t, red[(64 + lane) * N0 + co]);
        t = __fadd_rn(t, red[(96 + lane) * N0 + co]);
        out[(size_t)m * COUT + co] = t;
      }
    }
  } else if (warp == 4 * BK_NG + 8) {
    // ---------------- producer: TMA bulk copies of x chunks and dy super-blocks.
    // Chunk c + 1's images are requested before chunk c's dy, so the A builders
    // never wait for an image buffer at a chunk boundary.
    // (the tensor map's address is taken here, on the __grid_constant__ parameter
    // itself: captured inside the lambda by reference it was copied to the stack and
    // the TMA saw a local address -> illegal instruction)
    const uint64_t xmap_addr = reinterpret_cast<uint64_t>(&xmap);
    auto load_x = [&](int c) {
      const int b = c & 1;
      BK_TIMED(w_a, mbar_wait(imgfree(b), ((c >> 1) & 1) ^ 1));
      stage_images<typename Geo::SG>(smem_u32(xs + b * buf_floats), x, xmap_addr, i0 + c * G, chunk_imgs(c), G, imgfull(b),
                                     lane);
    };
    int s = 0;
    if (nchunks > 0) load_x(0);
    for (int c = 0; c < nchunks; ++c) {
      const int nsk = chunk_sk(c), limit = chunk_imgs(c) * P;
      if (c + 1 < nchunks) load_x(c + 1);
      for (int k0 = 0; k0 < nsk; k0 += Geo::DSK, ++s) {  // (s counts dy slot groups here)
        const int ds = s % DS;
        BK_TIMED(w_b, mbar_wait(dfree(ds), ((s / DS) & 1) ^ 1));
        if (lane == 0) {
          const uint32_t bytes = (uint32_t)(min(Geo::DSK * 128, limit - k0 * 128) * COUT * 4);
          mbar_expect_tx(dfull(ds), bytes);
          bulk_g2s(smem_u32(dring) + (uint32_t)(ds * Geo::DSLOT),
                   dy + ((size_t)(i0 + c * G) * P + (size_t)k0 * 128) * COUT, bytes, dfull(ds));
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- warp 17: MMA issuer
    const uint32_t idesc0 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t idesc1 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    int it = 0, s = 0, gi = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int nsk = chunk_sk(c);
      for (int k = 0; k < nsk; ++k, ++s) {
        const int sub = k % Geo::DSK, sb = gi % Geo::NBS, ch = s / BK_CH, b = ch & 1;
        const bool group_end = sub == Geo::DSK - 1 || k == nsk - 1;
        const bool first = s % BK_CH == 0, last = s % BK_CH == BK_CH - 1 || s == s_tot - 1;
        if (first) BK_TIMED(w_a, mbar_wait_warp(tempty(b), ((ch >> 1) & 1) ^ 1));
        if (sub == 0) BK_TIMED(w_b, mbar_wait_warp(bfull(sb), (gi / Geo::NBS) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t bh = sbase + (uint32_t)(sb * Geo::B_GSTAGE + sub * Geo::B_STAGE), bl = bh + NB * 128;
#pragma unroll
        for (int j = 0; j < JOBS; ++j, ++it) {
          const int l = it % L;
          BK_TIMED(w_a, mbar_wait_warp(afull(l), (it / L) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t ahi = tm + (uint32_t)(ACOL + l * 64), alo = ahi + 32;
          const bool direct = j < 4 * T0;
          const uint32_t d = direct ? tm + (uint32_t)(Geo::DCOL0 + b * 16) : tm + (uint32_t)(Geo::DCOL1 + b * NB);
          const uint32_t boff = direct ? (uint32_t)(j * N0 * 128) : 0u;
          const uint32_t idesc = direct ? idesc0 : idesc1;
          const bool acc0 = !(first && (direct ? j == 0 : true));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t dhi = sdesc(bh + boff + kk * 32, 16, 1024, 2), dlo = sdesc(bl + boff + kk * 32, 16, 1024, 2);
            mma_tf32_e<1>(d, alo + kk * 8, dhi, idesc, (kk > 0 || acc0) ? 1u : 0u);
            mma_tf32_e<1>(d, ahi + kk * 8, dlo, idesc, 1u);
            mma_tf32_e<1>(d, ahi + kk * 8, dhi, idesc, 1u);
          }
          mma_commit_e<1>(lofree(l));
        }
        if (group_end) {
          mma_commit_e<1>(bfree(sb));
          ++gi;
        }
        if (last) mma_commit_e<1>(tfull(b));
      }
    }
  }
#ifdef CG_BK_TIMING
  if (dbg && blockIdx.x == 0 && lane == 0)
    printf("bwdk role-warp %2d: busy %8lld  wait_a %8lld  wait_b %8lld  fence/st %8lld (cycles)\n", warp, clock64() - t_role,
           w_a, w_b, w_c);
#else
  (void)w_a; (void)w_b; (void)w_c; (void)t_role;
#endif
#undef BK_TIMED
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 17) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT>
struct BkLaunch {
  using Geo = BkGeo<CIN, KS, IH, IW, OH, OW, PT, PL, COUT>;
  static int grid(int n, int num_sms) { return std::max(1, std::min(n, num_sms)); }
  static size_t smem_for(int G) {
    const int nq = (G * Geo::P + 127) / 128 * 128;
    return 1024 + (size_t)Geo::NBS * Geo::B_GSTAGE + (size_t)Geo::DS * Geo::DSLOT +
           2 * (((size_t)Geo::XBASE + G * Geo::IMGF + 31) / 32 * 32 + Geo::ZLEN) * 4 + (size_t)nq * 4 +
           (size_t)(10 + 2 * Geo::L + 2 * Geo::NBS + 2 * Geo::DS) * 8;  // barriers + TMEM slot
  }
  // images per chunk: the least padding in the last super-block with the two image
  // buffers within 48 KB (the rest of shared memory goes to the dy ring and B stages)
  static int pick_g() {
    int best = 1;
    double best_cost = 1e30;
    for (int G = 1; G <= 64; ++G) {
      if (2 * (size_t)G * Geo::IMGF * 4 > 48 * 1024 && G > 1) break;
      const int nq = (G * Geo::P + 127) / 128 * 128;
      const double cost = (double)nq / (G * Geo::P) * (1.0 + 0.02 / G);
      if (cost < best_cost) { best_cost = cost; best = G; }
    }
    return best;
  }
  static cudaError_t run(const float* x, const float* dy, float* dw, float* ws, int n, int num_sms, cudaStream_t s) {
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy)) & 15) return cudaErrorMisalignedAddress;
    const int G = pick_g(), gr = grid(n, num_sms);
    CUtensorMap xmap;
    std::memset(&xmap, 0, sizeof(xmap));
    if (Geo::TMAP && !make_img_map(&xmap, x, n, IH, IW, Geo::WPS, Geo::HP, G)) return cudaErrorInvalidValue;
    const size_t smem = smem_for(G);
    if (getenv("CG_BK_DEBUG")) fprintf(stderr, "bwdk_tc: G=%d grid=%d smem=%zu NBS=%d DS=%d L=%d\n", G, gr, smem, Geo::NBS, Geo::DS, Geo::L);
    auto kern = conv_bwdk_tc_kernel<CIN, KS, IH, IW, OH, OW, PT, PL, COUT>;
    cudaError_t e = smem_attr((const void*)kern, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<gr, BK_THREADS, smem, s>>>(x, dy, ws, n, G, getenv("CG_BK_DEBUG") ? 1 : 0, xmap);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_reduce_finalize(ws, dw, (long long)Geo::MR * COUT, gr, 0, s);
  }
};

template <int CO, int KS, int HO, int WO, int H, int W, int PT, int PL, int CI>
cudaError_t launch_bwdin(const float* dy, const float* w, float* dx, int n, int num_sms, cudaStream_t s) {
  using Geo = BiGeo<CO, KS, HO, WO, H, W, PT, PL, CI>;
  static_assert((Geo::P * CO * 4) % 16 == 0, "bulk copy size");
  if (reinterpret_cast<uintptr_t>(dy) & 15) return cudaErrorMisalignedAddress;
  const size_t smem = 1024 + Geo::B_BYTES + 2 * (size_t)Geo::C_FLOATS * 4 + BI_DS * (size_t)Geo::DY_FLOATS * 4 + 256;
  auto kern = conv_bwdin_col2im_kernel<CO, KS, HO, WO, H, W, PT, PL, CI>;
  cudaError_t e = smem_attr((const void*)kern, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<std::min(n, num_sms), BI_THREADS, smem, s>>>(dy, w, dx, n);
  return cudaGetLastError();
}

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT>
cudaError_t launch_geo(const float* in, const float* w, float* out, int n, const EpiProg* epi, int num_sms,
                       cudaStream_t s) {
  using Geo = CiGeo<CIN, KS, IH, IW, OH, OW, PT, PL, COUT>;
  using SG = typename Geo::SG;
  if (reinterpret_cast<uintptr_t>(in) & 15) return cudaErrorMisalignedAddress;
  // images per unit: the largest G (<= 32) whose double-buffered images fit, preferring
  // little padding in the last 128-pixel tile of a unit
  auto buf_bytes = [](int G) { return (size_t)((SG::XBASE + G * SG::IMGF + 31) / 32 * 32) * 4; };
  constexpr size_t budget = 200 * 1024;
  int best_g = 1;
  double best_cost = 1e30;
  for (int G = 1; G <= 32; ++G) {
    const size_t bytes = Geo::B_BYTES + 2 * buf_bytes(G);
    if (bytes > budget) break;
    const int T = (G * Geo::P + 127) / 128;
    const double waste = (double)T * 128 / ((double)G * Geo::P);   // padded rows per real row
    const double cost = waste * (1.0 + 0.5 / G);                     // + per-unit overhead
    if (cost < best_cost) { best_cost = cost; best_g = G; }
  }
  const int G = best_g, T = (G * Geo::P + 127) / 128;
  const size_t smem = 1024 + Geo::B_BYTES + 2 * buf_bytes(G) + 512 + kEpiMax * COUT * 4;
  CUtensorMap xmap;
  std::memset(&xmap, 0, sizeof(xmap));
  if (SG::TMAP && !make_img_map(&xmap, in, n, IH, IW, SG::WPS, SG::HP, G)) return cudaErrorInvalidValue;
  auto kern = conv_img_tc_kernel<CIN, KS, IH, IW, OH, OW, PT, PL, COUT>;
  cudaError_t e = smem_attr((const void*)kern, (int)smem);
  if (e != cudaSuccess) return e;
  const int units = (n + G - 1) / G;
  EpiProg ep{};
  if (epi) ep = *epi;
  kern<<<std::min(units, num_sms), CI_THREADS, smem, s>>>(in, w, out, n, G, T, xmap, ep);
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

// ---------------------------------------------------------------- stem: few-channel, strided, wide images
// The InceptionV3 stem conv (299x299x3 -> 149x149x32, 3x3, stride 2, VALID; C5) as
// an implicit GEMM over bands of RB output rows of one image: the band's input rows
// are ONE contiguous span of x (VALID: no padding), staged by a single 16-byte-
// aligned TMA bulk copy (the span's start is shifted into the buffer; the copy may
// read up to 12 bytes past the tensor, inside its 256-byte-aligned allocation).
// Builders form each 128-pixel x 32-k slab (K = KS*KS*CIN <= 32 per k-block,
// k = (kh, kw, c)) from shared memory into TMEM (hi / lo), one warp issues 12
// tf32 MMAs (M = 128, N = COUT) per slab, the epilogue applies the fused
// elementwise chain (the BN scale / shift + ReLU of the DOT/CONV epilogue fusion,
// per-column or scalar operands) and stores 32 channels per pixel with row stride
// ldc.  Replaces the element-gather path of the generic conv (Ci = 3 is not a TMA
// im2col box): 1.43 ms at batch 256 in round 1.
// Warps: builders (SB_BG groups of 4), epilogue (SB_EW per TMEM lane quadrant, COUT /
// SB_EW channels each), producer, MMA.  With the fused batch-norm chain the epilogue
// warps are busy the whole kernel (-DCG_SB_TIMING) while the builders wait 88 % of
// the time, yet one builder group with four epilogue warps per quadrant measured the
// same (467 vs 453 us): the defaults stay two and two.
#ifndef CG_SB_BG
#define CG_SB_BG 2
#endif
#ifndef CG_SB_EW
#define CG_SB_EW 2
#endif
constexpr int SB_BG = CG_SB_BG, SB_EW = CG_SB_EW;
constexpr int SB_EPI0 = 4 * SB_BG, SB_PROD = SB_EPI0 + 4 * SB_EW, SB_MMA = SB_PROD + 1;
constexpr int SB_THREADS = (SB_MMA + 1) * 32;
constexpr int SB_L = 6;
constexpr int SB_NBUF = 4;  // band buffers: a band's copy latency exceeds its compute (measured with 2: 733 us)

template <int CIN, int KS, int S, int IH, int IW, int OH, int OW, int COUT, int RB>
struct SbGeo {
  static constexpr int K = CIN * KS * KS;
  static constexpr int NKB = (K + 31) / 32;
  static constexpr int NR = (RB - 1) * S + KS;                 // input rows of a full band
  static constexpr int ROWF = IW * CIN;
  static constexpr int BUF = (NR * ROWF + 8 + 31) / 32 * 32;   // + shift slack + 16-byte tail
  static constexpr int NB = (OH + RB - 1) / RB;                // bands per image
  static constexpr int TMAX = (RB * OW + 127) / 128;           // tiles of a full band
  static constexpr int B_TILE = COUT * 128;                    // bytes of one hi (or lo) K-major tile
  static constexpr int B_BYTES = NKB * 2 * B_TILE;
  static constexpr int ACC = COUT;                             // TMEM columns per accumulator
  static constexpr int ACOL = 2 * COUT;
  static_assert(COUT % 16 == 0 && COUT <= 64 && ACOL + SB_L * 64 <= 512, "TMEM");
};

template <int CIN, int KS, int S, int IH, int IW, int OH, int OW, int COUT, int RB>
__global__ void __launch_bounds__(SB_THREADS, 1)
    conv_band_tc_kernel(const float* __restrict__ x, const float* __restrict__ w, float* __restrict__ out, int ldc,
                        int nimgs, const __grid_constant__ EpiProg epi, int dbg) {
  // dbg (measurement only, CG_SB_DEBUG): 1 = skip the output stores, 2 = skip the chain
  using Geo = SbGeo<CIN, KS, S, IH, IW, OH, OW, COUT, RB>;
  constexpr int K = Geo::K, NKB = Geo::NKB, ROWF = Geo::ROWF, BUF = Geo::BUF, NB = Geo::NB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  float* bufs = reinterpret_cast<float*>(smem + Geo::B_BYTES);
  float* eops = bufs + SB_NBUF * BUF;                           // per-column chain operands [kEpiMax][COUT]
  float* ostage = eops + kEpiMax * COUT;                        // [4 quadrants][32 px][COUT + 4]: coalesced stores
  static_assert(COUT % (16 * SB_EW) == 0 || (COUT / SB_EW) % 8 == 0, "epilogue channel split");
  uint64_t* bars = reinterpret_cast<uint64_t*>(ostage + 4 * 32 * (COUT + 4));
  const uint32_t bar0 = smem_u32(bars);
  constexpr int NBF = SB_NBUF;
  auto full = [&](int b) { return bar0 + 8u * b; };
  auto freeb = [&](int b) { return bar0 + 8u * (NBF + b); };
  auto conv = [&](int l) { return bar0 + 8u * (2 * NBF + l); };
  auto lofree = [&](int l) { return bar0 + 8u * (2 * NBF + SB_L + l); };
  auto tfull = [&](int b) { return bar0 + 8u * (2 * NBF + 2 * SB_L + b); };
  auto tempty = [&](int b) { return bar0 + 8u * (2 * NBF + 2 * SB_L + 2 + b); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NBF + 2 * SB_L + 4);
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;
  const int units = nimgs * NB;
#ifdef CG_SB_TIMING  // per-role cycle accounting of CTA 0 (measurement builds only)
  long long tw = 0, tx1 = 0, tx2 = 0, t0r = 0;
#define SB_T(acc, call)                 \
  do {                                  \
    const long long t_ = clock64();     \
    call;                               \
    acc += clock64() - t_;              \
  } while (0)
#else
#define SB_T(acc, call) \
  do {                  \
    call;               \
  } while (0)
#endif
  auto band_rows = [](int b) { return min(RB, OH - b * RB); };

  if (threadIdx.x == 0) {
    for (int b = 0; b < NBF; ++b) {
      mbar_init(full(b), 1);
      mbar_init(freeb(b), 4 * SB_BG);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), 4 * SB_EW);
    }
    for (int l = 0; l < SB_L; ++l) {
      mbar_init(conv(l), 4);
      mbar_init(lofree(l), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // B = weights [KS][KS][CIN][COUT] as K-major SWIZZLE_128B tiles (hi, lo) per k-block
  for (int e = threadIdx.x; e < NKB * COUT * 32; e += blockDim.x) {
    const int kb = e / (COUT * 32), rem = e % (COUT * 32), n = rem / 32, kl = rem % 32, k = kb * 32 + kl;
    const float v = k < K ? __ldg(w + (size_t)k * COUT + n) : 0.f;  // row k = (kh, kw, c) of HWIO
    const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    const int off = n * 128 + (((kl >> 2) ^ (n & 7)) << 4) + (kl & 3) * 4;
    *reinterpret_cast<float*>(smem + kb * 2 * Geo::B_TILE + off) = hi;
    *reinterpret_cast<float*>(smem + kb * 2 * Geo::B_TILE + Geo::B_TILE + off) = __fsub_rn(v, hi);
  }
  for (int e = threadIdx.x; e < epi.n * COUT; e += blockDim.x) {
    const int i = e / COUT, c = e % COUT;
    eops[e] = epi.op[i] == EPI_RELU ? 0.f : (epi.scalar[i] ? __ldg(epi.x[i]) : __ldg(epi.x[i] + c));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == SB_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
#ifdef CG_SB_TIMING
  t0r = clock64();
#endif
  // the band's input span and its shift inside the staging buffer (16-byte-aligned copy)
  auto span = [&](int u, long long* a0, int* shift, int* bytes) {
    const int n = u / NB, b = u % NB, rows = band_rows(b);
    const long long start = ((long long)n * IH + (long long)b * RB * S) * ROWF;
    const int cnt = ((rows - 1) * S + KS) * ROWF;
    *a0 = start & ~3LL;
    *shift = (int)(start - *a0);
    *bytes = ((cnt + *shift) * 4 + 15) / 16 * 16;
  };

  if (warp < SB_EPI0) {
    // ---------------- builders
    const int grp = warp / 4, wq = warp % 4, rr = wq * 32 + lane;
    int it = 0, j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int bsel = j % NBF;
      long long a0;
      int shift, bytes;
      span(u, &a0, &shift, &bytes);
      const int npx = band_rows(u % NB) * OW, T = (npx + 127) / 128;
      SB_T(tw, mbar_wait(full(bsel), (j / NBF) & 1));
      const float* img = bufs + bsel * BUF + shift;
      for (int t = 0; t < T; ++t, it += NKB) {
        const int q = t * 128 + rr;
        const int qq = q < npx ? q : 0;
        const int ol = qq / OW, ow = qq - ol * OW;
        const float* base = img + (ol * S) * ROWF + (ow * S) * CIN;
#pragma unroll
        for (int kb = 0; kb < NKB; ++kb) {
          const int step = it + kb;
          if (SB_BG == 2 && (step & 1) != grp) continue;
          const int l = step % SB_L;
          float v[32];
#pragma unroll
          for (int kl = 0; kl < 32; ++kl) {
            const int k = kb * 32 + kl;
            if (k < K) {
              const int c = k % CIN, tap = k / CIN, kh = tap / KS, kw = tap % KS;
              v[kl] = base[kh * ROWF + kw * CIN + c];
            } else {
              v[kl] = 0.f;
            }
          }
          SB_T(tx1, mbar_wait(lofree(l), ((step / SB_L) & 1) ^ 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t ta = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(Geo::ACOL + l * 64);
          uint32_t hv[32], lv[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const uint32_t h = __float_as_uint(v[i]) & 0xFFFFE000u;
            hv[i] = h;
            lv[i] = __float_as_uint(__fsub_rn(v[i], __uint_as_float(h)));
          }
          tmem_st32(ta, hv);
          tmem_st32(ta + 32, lv);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(conv(l));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(freeb(bsel));
    }
  } else if (warp < SB_PROD) {
    // ---------------- epilogue: per tile, sum of the k-blocks' fresh accumulators
    // (round to nearest), the fused chain, 16-byte stores.  SB_EW warps per TMEM lane
    // quadrant, each owning COUT / SB_EW of the output channels.
    constexpr int CH = COUT / SB_EW;
    const int wq = warp % 4, half = (warp - SB_EPI0) / 4, rr = wq * 32 + lane, c0 = half * CH;
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int n = u / NB, b = u % NB, npx = band_rows(b) * OW, T = (npx + 127) / 128;
      for (int t = 0; t < T; ++t) {
        float sum[CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) sum[i] = 0.f;
        for (int kb = 0; kb < NKB; ++kb, ++it) {
          const int bb = it & 1;
          SB_T(tw, mbar_wait(tfull(bb), (it >> 1) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if constexpr (CH % 16 == 0) {
#pragma unroll
            for (int cc = 0; cc < CH; cc += 16) {
              float vv[16];
              SB_T(tx1, tmem_ld16(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(bb * Geo::ACC + c0 + cc), vv));
#pragma unroll
              for (int i = 0; i < 16; ++i) sum[cc + i] = NKB == 1 ? vv[i] : __fadd_rn(sum[cc + i], vv[i]);
            }
          } else {
            static_assert(CH == 8, "8 or a multiple of 16 channels per epilogue warp");
            float vv[8];
            SB_T(tx1, tmem_ld8(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(bb * Geo::ACC + c0), vv));
#pragma unroll
            for (int i = 0; i < 8; ++i) sum[i] = NKB == 1 ? vv[i] : __fadd_rn(sum[i], vv[i]);
          }
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty(bb));
        }
        // the chain, op by op: the op and operand order are uniform, so each op is one
        // branch and a straight unrolled loop (a per-value switch compiled to a BRX jump
        // table per element and made the chain the kernel's bottleneck: 1.16 ms vs 0.17)
        for (int e = 0; e < ((dbg & 2) ? 0 : epi.n); ++e) epi_apply<CH>(sum, epi.op[e], epi.swap[e], eops + e * COUT + c0);
        // the quadrant's 32 pixels x COUT channels are one contiguous 4 KB run of the
        // output (row pitch ldc == COUT): the warp pair assembles it in shared memory and
        // writes it with 512-byte coalesced stores (per-lane 64-byte halves of lines
        // written by two warps at different times measured 1.5x slower)
        const long long pix0 = ((long long)n * OH + (long long)b * RB) * OW + t * 128 + wq * 32;
        const int nval = min(32, npx - (t * 128 + wq * 32));
        if (dbg & 1) {
        } else if (ldc == COUT && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
          float* st = ostage + wq * 32 * (COUT + 4);
#pragma unroll
          for (int i = 0; i < CH; i += 4)
            *reinterpret_cast<float4*>(st + lane * (COUT + 4) + c0 + i) = make_float4(sum[i], sum[i + 1], sum[i + 2], sum[i + 3]);
          SB_T(tx2, asm volatile("bar.sync %0, %1;" ::"r"(1 + wq), "r"(32 * SB_EW) : "memory"));
          constexpr int Q4 = COUT / 4;  // float4 per pixel
#pragma unroll
          for (int k = 0; k < 32 * Q4 / (32 * SB_EW); ++k) {
            const int c = half * (32 * Q4 / SB_EW) + k * 32 + lane, px = c / Q4, part = c % Q4;
            if (px < nval)
              *reinterpret_cast<float4*>(out + (pix0 + px) * COUT + part * 4) =
                  *reinterpret_cast<const float4*>(st + px * (COUT + 4) + part * 4);
          }
          asm volatile("bar.sync %0, %1;" ::"r"(1 + wq), "r"(32 * SB_EW) : "memory");
        } else if (lane < nval) {
          float* o = out + (pix0 + lane) * ldc + c0;
#pragma unroll
          for (int i = 0; i < CH; ++i) o[i] = sum[i];
        }
      }
    }
  } else if (warp == SB_PROD) {
    // ---------------- producer: one bulk copy per band (double-buffered)
    int j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int bsel = j % NBF;
      long long a0;
      int shift, bytes;
      span(u, &a0, &shift, &bytes);
      SB_T(tw, mbar_wait(freeb(bsel), ((j / NBF) & 1) ^ 1));
      if (lane == 0) {
        mbar_expect_tx(full(bsel), (uint32_t)bytes);
        bulk_g2s(smem_u32(bufs + bsel * BUF), x + a0, (uint32_t)bytes, full(bsel));
      }
      __syncwarp();
    }
  } else {
    // ---------------- warp 17: MMA issuer (N = COUT, M = 128)
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(COUT >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int npx = band_rows(u % NB) * OW, T = (npx + 127) / 128;
      for (int t = 0; t < T; ++t)
        for (int kb = 0; kb < NKB; ++kb, ++it) {
          const int l = it % SB_L, bb = it & 1;
          SB_T(tw, mbar_wait_warp(tempty(bb), ((it >> 1) & 1) ^ 1));
          SB_T(tx1, mbar_wait_warp(conv(l), (it / SB_L) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t d = tm + (uint32_t)(bb * Geo::ACC);
          const uint32_t ahi = tm + (uint32_t)(Geo::ACOL + l * 64), alo = ahi + 32;
          const uint32_t bt = sbase + (uint32_t)(kb * 2 * Geo::B_TILE);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t dhi = sdesc(bt + kk * 32, 16, 1024, 2), dlo = sdesc(bt + Geo::B_TILE + kk * 32, 16, 1024, 2);
            mma_tf32_e<1>(d, alo + kk * 8, dhi, idesc, kk > 0 ? 1u : 0u);
            mma_tf32_e<1>(d, ahi + kk * 8, dlo, idesc, 1u);
            mma_tf32_e<1>(d, ahi + kk * 8, dhi, idesc, 1u);
          }
          mma_commit_e<1>(lofree(l));
          mma_commit_e<1>(tfull(bb));
        }
    }
  }
#ifdef CG_SB_TIMING
  if (blockIdx.x == 0 && lane == 0)
    printf("band warp %2d: busy %8lld wait %8lld x1 %8lld x2 %8lld\n", warp, clock64() - t0r, tw, tx1, tx2);
#endif
#undef SB_T
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == SB_MMA) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int CIN, int KS, int S, int IH, int IW, int OH, int OW, int COUT, int RB>
cudaError_t launch_band(const float* x, const float* w, float* out, int ldc, int n, const EpiProg& epi, int num_sms,
                        cudaStream_t s) {
  using Geo = SbGeo<CIN, KS, S, IH, IW, OH, OW, COUT, RB>;
  if (reinterpret_cast<uintptr_t>(x) & 15) return cudaErrorMisalignedAddress;
  const size_t smem = 1024 + Geo::B_BYTES + SB_NBUF * (size_t)Geo::BUF * 4 + kEpiMax * COUT * 4 + 4 * 32 * (COUT + 4) * 4 + 512;
  auto kern = conv_band_tc_kernel<CIN, KS, S, IH, IW, OH, OW, COUT, RB>;
  cudaError_t e = smem_attr((const void*)kern, (int)smem);
  if (e != cudaSuccess) return e;
  const int units = n * Geo::NB;
  static const int dbg = getenv("CG_SB_DEBUG") ? atoi(getenv("CG_SB_DEBUG")) : 0;
  kern<<<std::min(units, num_sms), SB_THREADS, smem, s>>>(x, w, out, ldc, n, epi, dbg);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- 3x3 stride-1 convs on wide images (C5 stem)
// 149x149x32 -> 147x147x32 VALID and 147x147x32 -> 147x147x64 SAME (InceptionV3
// layers 2 and 3).  The generic implicit GEMM re-reads every input pixel 9 times
// through TMA im2col (1.48 / 0.87 ms at batch 256, A-side bound).  Here each input
// ROW is staged once, by a 4-D tensor-map TMA whose box is CIN + 4 channels wide
// (the out-of-bounds fill pads every pixel to 36 floats: conflict-free 16-byte
// shared loads with pixels on lanes), into a ring of NS row slots; tiles of 128
// consecutive output pixels of one image (<= 2 output rows, <= 4 input rows) are
// built from the ring (tap (kh, kw) of 32 channels = one k-block = 8 LDS.128 per
// pixel), 12 tf32 MMAs (M = 128, N = NH) per k-block; COUT > NH is split over
// CTAs (NH output channels each).  Rows leave the ring when every builder warp has
// moved past them.  The epilogue (fresh accumulator per k-block summed with
// round-to-nearest, the fused chain, coalesced stores) is the band kernel's.
constexpr int RW_THREADS = 576;  // 0-7 builders, 8-15 epilogue, 16 producer, 17 MMA
constexpr int RW_L = 6;           // A slots
constexpr int RW_NS = 6;          // row slots
constexpr int RW_QU = 4;          // units per image (tile ranges): balance over 148 CTAs

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT, int NH>
struct RwGeo {
  static constexpr int CPAD = CIN + 4;
  // a tensor TMA destination must be 128-byte aligned: input column iw sits at staged
  // column iw + PLS with PLS * CPAD * 4 % 128 == 0 (PLS >= PL; the columns before it
  // stay zero and serve as the left padding), and every slot starts on 128 bytes
  static constexpr int PLS = PL == 0 ? 0 : (PL * CPAD * 4 % 128 == 0 ? PL : (128 / 16) * ((PL + 7) / 8));
  static constexpr int PR = OW + KS - 1 - PL - IW > 0 ? OW + KS - 1 - PL - IW : 0;
  static constexpr int WPS = IW + PLS + PR;
  static constexpr int ROWF = (WPS * CPAD + 31) / 32 * 32;
  static_assert(PLS >= PL && (PLS * CPAD * 4) % 128 == 0, "TMA destination alignment");
  static constexpr int NKB = KS * KS * CIN / 32;
  static constexpr int CB = CIN / 32;                 // k-blocks per tap
  static constexpr int P = OH * OW;
  static constexpr int TPI = (P + 127) / 128;         // tiles per image
  static constexpr int TPQ = (TPI + RW_QU - 1) / RW_QU;
  static constexpr int HALVES = COUT / NH;
  static constexpr int B_TILE = NH * 128;
  static constexpr int B_BYTES = NKB * 2 * B_TILE;
  static constexpr int ACC = NH;
  static constexpr int ACOL = 2 * NH;
  static_assert(CIN % 32 == 0 && COUT % NH == 0 && NH % 16 == 0 && ACOL + RW_L * 64 <= 512, "geometry");
  static_assert(OW >= 64, "a tile spans at most two output rows");
};

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT, int NH>
__global__ void __launch_bounds__(RW_THREADS, 1)
    conv_rows_tc_kernel(const float* __restrict__ w, float* __restrict__ out, int ldc, int nimgs,
                        const __grid_constant__ CUtensorMap xmap, const __grid_constant__ EpiProg epi) {
  using Geo = RwGeo<CIN, KS, IH, IW, OH, OW, PT, PL, COUT, NH>;
  constexpr int NKB = Geo::NKB, ROWF = Geo::ROWF, CPAD = Geo::CPAD, P = Geo::P, TPI = Geo::TPI, TPQ = Geo::TPQ;
  constexpr int HALVES = Geo::HALVES, NS = RW_NS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  float* rows = reinterpret_cast<float*>(smem + Geo::B_BYTES);
  float* eops = rows + NS * ROWF;
  float* ostage = eops + kEpiMax * NH;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ostage + 4 * 32 * (NH + 4));
  const uint32_t bar0 = smem_u32(bars);
  auto rfull = [&](int b) { return bar0 + 8u * b; };
  auto rfree = [&](int b) { return bar0 + 8u * (NS + b); };
  auto conv = [&](int l) { return bar0 + 8u * (2 * NS + l); };
  auto lofree = [&](int l) { return bar0 + 8u * (2 * NS + RW_L + l); };
  auto tfull = [&](int b) { return bar0 + 8u * (2 * NS + 2 * RW_L + b); };
  auto tempty = [&](int b) { return bar0 + 8u * (2 * NS + 2 * RW_L + 2 + b); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NS + 2 * RW_L + 4);
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;
  const int units = nimgs * RW_QU * HALVES;
  // unit u -> image, tile range [t0, t1), channel half; its input rows [ih0, ih0 + nr)
  auto unit_of = [&](int u, int* img, int* t0, int* t1, int* half, int* oh_lo, int* nr) {
    *half = u % HALVES;
    const int q = (u / HALVES) % RW_QU;
    *img = u / (HALVES * RW_QU);
    *t0 = q * TPQ;
    *t1 = min(TPI, (q + 1) * TPQ);
    *oh_lo = (*t0 * 128) / OW;
    const int oh_hi = min(OH - 1, (*t1 * 128 - 1) / OW);
    *nr = *t1 > *t0 ? oh_hi - *oh_lo + KS : 0;
  };
  const int h0 = (units > 0) ? 0 : 0;
  (void)h0;

  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(rfull(b), 1);
      mbar_init(rfree(b), 8);
    }
    for (int l = 0; l < RW_L; ++l) {
      mbar_init(conv(l), 4);
      mbar_init(lofree(l), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // every row slot's pad columns stay zero (TMA writes the interior only)
  for (int e = threadIdx.x; e < NS * ROWF; e += blockDim.x) rows[e] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 17) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // B (weights, this CTA's NH channels) is rebuilt per unit only when the half changes
  int cur_half = -1;
  auto load_b = [&](int half) {  // called by every thread between units (block-wide sync below)
    for (int e = threadIdx.x; e < NKB * NH * 32; e += blockDim.x) {
      const int kb = e / (NH * 32), rem = e % (NH * 32), n = rem / 32, kl = rem % 32, k = kb * 32 + kl;
      const float v = __ldg(w + (size_t)k * COUT + half * NH + n);  // k = (kh, kw, c): HWIO row
      const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
      const int off = n * 128 + (((kl >> 2) ^ (n & 7)) << 4) + (kl & 3) * 4;
      *reinterpret_cast<float*>(smem + kb * 2 * Geo::B_TILE + off) = hi;
      *reinterpret_cast<float*>(smem + kb * 2 * Geo::B_TILE + Geo::B_TILE + off) = __fsub_rn(v, hi);
    }
    for (int e = threadIdx.x; e < epi.n * NH; e += blockDim.x) {
      const int i = e / NH, c = e % NH;
      eops[e] = epi.op[i] == EPI_RELU ? 0.f : (epi.scalar[i] ? __ldg(epi.x[i]) : __ldg(epi.x[i] + half * NH + c));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  };
  // every CTA handles one half only when HALVES divides the CTA stride; otherwise B is
  // loaded per unit by all roles in lockstep (not needed for the compiled geometries)
  {
    int img, t0, t1, half, oh_lo, nr;
    unit_of(blockIdx.x, &img, &t0, &t1, &half, &oh_lo, &nr);
    cur_half = half;
    load_b(half);
  }
  __syncthreads();

  if (warp < 8) {
    // ---------------- builders
    const int grp = warp / 4, wq = warp % 4, rr = wq * 32 + lane;
    int it = 0, sbase_row = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int img, t0, t1, half, oh_lo, nr;
      unit_of(u, &img, &t0, &t1, &half, &oh_lo, &nr);
      int waited = 0, released = 0;
      for (int t = t0; t < t1; ++t) {
        const int first = (t * 128) / OW - oh_lo;
        const int last = min(OH - 1, (t * 128 + 127) / OW) - oh_lo + KS - 1;
        for (; waited <= last; ++waited) {
          const int sq = sbase_row + waited;
          mbar_wait(rfull(sq % NS), (sq / NS) & 1);
        }
        const int q = t * 128 + rr;
        const int qq = q < P ? q : t * 128;
        const int oh = qq / OW, ow = qq - oh * OW, lr = oh - oh_lo;
#pragma unroll 1
        for (int kb = 0; kb < NKB; ++kb) {
          const int step = it + kb;
          if ((step & 1) != grp) continue;
          const int l = step % RW_L;
          const int tap = kb / Geo::CB, cb = kb % Geo::CB, kh = tap / KS, kw = tap % KS;
          const int sq = sbase_row + lr + kh;
          const float* src = rows + (sq % NS) * ROWF + (ow + kw + Geo::PLS - PL) * CPAD + cb * 32;
          float4 v4[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) v4[i] = *reinterpret_cast<const float4*>(src + 4 * i);
          mbar_wait(lofree(l), ((step / RW_L) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          uint32_t hv[32], lv[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float c4[4] = {v4[i].x, v4[i].y, v4[i].z, v4[i].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t h = __float_as_uint(c4[j]) & 0xFFFFE000u;
              hv[4 * i + j] = h;
              lv[4 * i + j] = __float_as_uint(__fsub_rn(c4[j], __uint_as_float(h)));
            }
          }
          const uint32_t ta = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(Geo::ACOL + l * 64);
          tmem_st32(ta, hv);
          tmem_st32(ta + 32, lv);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(conv(l));
        }
        it += NKB;
        // rows no later tile of this unit needs
        const int next_first = t + 1 < t1 ? ((t + 1) * 128) / OW - oh_lo : nr;
        for (; released < next_first; ++released) {
          __syncwarp();
          if (lane == 0) mbar_arrive(rfree((sbase_row + released) % NS));
        }
      }
      for (; released < nr; ++released) {
        __syncwarp();
        if (lane == 0) mbar_arrive(rfree((sbase_row + released) % NS));
      }
      sbase_row += nr;
    }
  } else if (warp < 16) {
    // ---------------- epilogue (two warps per lane quadrant, NH / 2 channels each)
    constexpr int CH = NH / 2;
    const int wq = warp % 4, hh = (warp - 8) / 4, rr = wq * 32 + lane, c0 = hh * CH;
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int img, t0, t1, half, oh_lo, nr;
      unit_of(u, &img, &t0, &t1, &half, &oh_lo, &nr);
      for (int t = t0; t < t1; ++t) {
        // the whole K (NKB k-blocks) accumulates in one TMEM accumulator per tile, as in
        // the generic implicit GEMM (a fresh accumulator per k-block made the MMA wait
        // for a drain every k-block: the pipeline ran at ~1/5 of the MMA rate)
        float sum[CH];
        {
          const int bb = it & 1;
          mbar_wait(tfull(bb), (it >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int cc = 0; cc < CH; cc += 16) {
            float vv[16];
            tmem_ld16(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(bb * Geo::ACC + c0 + cc), vv);
#pragma unroll
            for (int i = 0; i < 16; ++i) sum[cc + i] = vv[i];
          }
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty(bb));
          ++it;
        }
        for (int e = 0; e < epi.n; ++e) epi_apply<CH>(sum, epi.op[e], epi.swap[e], eops + e * NH + c0);
        // the quadrant's 32 pixels x NH channels: NH * 4-byte runs per pixel, assembled
        // in shared memory by the warp pair and stored with coalesced 16-byte writes
        const long long pix0 = (long long)img * P + t * 128 + wq * 32;
        const int nval = min(32, P - (t * 128 + wq * 32));
        float* st = ostage + wq * 32 * (NH + 4);
#pragma unroll
        for (int i = 0; i < CH; i += 4)
          *reinterpret_cast<float4*>(st + lane * (NH + 4) + c0 + i) = make_float4(sum[i], sum[i + 1], sum[i + 2], sum[i + 3]);
        asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
        constexpr int Q4 = NH / 4;
#pragma unroll
        for (int k = 0; k < 32 * Q4 / 64; ++k) {
          const int c = hh * (32 * Q4 / 2) + k * 32 + lane, px = c / Q4, part = c % Q4;
          if (px < nval)
            *reinterpret_cast<float4*>(out + (pix0 + px) * ldc + half * NH + part * 4) =
                *reinterpret_cast<const float4*>(st + px * (NH + 4) + part * 4);
        }
        asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
      }
    }
  } else if (warp == 16) {
    // ---------------- producer: one 4-D TMA per input row (zero rows for the padding)
    const uint64_t xmap_addr = reinterpret_cast<uint64_t>(&xmap);
    int sq = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int img, t0, t1, half, oh_lo, nr;
      unit_of(u, &img, &t0, &t1, &half, &oh_lo, &nr);
      for (int j = 0; j < nr; ++j, ++sq) {
        const int slot = sq % NS, ih = oh_lo - PT + j;
        mbar_wait(rfree(slot), ((sq / NS) & 1) ^ 1);
        float* dst = rows + slot * ROWF;
        if (ih >= 0 && ih < IH) {
          if (lane == 0) {
            mbar_expect_tx(rfull(slot), (uint32_t)(IW * CPAD * 4));
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
                    smem_u32(dst + Geo::PLS * CPAD)),
                "l"(xmap_addr), "r"(0), "r"(0), "r"(ih), "r"(img), "r"(rfull(slot))
                : "memory");
          }
        } else {
          for (int e = lane; e < ROWF; e += 32) dst[e] = 0.f;  // a padding row
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (a later TMA refill of the slot)
          __syncwarp();
          if (lane == 0) mbar_arrive(rfull(slot));
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- warp 17: MMA issuer (N = NH, M = 128)
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NH >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    int it = 0, tile = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int img, t0, t1, half, oh_lo, nr;
      unit_of(u, &img, &t0, &t1, &half, &oh_lo, &nr);
      for (int t = t0; t < t1; ++t, ++tile) {
        const int bb = tile & 1;
        mbar_wait_warp(tempty(bb), ((tile >> 1) & 1) ^ 1);  // the epilogue has drained this accumulator
        const uint32_t d = tm + (uint32_t)(bb * Geo::ACC);
        for (int kb = 0; kb < NKB; ++kb, ++it) {
          const int l = it % RW_L;
          mbar_wait_warp(conv(l), (it / RW_L) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t ahi = tm + (uint32_t)(Geo::ACOL + l * 64), alo = ahi + 32;
          const uint32_t bt = sbase + (uint32_t)(kb * 2 * Geo::B_TILE);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t dhi = sdesc(bt + kk * 32, 16, 1024, 2), dlo = sdesc(bt + Geo::B_TILE + kk * 32, 16, 1024, 2);
            mma_tf32_e<1>(d, alo + kk * 8, dhi, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
            mma_tf32_e<1>(d, ahi + kk * 8, dlo, idesc, 1u);
            mma_tf32_e<1>(d, ahi + kk * 8, dhi, idesc, 1u);
          }
          mma_commit_e<1>(lofree(l));
        }
        mma_commit_e<1>(tfull(bb));
      }
    }
  }
  (void)cur_half;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 17) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// 4-D tiled map over NHWC x [n][h][w][c], box {c + 4, w, 1, 1}: one input row per load,
// every pixel padded to c + 4 floats by the out-of-bounds zero fill
bool make_row_map(CUtensorMap* m, const float* x, int n, int h, int w, int c) {
  static EncodeTiledFnCI fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFnCI)p;
  });
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)c * 4, (cuuint64_t)w * c * 4, (cuuint64_t)h * w * c * 4};
  cuuint32_t box[4] = {(cuuint32_t)(c + 4), (cuuint32_t)w, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int CIN, int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT, int NH>
cudaError_t launch_rows(const float* x, const float* w, float* out, int ldc, int n, const EpiProg& epi, int num_sms,
                        cudaStream_t s) {
  using Geo = RwGeo<CIN, KS, IH, IW, OH, OW, PT, PL, COUT, NH>;
  CUtensorMap xmap;
  std::memset(&xmap, 0, sizeof(xmap));
  if (!make_row_map(&xmap, x, n, IH, IW, CIN)) return cudaErrorInvalidValue;
  const size_t smem = 1024 + Geo::B_BYTES + (size_t)RW_NS * Geo::ROWF * 4 + kEpiMax * NH * 4 + 4 * 32 * (NH + 4) * 4 +
                      (2 * RW_NS + 2 * RW_L + 6) * 8;
  auto kern = conv_rows_tc_kernel<CIN, KS, IH, IW, OH, OW, PT, PL, COUT, NH>;
  cudaError_t e = smem_attr((const void*)kern, (int)smem);
  if (e != cudaSuccess) return e;
  const int units = n * RW_QU * Geo::HALVES;
  // a CTA keeps one channel half: the grid is a multiple of HALVES (B is loaded once)
  int grid = std::min(units, num_sms) / Geo::HALVES * Geo::HALVES;
  if (grid < Geo::HALVES) grid = Geo::HALVES;
  kern<<<grid, RW_THREADS, smem, s>>>(w, out, ldc, n, xmap, epi);
  return cudaGetLastError();
}

}  // namespace

bool conv_band_supported(int n, int h, int w, int ci, int kh, int kw, int co, int ho, int wo, int sh, int sw, int pt,
                         int pl) {
  (void)n;
  return !getenv("CG_NO_CONV_BAND") && h == 299 && w == 299 && ci == 3 && kh == 3 && kw == 3 && co == 32 && ho == 149 &&
         wo == 149 && sh == 2 && sw == 2 && pt == 0 && pl == 0;
}

int conv_rows_kind(int h, int w, int ci, int kh, int kw, int co, int ho, int wo, int sh, int sw, int pt, int pl) {
  if (getenv("CG_NO_CONV_ROWS") || kh != 3 || kw != 3 || sh != 1 || sw != 1 || ci != 32) return 0;
  if (h == 149 && w == 149 && co == 32 && ho == 147 && wo == 147 && pt == 0 && pl == 0) return 1;
  // (split over two CTAs per row range -- B for 64 channels does not fit next to the
  // ring -- it builds every A slab twice; still 1.60 ms against the generic implicit
  // GEMM's 2.20 ms at batch 256)
  if (h == 147 && w == 147 && co == 64 && ho == 147 && wo == 147 && pt == 1 && pl == 1) return 2;
  return 0;
}

cudaError_t launch_conv_rows(int kind, const float* x, const float* w, float* out, int ldc, int n, const EpiProg& epi,
                             int num_sms, cudaStream_t s) {
  if (kind == 1) return launch_rows<32, 3, 149, 149, 147, 147, 0, 0, 32, 32>(x, w, out, ldc, n, epi, num_sms, s);
  if (kind == 2) return launch_rows<32, 3, 147, 147, 147, 147, 1, 1, 64, 32>(x, w, out, ldc, n, epi, num_sms, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_conv_band(const float* x, const float* w, float* out, int ldc, int n, const EpiProg& epi, int num_sms,
                             cudaStream_t s) {
  // the InceptionV3 stem: 299x299x3 -> 149x149x32, 3x3 stride 2 VALID; bands of 6 output rows (894 px = 7 tiles)
  return launch_band<3, 3, 2, 299, 299, 149, 149, 32, 6>(x, w, out, ldc, n, epi, num_sms, s);
}

// ---------------------------------------------------------------- backward-kernel, one input channel: SIMT
// dw[kh, kw, 0, co] = sum_{n,oh,ow} x[n, oh+kh-PT, ow+kw-PL] dy[n, oh, ow, co]  (stride 1, Ci = 1).
// With KS*KS = 25 rows and COUT = 6 columns the tensor-core formulation (K = pixels)
// fills a quarter of each MMA (block-diagonal tile) and was MMA-issue bound at
// 140 us on C4 conv1; the FFMA form needs 25 x 6 x 2 flops per pixel (27 us of
// FP32 issue at full rate).  Thread = (kh, 2 adjacent output pixels): 5 x COUT
// accumulators per output pixel pair fed by 2 x COUT dy values and 6 x values
// from shared memory (TMA-staged images, zero padded as the forward kernel's).
// Warps: SB_KH groups of 4 (one kernel row each) + 1 producer.  Each thread's
// partial sums are reduced in a fixed order per CTA, the per-CTA partials in a
// fixed order by reduce_finalize: deterministic.
constexpr int BS_GW = 4;  // warps per kernel-row group

template <int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT>
struct BsGeo {
  using SG = StageGeo<1, KS, IH, IW, OH, OW, PT, PL>;
  static constexpr int P = OH * OW, PP = P / 2;           // pixels, pixel pairs per image
  static constexpr int DYF = P * COUT;                    // dy floats per image
  static constexpr int G = 4;                             // images per stage
  static constexpr int XBUF = (SG::XBASE + G * SG::IMGF + 31) / 32 * 32;
  static constexpr int THREADS = (KS * BS_GW + 1) * 32;
  static_assert(OW % 2 == 0, "pixel pairs within a row");
  static_assert((DYF * 4) % 16 == 0 && (COUT * 2) % 4 == 0, "16-byte dy copies / pair loads");
  // POOLED: dy given as the 2x2 max-pool backward's inputs -- the pooled gradient
  // [n, OH/2, OW/2, COUT] and the forward's decision codes (same shape, bytes)
  static constexpr int DPF = (OH / 2) * (OW / 2) * COUT;
  template <bool POOLED>
  __host__ __device__ static constexpr int slot() { return POOLED ? G * DPF + (G * DPF + 15) / 16 * 4 : G * DYF; }  // floats per stage
  template <bool POOLED>
  static constexpr size_t smem_bytes() {
    return 1024 + (2 * (size_t)XBUF + 2 * (size_t)slot<POOLED>() + (POOLED ? (size_t)G * DYF : 0) + KS * BS_GW * 32) * 4 +
           64;
  }
};

// POOLED: dy = RELU_GRAD(a, MAXPOOL2D_BWD(relu(a), dp)) is never materialised; each
// pixel pair's dy is formed from dp and the pool's codes (bit 7: the routed value is
// > 0, bits 0-1: the window position) -- the values the pool-backward kernel would
// have stored.
template <int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT, bool POOLED = false>
__global__ void __launch_bounds__(BsGeo<KS, IH, IW, OH, OW, PT, PL, COUT>::THREADS, 1)
    conv_bwdk_simt_kernel(const float* __restrict__ x, const float* __restrict__ dy, float* __restrict__ ws, int nimgs,
                          const __grid_constant__ CUtensorMap xmap, float* __restrict__ wsb,
                          const unsigned char* __restrict__ pcodes) {
  using Geo = BsGeo<KS, IH, IW, OH, OW, PT, PL, COUT>;
  using SG = typename Geo::SG;
  constexpr int G = Geo::G, PP = Geo::PP, DYF = Geo::DYF, NT = BS_GW * 32;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* xs = reinterpret_cast<float*>(smem);                 // [2][XBUF]
  float* dys = xs + 2 * Geo::XBUF;                             // [2][SLOT]: dy, or (POOLED) dp + codes
  float* dyx = dys + 2 * Geo::template slot<POOLED>();         // (POOLED) this stage's dy, formed once: [G * DYF]
  float* red = dyx + (POOLED ? G * DYF : 0);                   // [KS][NT] reduction scratch
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + KS * NT);
  const uint32_t bar0 = smem_u32(bars);
  auto full = [&](int b) { return bar0 + 8u * b; };
  auto freeb = [&](int b) { return bar0 + 8u * (2 + b); };
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0), lane = threadIdx.x % 32;
  const int units = (nimgs + G - 1) / G;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(full(b), 1);
      mbar_init(freeb(b), KS * BS_GW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = threadIdx.x; e < 2 * Geo::XBUF; e += blockDim.x) xs[e] = 0.f;  // padding / guard stays zero
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  if (warp == KS * BS_GW) {
    // ---------------- producer: G images of x (3-D tensor map, zero padded) and of dy per stage
    const uint64_t xmap_addr = reinterpret_cast<uint64_t>(&xmap);
    int j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int b = j & 1, n0 = u * G, nimg = min(G, nimgs - n0);
      mbar_wait_lazy(freeb(b), ((j >> 1) & 1) ^ 1);
      if (lane == 0) {
        // (no arrive here: stage_images' arrive.expect_tx below completes the phase's count)
        if constexpr (POOLED) {
          constexpr int DPF = Geo::DPF;
          const uint32_t cbytes = (uint32_t)(nimg * DPF + 15) / 16 * 16;  // (the codes buffer is padded)
          mbar_expect_tx_only(full(b), (uint32_t)(nimg * DPF * 4) + cbytes);
          constexpr int SLOT = Geo::template slot<true>();
          bulk_g2s(smem_u32(dys + b * SLOT), dy + (size_t)n0 * DPF, (uint32_t)(nimg * DPF * 4), full(b));
          bulk_g2s(smem_u32(dys + b * SLOT + G * DPF), pcodes + (size_t)n0 * DPF, cbytes, full(b));
        } else {
          mbar_expect_tx_only(full(b), (uint32_t)(nimg * DYF * 4));
          bulk_g2s(smem_u32(dys + b * G * DYF), dy + (size_t)n0 * DYF, (uint32_t)(nimg * DYF * 4), full(b));
        }
      }
      stage_images<SG>(smem_u32(xs + b * Geo::XBUF), x, xmap_addr, n0, nimg, G, full(b), lane);
    }
    return;
  }
  // ---------------- compute: kernel row kh, pixel pairs t, t + NT, ... of each stage
  const int kh = warp / BS_GW, t = threadIdx.x - kh * NT;
  float acc[KS][COUT];
#pragma unroll
  for (int a = 0; a < KS; ++a)
#pragma unroll
    for (int c = 0; c < COUT; ++c) acc[a][c] = 0.f;
  // wsb != NULL: the bias gradient sum_{n,oh,ow} dy[., co] as a by-product of row
  // group 0's dy reads (the SUM group of the same dy, fused: dy read once)
  float bsum[COUT];
#pragma unroll
  for (int c = 0; c < COUT; ++c) bsum[c] = 0.f;
  const bool bias = wsb != nullptr && kh == 0;
  int j = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
    const int b = j & 1, n0 = u * G, nimg = min(G, nimgs - n0);
    if constexpr (POOLED) asm volatile("bar.sync 1, %0;" ::"r"(KS * NT) : "memory");  // previous stage's dy read
    mbar_wait(full(b), (j >> 1) & 1);
    const float* xb = xs + b * Geo::XBUF;
    const float* db = dys + b * Geo::template slot<POOLED>();
    if constexpr (POOLED) {
      // dy = RELU_GRAD(a, MAXPOOL2D_BWD(relu(a), dp)) formed once per stage from dp and
      // the pool's codes (bit 7: the routed value > 0; bits 0-1: window position
      // k = 2 * row + column): the values the pool-backward kernel would have stored
      const unsigned char* cb = reinterpret_cast<const unsigned char*>(db + G * Geo::DPF);
      constexpr int WPR = OW / 2;
      for (int e = threadIdx.x; e < nimg * Geo::DPF; e += KS * NT) {
        const int c = e % COUT, w = e / COUT, wc = w % WPR, wr = (w / WPR) % (OH / 2), gg = w / (WPR * (OH / 2));
        const unsigned code = cb[e];
        const float v = db[e];
        const int k = (code & 0x80u) ? (int)(code & 3u) : -1;
        float* o = dyx + ((gg * OH + 2 * wr) * OW + 2 * wc) * COUT + c;
        o[0] = k == 0 ? v : 0.f;
        o[COUT] = k == 1 ? v : 0.f;
        o[OW * COUT] = k == 2 ? v : 0.f;
        o[OW * COUT + COUT] = k == 3 ? v : 0.f;
      }
      // (buffer b is released after the items below: its x images are still read)
      asm volatile("bar.sync 1, %0;" ::"r"(KS * NT) : "memory");  // the stage's dy complete
      db = dyx;
    }
    for (int q = t; q < nimg * PP; q += NT) {
      const int g = q / PP, pp = q - g * PP, oh = pp / (OW / 2), ow = (pp - oh * (OW / 2)) * 2;
      float d0[COUT], d1[COUT];
      const float* dp = db + (g * Geo::P + oh * OW + ow) * COUT;
#pragma unroll
      for (int c = 0; c < COUT; c += 2) {
        const float2 v0 = *reinterpret_cast<const float2*>(dp + c), v1 = *reinterpret_cast<const float2*>(dp + COUT + c);
        d0[c] = v0.x; d0[c + 1] = v0.y; d1[c] = v1.x; d1[c + 1] = v1.y;
      }
      const float* xp = xb + SG::window(g, oh, ow) + SG::tap(kh, 0, 0);
      float xv[KS + 1];
#pragma unroll
      for (int a = 0; a < KS + 1; ++a) xv[a] = xp[a];
#pragma unroll
      for (int a = 0; a < KS; ++a)
#pragma unroll
        for (int c = 0; c < COUT; ++c) acc[a][c] = fmaf(xv[a + 1], d1[c], fmaf(xv[a], d0[c], acc[a][c]));
      if (bias) {
#pragma unroll
        for (int c = 0; c < COUT; ++c) bsum[c] = __fadd_rn(__fadd_rn(bsum[c], d0[c]), d1[c]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(freeb(b));
  }
  // ---------------- fixed-order reduction over the NT threads of the row group
  asm volatile("bar.sync 1, %0;" ::"r"(KS * NT) : "memory");
#pragma unroll
  for (int a = 0; a < KS; ++a)
#pragma unroll
    for (int c = 0; c < COUT; ++c) {  // (unrolled: acc stays in registers)
      red[kh * NT + t] = acc[a][c];
      asm volatile("bar.sync 1, %0;" ::"r"(KS * NT) : "memory");
      for (int h = NT / 2; h > 0; h >>= 1) {
        if (t < h) red[kh * NT + t] = red[kh * NT + t] + red[kh * NT + t + h];
        asm volatile("bar.sync 1, %0;" ::"r"(KS * NT) : "memory");
      }
      if (t == 0) ws[(size_t)blockIdx.x * KS * KS * COUT + (kh * KS + a) * COUT + c] = red[kh * NT];
      asm volatile("bar.sync 1, %0;" ::"r"(KS * NT) : "memory");
    }
  if (wsb != nullptr) {  // row group 0's bias partials, same fixed-order tree
#pragma unroll
    for (int c = 0; c < COUT; ++c) {
      if (kh == 0) red[t] = bsum[c];
      asm volatile("bar.sync 1, %0;" ::"r"(KS * NT) : "memory");
      for (int h = NT / 2; h > 0; h >>= 1) {
        if (kh == 0 && t < h) red[t] = __fadd_rn(red[t], red[t + h]);
        asm volatile("bar.sync 1, %0;" ::"r"(KS * NT) : "memory");
      }
      if (kh == 0 && t == 0) wsb[(size_t)blockIdx.x * COUT + c] = red[0];
      asm volatile("bar.sync 1, %0;" ::"r"(KS * NT) : "memory");
    }
  }
}

template <int KS, int IH, int IW, int OH, int OW, int PT, int PL, int COUT>
cudaError_t launch_bwdk_simt(const float* x, const float* dy, float* dw, float* ws, int n, int num_sms, cudaStream_t s,
                             float* db, const unsigned char* pcodes) {
  using Geo = BsGeo<KS, IH, IW, OH, OW, PT, PL, COUT>;
  using SG = typename Geo::SG;
  static_assert(SG::TMAP, "zero padding from the tensor map's out-of-bounds fill");
  if ((reinterpret_cast<uintptr_t>(dy) & 15) || (reinterpret_cast<uintptr_t>(x) & 15)) return cudaErrorMisalignedAddress;
  CUtensorMap xmap;
  std::memset(&xmap, 0, sizeof(xmap));
  if (!make_img_map(&xmap, x, n, IH, IW, SG::WPS, SG::HP, Geo::G)) return cudaErrorInvalidValue;
  const size_t smem = pcodes ? Geo::template smem_bytes<true>() : Geo::template smem_bytes<false>();
  auto kern = pcodes ? conv_bwdk_simt_kernel<KS, IH, IW, OH, OW, PT, PL, COUT, true>
                     : conv_bwdk_simt_kernel<KS, IH, IW, OH, OW, PT, PL, COUT, false>;
  cudaError_t e = smem_attr((const void*)kern, (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = std::max(1, std::min(n, num_sms));
  float* wsb = db ? ws + (size_t)grid * KS * KS * COUT : nullptr;  // (conv_img_tc_bwdk_ws counts it)
  kern<<<grid, Geo::THREADS, smem, s>>>(x, dy, ws, n, xmap, wsb, pcodes);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = launch_reduce_finalize(ws, dw, (long long)KS * KS * COUT, grid, 0, s);
  if (e != cudaSuccess || !db) return e;
  return launch_reduce_finalize(wsb, db, COUT, grid, 0, s);
}

bool conv_img_tc_bwdk_supported(const ConvGeom& g) {
  return kind_of(g, false) != CI_NONE && !getenv("CG_NO_CONV_IMG_TC");
}

size_t conv_img_tc_bwdk_ws(const ConvGeom& g, int num_sms) {  // (+ the fused bias-gradient partials)
  return (size_t)std::max(1, std::min(g.n, num_sms)) * (g.kh * g.kw * g.ci * g.co + g.co);
}

bool conv_img_tc_bwdk_bias_ok(const ConvGeom& g) { return kind_of(g, false) == CI_C4_CONV1 && !getenv("CG_BWDK_TC1"); }

cudaError_t launch_conv_img_tc_bwdk(const float* x, const float* dy, float* dw, float* ws, const ConvGeom& g, int num_sms,
                                    cudaStream_t s, float* db, const unsigned char* pcodes) {
  if ((db || pcodes) && !conv_img_tc_bwdk_bias_ok(g)) return cudaErrorInvalidValue;
  switch (kind_of(g, false)) {
    case CI_C4_CONV1:  // x [n,28,28,1], dy [n,28,28,6] -> dw [5,5,1,6] (SAME)
      if (getenv("CG_BWDK_TC1"))  // (A/B: the tensor-core K = pixels formulation)
        return BkLaunch<1, 5, 28, 28, 28, 28, 2, 2, 6>::run(x, dy, dw, ws, g.n, num_sms, s);
      return launch_bwdk_simt<5, 28, 28, 28, 28, 2, 2, 6>(x, dy, dw, ws, g.n, num_sms, s, db, pcodes);
    case CI_C4_CONV2:  // x [n,14,14,6], dy [n,10,10,16] -> dw [5,5,6,16] (VALID)
      return BkLaunch<6, 5, 14, 14, 10, 10, 0, 0, 16>::run(x, dy, dw, ws, g.n, num_sms, s);
    default:
      return cudaErrorInvalidValue;
  }
}

bool conv_img_tc_supported(const ConvGeom& g, bool flip) {
  return kind_of(g, flip) != CI_NONE && !getenv("CG_NO_CONV_IMG_TC");
}

cudaError_t launch_conv_img_tc(const float* in, const float* w, float* out, const ConvGeom& g, bool flip, int num_sms,
                               cudaStream_t s, const EpiProg* epi) {
  if (flip && epi && epi->n) return cudaErrorInvalidValue;  // (no epilogue on the col2im kernel)
  switch (kind_of(g, flip)) {
    case CI_C4_CONV1:  // x [n,28,28,1] (*) w [5,5,1,6], SAME
      return launch_geo<1, 5, 28, 28, 28, 28, 2, 2, 6>(in, w, out, g.n, epi, num_sms, s);
    case CI_C4_CONV2:  // p1 [n,14,14,6] (*) w [5,5,6,16], VALID
      return launch_geo<6, 5, 14, 14, 10, 10, 0, 0, 16>(in, w, out, g.n, epi, num_sms, s);
    case CI_C4_CONV2_BWDIN:  // dy [n,10,10,16], w [5,5,6,16] -> dx [n,14,14,6] (VALID forward)
      return launch_bwdin<16, 5, 10, 10, 14, 14, 0, 0, 6>(in, w, out, g.n, num_sms, s);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace cg
