// DOT nodes on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   C[M,N] = op(A)[M,K] . op(B)[K,N]      fp32 in, fp32 out  (SURVEY §8(c) c1-defs DOT)
//
// tcgen05 has no fp32-input MMA, so every fp32 operand x is split into
// hi = x & 0xFFFFE000 (exactly representable in TF32) and lo = x - hi (exact in
// fp32), and the product is accumulated as  hi.hi + hi.lo + lo.hi  ("3xTF32",
// The kind::tf32 datapath itself truncates an fp32 operand to exactly hi (measured:
// tools/tf32_probe.py, tests test_tf32_truncation_probe), so the raw tile serves
// as the hi operand and only lo is written back to shared memory.
// SURVEY §8(c) c12) in fp32 TMEM accumulators.  The dropped lo.lo term is
// < 2^-20 relative, so the result has fp32-GEMM accuracy.
// Integer-valued operands with |x| < 2^11 have lo == 0 and are multiplied exactly.
//
// Operand paths.  The 3 MMAs per k-step read shared memory through the same
// 128 B/clk/SM port as the TMA writes and the split's loads/stores; with both
// operands in shared memory that port, not the tensor core, bounded the kernel
// (~190 KB per 32-deep k-slab of a 128 x 128 tile against 768 MMA cycles).  So
// A goes to TENSOR MEMORY: the split warps read each A row once from the
// staged tile and write its hi and lo parts with tcgen05.st (TMEM write
// 256 B/clk); the MMAs take A from TMEM (tcgen05.mma ... [d], [a_tmem], b_desc)
// and only B is read from shared memory.  TMEM budget per CTA (512 columns):
// two BN-column accumulators + LSTAGES x (32 hi + 32 lo) A columns, so BN <= 128.
// Operand majorness: A may be K-major (ta = 0, SWIZZLE_128B rows) or M-major
// (ta = 1, SWIZZLE_128B_ATOM_32B boxes) in shared memory -- the split reads
// either and writes TMEM rows (TMEM A is always K-major); B is N-major when tb = 0
// and K-major when tb = 1, both native UMMA smem layouts (idesc bit 16).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "dot_tc.h"
#include "conv_img_tc.h"
#include "kernels.h"

#include <algorithm>

namespace cg {

namespace {

constexpr int BM = 128, BK = 32;
// Tile configurations (N = 32 / 64 / 128 columns per unit).  Three rings, each
// advancing once per 32-deep k-block:
//   A ring  (SA stages)  TMA / gather destination of the raw A tile; freed by the
//                        split warps as soon as they hold their row in registers
//   B ring  (SB stages)  raw B tile (also the hi operand the MMAs read); freed by
//                        the MMA commit
//   lo ring (LSTAGES)    smem B lo tile + TMEM A hi/lo columns; split -> MMA
// Separating A from B keeps the A stage lifetime at "load latency + split"
// instead of "... + the MMAs of every earlier stage", so the same shared memory
// buys a deeper B prefetch.
template <int BNT, int CG = 1, bool GATHER = false>
struct TC {
  static constexpr int BN = BNT;
  static constexpr int TILE_A = BM * BK * 4;           // 16 KiB
  static constexpr int TILE_B = BNT / CG * BK * 4;     // this CTA's share of the B tile
  static constexpr int LO_BYTES = TILE_B;              // B lo in shared memory (A hi/lo live in TMEM)
  static constexpr int LSTAGES = 4;                    // lo ring (smem B lo + TMEM A hi/lo)
  static constexpr int ACOL = 2 * BNT;                 // first TMEM column of the A stages
  static_assert(ACOL + LSTAGES * 2 * BK <= 512, "TMEM: accumulators + A stages");
  static constexpr int EPI_BYTES = kEpiMax * BNT * 4;
  // im2col-gathered A tiles are cp.async loads with a long L2 latency: a deeper A ring
  static constexpr int SA_WANT = GATHER ? 8 : 4;
  static constexpr int SA_FIT = (220 * 1024 - EPI_BYTES - LSTAGES * LO_BYTES - 3 * TILE_B) / TILE_A;
  static constexpr int SA = SA_FIT < SA_WANT ? SA_FIT : SA_WANT;
  static constexpr int SB_FIT = (220 * 1024 - EPI_BYTES - SA * TILE_A - LSTAGES * LO_BYTES) / TILE_B;
  static constexpr int SB = SB_FIT > 8 ? 8 : SB_FIT;
  static constexpr int A_BASE = 0;
  static constexpr int B_BASE = SA * TILE_A;
  static constexpr int LO_BASE = B_BASE + SB * TILE_B;
  static constexpr int EPI_BASE = LO_BASE + LSTAGES * LO_BYTES;   // fused-epilogue operands [kEpiMax][BN]
  static constexpr int BAR_BASE = EPI_BASE + EPI_BYTES;
  static constexpr int SMEM_BYTES = BAR_BASE + 1024 /*barriers*/ + 1024 /*alignment slack*/;
  static_assert(SA >= 4 && SB >= 3, "pipeline depth");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};
// warps: 0 TMA, 1 MMA, 2-5 split group 0, 6-9 epilogue, [10-13 im2col gather],
// then split group 1 (10-13, or 14-17 with the gather).  The two split groups
// take alternate k-blocks: one group's per-k-block latency chain (LDS -> split ->
// tcgen05.st / STS -> fences -> arrive) is longer than the 3 x 4 MMAs it feeds.
constexpr int THREADS = 448;
constexpr int THREADS_GATHER = 576;

#include "tc_prims.cuh"

// Descriptor of one K=8 slice `kk` (0..3) of a 128 x 32 operand tile.
//  K-major tile : 128 rows (M or N) x 128 B (32 k), row r at r*128 B, TMA SWIZZLE_128B
//                 -> SBO = 1024 B (8-row groups), LBO unused (16 B); slice kk at +32 B
//  MN-major tile: 4 boxes of [32 k-rows][32 mn] (4 KiB each), box j at j*4 KiB, k-row
//                 r at r*128 B, TMA SWIZZLE_128B_ATOM_32B (32-byte chunks, 4-row period)
//                 -> LBO = 4096 B (next 32 mn), SBO = 512 B (next 4 k-rows); slice kk at +1024 B
__device__ __forceinline__ uint64_t tile_desc(uint32_t tile, int mn_major, int kk) {
  return mn_major ? sdesc(tile + kk * 1024, 4096, 512, 1) : sdesc(tile + kk * 32, 16, 1024, 2);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

// Persistent, warp-specialised kernel; one CTA per SM walks the work units
// u = (split z, m-tile, n-tile) with the n-tile fastest.  Roles:
//   warp 0        TMA producer (B; and A for DOT)
//   warp 1        TMEM allocator (all 512 columns) + MMA issuer (one thread); two
//                 BN-column accumulators so the epilogue of unit j overlaps the MMAs of j+1
//   warps 2-5     split of each stage: A row -> TMEM hi/lo columns (one row per
//                 thread, TMEM lane quadrant = warp % 4); B -> lo tile in shared
//                 memory (the raw B tile is the hi operand)
//   warps 6-9     epilogue: tcgen05.ld TMEM -> registers -> C (TMEM lane quadrant = warp % 4)
//   warps 10-13   (GATHER) implicit im2col: A rows gathered from the NHWC input,
//                 16-byte cp.async straight into the SWIZZLE_128B K-major layout
//                 (zero-fill outside the image = the padding)
// Pipelines: full/conv/empty per smem stage (producer -> split -> MMA -> producer)
// and tfull/tempty per accumulator (MMA -> epilogue -> MMA); the stage index and
// phase run on a k-block counter that continues across units, so the producers
// prefetch the next unit while the current one finishes.
// CG = 2: a CTA pair (cluster of 2) computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 issued by the leader: each CTA holds its 128 rows of A
// and half of the B columns, so per-SM operand traffic and split work drop by a
// third; the follower's split and epilogue warps arrive on the leader's barriers,
// the MMA commits multicast to both CTAs.
template <bool GATHER, int BNT, int CG>
__global__ void __launch_bounds__(GATHER ? THREADS_GATHER : THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, float* __restrict__ C,
                   int M, int N, int K, int a_mn, int b_mn, int kb_per_split, int splits, ConvA cv, int raw_hi,
                   const __grid_constant__ EpiProg epi, float* __restrict__ dbg, int ldc,
                   const __grid_constant__ OutSegs segs) {
  using T = TC<BNT, CG, GATHER>;
  constexpr int BN = T::BN, SA = T::SA, SB = T::SB, LSTAGES = T::LSTAGES, BNH = BNT / CG;
  constexpr int TILE_A = T::TILE_A, TILE_B = T::TILE_B, LO_BYTES = T::LO_BYTES;
  constexpr int A_BASE = T::A_BASE, B_BASE = T::B_BASE, LO_BASE = T::LO_BASE, BAR_BASE = T::BAR_BASE, ACOL = T::ACOL;
  extern __shared__ uint8_t smem_raw[];
  // align to 1024 B by pointer arithmetic on the __shared__ array (keeps the shared
  // address space visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = (uint64_t*)(smem + BAR_BASE);
  const uint32_t bar0 = smem_u32(bars);
  auto fullA = [&](int s) { return bar0 + 8u * s; };
  auto emptyA = [&](int s) { return bar0 + 8u * (SA + s); };
  auto fullB = [&](int s) { return bar0 + 8u * (2 * SA + s); };
  auto emptyB = [&](int s) { return bar0 + 8u * (2 * SA + SB + s); };
  auto conv = [&](int l) { return bar0 + 8u * (2 * SA + 2 * SB + l); };
  auto lofree = [&](int l) { return bar0 + 8u * (2 * SA + 2 * SB + LSTAGES + l); };
  auto tfull = [&](int b) { return bar0 + 8u * (2 * SA + 2 * SB + 2 * LSTAGES + b); };
  auto tempty = [&](int b) { return bar0 + 8u * (2 * SA + 2 * SB + 2 * LSTAGES + 2 + b); };
  uint32_t* tmem_slot = (uint32_t*)(smem + BAR_BASE + 512);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const bool leader = rank == 0;
  const int tiles_m = (M + BM * CG - 1) / (BM * CG), tiles_n = (N + BN - 1) / BN;
  const int units = tiles_m * tiles_n * splits;
  const int nkt = (K + BK - 1) / BK;
  const int u_first = blockIdx.x / CG, u_step = gridDim.x / CG;
  // unit -> (z, m0 (this CTA's rows), n0, kb0, nk)
  auto unit = [&](int u, int& z, int& m0, int& n0, int& kb0, int& nk) {
    const int per = tiles_m * tiles_n;
    z = u / per;
    const int rem = u - z * per;
    m0 = (rem / tiles_n) * BM * CG + (int)rank * BM;
    n0 = (rem % tiles_n) * BN;
    kb0 = z * kb_per_split;
    nk = min(nkt - kb0, kb_per_split);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init(fullA(s), GATHER && !cv.tma ? 128 : 1);
      mbar_init(emptyA(s), 4);  // the 4 split warps of this CTA
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(fullB(s), 1);
      mbar_init(emptyB(s), 1);
    }
    for (int l = 0; l < LSTAGES; ++l) {
      mbar_init(conv(l), 4 * CG);
      mbar_init(lofree(l), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), 4 * CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (!GATHER || cv.tma) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2) cluster_sync();  // both CTAs' barriers initialised before any remote arrive
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int it = 0;
      for (int u = u_first; u < units; u += u_step) {
        int z, m0, n0, kb0, nk;
        unit(u, z, m0, n0, kb0, nk);
        // im2col TMA: traversal start = input position of this unit's first output pixel;
        // k-slab -> (tap (kh, kw) = im2col offsets, 32 channels from ci)
        int xw = 0, xh = 0, xn = 0, ci = 0, kh = 0, kw = 0;
        if (GATHER && cv.tma) {
          const int hw = cv.Ho * cv.Wo;
          xn = m0 / hw;
          const int q = m0 - xn * hw, ho = q / cv.Wo, wo = q - ho * cv.Wo;
          xh = ho * cv.sh - cv.pt;
          xw = wo * cv.sw - cv.pl;
          const int k0 = kb0 * BK, tap = k0 / cv.Ci;
          ci = k0 - tap * cv.Ci;
          kh = tap / cv.KW;
          kw = tap - kh * cv.KW;
        }
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int sa = it % SA, sb = it % SB;
          const int nb = n0 + (int)rank * BNH;
          const int k0 = (kb0 + kb) * BK;
          if (GATHER && cv.tma == 1) {  // one 128 x 32-channel box (one tap)
            mbar_wait(emptyA(sa), ((it / SA) & 1) ^ 1);
            mbar_expect_tx(fullA(sa), TILE_A);
            tma_load_im2col(sbase + A_BASE + sa * TILE_A, &mapA, ci, xw, xh, xn, (uint16_t)kw, (uint16_t)kh, fullA(sa));
            ci += BK;
            if (ci == cv.Ci) { ci = 0; if (++kw == cv.KW) { kw = 0; ++kh; } }
          } else if (GATHER && cv.tma == 2) {  // two 128 x 16-channel boxes (each within one tap)
            mbar_wait(emptyA(sa), ((it / SA) & 1) ^ 1);
            mbar_expect_tx(fullA(sa), TILE_A);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              // a half-slab past K (K % 32 == 16) loads from image N: out of bounds -> zeros
              const bool in_k = k0 + 16 * h < K;
              tma_load_im2col(sbase + A_BASE + sa * TILE_A + h * (TILE_A / 2), &mapA, ci, xw, xh, in_k ? xn : 1 << 30,
                              (uint16_t)kw, (uint16_t)kh, fullA(sa));
              ci += 16;
              if (ci == cv.Ci) { ci = 0; if (++kw == cv.KW) { kw = 0; ++kh; } }
            }
          }
          if (!GATHER) {
            mbar_wait(emptyA(sa), ((it / SA) & 1) ^ 1);
            const uint32_t st = sbase + A_BASE + sa * TILE_A;
            mbar_expect_tx(fullA(sa), TILE_A);
            if (a_mn) {
              for (int j = 0; j < BM / 32; ++j) tma_load_2d(st + j * 4096, &mapA, m0 + 32 * j, k0, fullA(sa));
            } else {
              tma_load_2d(st, &mapA, k0, m0, fullA(sa));
            }
          }
          mbar_wait(emptyB(sb), ((it / SB) & 1) ^ 1);
          const uint32_t bt = sbase + B_BASE + sb * TILE_B;
          mbar_expect_tx(fullB(sb), TILE_B);  // (this CTA's B share)
          if (b_mn) {
            for (int j = 0; j < BNH / 32; ++j) tma_load_2d(bt + j * 4096, &mapB, nb + 32 * j, k0, fullB(sb));
          } else {
            tma_load_2d(bt, &mapB, k0, nb, fullB(sb));
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // ---------------- MMA issuer (the leader CTA of a pair)
      // The whole warp walks the loop (its indices stay warp-uniform, so descriptors
      // live in uniform registers); one elected lane issues each tcgen05 op.  Issued
      // from a single lane the operands went through R2UR.BROADCAST loops and every
      // MMA cost ~108 cycles regardless of N (ncu + CG_TC_BN sweep).
      // instruction descriptor: D f32, A/B tf32, majors, N>>3, M>>4
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)b_mn << 16) |  // A (TMEM) K-major
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((BM * CG) >> 4) << 24);
      const uint64_t kstep = b_mn ? 64 : 2;  // descriptor address advance per K=8 slice (1024 B or 32 B, in 16 B)
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);  // (uniform)
      int it = 0, j = 0;
      for (int u = u_first; u < units; u += u_step, ++j) {
        int z, m0, n0, kb0, nk;
        unit(u, z, m0, n0, kb0, nk);
        const int b = j & 1;
        mbar_wait_warp(tempty(b), ((j >> 1) & 1) ^ 1);  // the epilogue has drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tm + (uint32_t)(b * BN);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int sb = it % SB, l = it % LSTAGES;
          mbar_wait_warp(conv(l), (it / LSTAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t dhi = tile_desc(sbase + B_BASE + sb * TILE_B, b_mn, 0);
          const uint64_t dlo = tile_desc(sbase + LO_BASE + l * LO_BYTES, b_mn, 0);
          const uint32_t ahi = tm + (uint32_t)(ACOL + l * 2 * BK), alo = ahi + BK;  // TMEM columns
          if (raw_hi != 4) {  // (4: measurement probe without MMAs)
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint32_t acc0 = (kb > 0 || kk > 0) ? 1u : 0u;
              // small terms first, then the leading hi.hi product
              if (raw_hi != 2) {
                mma_tf32_e<CG>(d, alo + kk * 8, dhi + kk * kstep, idesc, acc0);
                mma_tf32_e<CG>(d, ahi + kk * 8, dlo + kk * kstep, idesc, 1u);
              }
              mma_tf32_e<CG>(d, ahi + kk * 8, dhi + kk * kstep, idesc, raw_hi != 2 ? 1u : acc0);
            }
          }
          mma_commit_e<CG>(emptyB(sb));  // frees the raw B slot once these MMAs have read it
          mma_commit_e<CG>(lofree(l));   // and the lo slot
        }
        mma_commit_e<CG>(tfull(b));
      }
    }
  } else if (warp < 6 || warp >= (GATHER ? 14 : 10)) {
    // ---------------- split warps (two groups of 4, alternate k-blocks)
    const int grp = warp < 6 ? 0 : 1;                       // split group: k-blocks with it % 2 == grp
    const int t = (threadIdx.x - (grp ? (GATHER ? 448 : 320) : 64));  // 0..127: B chunks
    const int wq = warp % 4;         // TMEM lane quadrant this warp may access
    const int rr = wq * 32 + lane;   // the A tile row this thread owns
    int it = 0;
    for (int u = u_first; u < units; u += u_step) {
      int z, m0, n0, kb0, nk;
      unit(u, z, m0, n0, kb0, nk);
      for (int kb = 0; kb < nk; ++kb, ++it) {
        if ((it & 1) != grp) continue;
        const int sa = it % SA, sb = it % SB, l = it % LSTAGES;
        mbar_wait(fullA(sa), (it / SA) & 1);
        mbar_wait(lofree(l), ((it / LSTAGES) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");  // the MMAs that read this TMEM stage are done
        if (raw_hi == 3) {  // measurement probe: no split work (pipeline without the split)
          __syncwarp();
          if (lane == 0) mbar_arrive(emptyA(sa));
          mbar_wait(fullB(sb), (it / SB) & 1);
          if (lane == 0) {
            if (CG == 1 || leader) mbar_arrive(conv(l));
            else mbar_arrive_cta(conv(l), 0);
          }
          continue;
        }
        const uint32_t st = sbase + A_BASE + sa * TILE_A;
        if (dbg && u == 0 && kb == 0 && t < 8) dbg[t] = reinterpret_cast<float*>(smem + A_BASE)[t];  // A raw
        // A row rr (32 k values) -> registers.  K-major (TMA SWIZZLE_128B or the
        // gather's identical layout): 16-byte chunk c of row r sits at chunk c ^ (r & 7).
        // M-major (TMA SWIZZLE_128B_ATOM_32B, boxes [32 k][32 m] of 4 KiB): the 32-byte
        // chunk of element (k, m) is (m % 32) / 8 ^ (k & 3) within k-row k.
        uint32_t hv[32], lv[32];
        if (!GATHER && a_mn) {
          const uint32_t box = st + (uint32_t)(rr >> 5) * 4096u + (uint32_t)((lane & 7) << 2);
#pragma unroll
          for (int k = 0; k < 32; ++k) hv[k] = __float_as_uint(lds32(box + k * 128 + ((((lane >> 3) ^ (k & 3))) << 5)));
        } else if (GATHER && cv.tma == 2) {
          // two [128][16] SWIZZLE_64B half-tiles: 16-byte chunk c of row r at c ^ ((r >> 1) & 3)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t row = st + (uint32_t)h * (TILE_A / 2) + (uint32_t)rr * 64u;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float4 v = lds128(row + ((c ^ ((rr >> 1) & 3)) << 4));
              hv[16 * h + 4 * c] = __float_as_uint(v.x);
              hv[16 * h + 4 * c + 1] = __float_as_uint(v.y);
              hv[16 * h + 4 * c + 2] = __float_as_uint(v.z);
              hv[16 * h + 4 * c + 3] = __float_as_uint(v.w);
            }
          }
        } else {
          const uint32_t row = st + (uint32_t)rr * 128u;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = lds128(row + ((c ^ (rr & 7)) << 4));
            hv[4 * c] = __float_as_uint(v.x);
            hv[4 * c + 1] = __float_as_uint(v.y);
            hv[4 * c + 2] = __float_as_uint(v.z);
            hv[4 * c + 3] = __float_as_uint(v.w);
          }
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const uint32_t h = hv[k] & 0xFFFFE000u;
          lv[k] = __float_as_uint(__fsub_rn(__uint_as_float(hv[k]), __uint_as_float(h)));
          hv[k] = h;
        }
        const uint32_t ta = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(ACOL + l * 2 * BK);
        if (raw_hi != 7) tmem_st32(ta, hv);  // (7: measurement probe without the hi store)
        if (raw_hi != 2) tmem_st32(ta + BK, lv);
        __syncwarp();
        if (lane == 0) mbar_arrive(emptyA(sa));  // the row is in registers / TMEM: A slot free
        mbar_wait(fullB(sb), (it / SB) & 1);
        if (dbg && u == 0 && kb == 0 && t < 8) dbg[8 + t] = reinterpret_cast<float*>(smem + B_BASE)[t];  // B raw
        // B: lo tile in shared memory (the raw tile is read as hi by the tensor core,
        // which truncates fp32 operands to TF32; with raw_hi == 0 hi is written too)
        if (raw_hi != 2 && raw_hi != 6) {  // (6: measurement probe without the B split)
          const uint32_t hb = sbase + B_BASE + sb * TILE_B + t * 16, lb = sbase + LO_BASE + l * LO_BYTES + t * 16;
          constexpr int PER = TILE_B / 16 / 128;
          float4 v[PER];
#pragma unroll
          for (int q = 0; q < PER; ++q) v[q] = lds128(hb + q * 2048);
#pragma unroll
          for (int q = 0; q < PER; ++q) {
            float4 h, lo;
            h.x = __uint_as_float(__float_as_uint(v[q].x) & 0xFFFFE000u);
            h.y = __uint_as_float(__float_as_uint(v[q].y) & 0xFFFFE000u);
            h.z = __uint_as_float(__float_as_uint(v[q].z) & 0xFFFFE000u);
            h.w = __uint_as_float(__float_as_uint(v[q].w) & 0xFFFFE000u);
            lo.x = __fsub_rn(v[q].x, h.x);
            lo.y = __fsub_rn(v[q].y, h.y);
            lo.z = __fsub_rn(v[q].z, h.z);
            lo.w = __fsub_rn(v[q].w, h.w);
            if (!raw_hi) sts128(hb + q * 2048, h);
            sts128(lb + q * 2048, lo);
          }
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy);
        // TMEM stores complete and ordered before the arrive
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (CG == 1 || leader) mbar_arrive(conv(l));
          else mbar_arrive_cta(conv(l), 0);
        }
      }
    }
  } else if (warp < 10) {
    // ---------------- warps 6..9: epilogue; this warp may touch TMEM lanes [32*(warp%4), +32)
    const int sub = warp % 4;
    const bool vec = (N % 4) == 0 && (ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
    int j = 0;
    for (int u = u_first; u < units; u += u_step, ++j) {
      int z, m0, n0, kb0, nk;
      unit(u, z, m0, n0, kb0, nk);
      const int b = j & 1;
      mbar_wait(tfull(b), (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (dbg && u == 0 && sub == 0 && lane == 0) {
        dbg[16] = __uint_as_float(tmem);
        dbg[17] = (float)nk;
      }
      const int row = m0 + sub * 32 + lane;
      float* Cz = C + (size_t)z * M * N;
      if (epi.n) {  // this unit's per-column operands -> shared memory (named barrier: the 4 epilogue warps)
        float* es = reinterpret_cast<float*>(smem + T::EPI_BASE);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int i = threadIdx.x - 192; i < epi.n * BN; i += 128) {
          const int e = i / BN, c = i - e * BN, col = n0 + c;
          const float* xv = epi.x[e];
          if (segs.n && col < N) {  // column-routed: the segment's own operand vector
            int sg = 0;
            while (sg + 1 < segs.n && col >= segs.col[sg + 1]) ++sg;
            xv = segs.ex[sg][e] - segs.col[sg];
          }
          es[i] = epi.op[e] == EPI_RELU || epi.scalar[e] == 2
                      ? 0.f
                      : (epi.scalar[e] ? __ldg(epi.x[e]) : (col < N ? __ldg(xv + col) : 0.f));
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      const int cend = min(BN, N - n0);  // columns of this unit that exist (padding chunks skipped)
#pragma unroll 1
      for (int c0 = 0; c0 < cend; c0 += 16) {
        uint32_t r[16];
        const uint32_t taddr = tmem + ((uint32_t)(sub * 32) << 16) + (uint32_t)(b * BN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
              "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (epi.n) {  // fused elementwise epilogue, IEEE-rounded per op like the unfused kernel
          const float* es = reinterpret_cast<const float*>(smem + T::EPI_BASE) + c0;
          float vv[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) vv[q] = __uint_as_float(r[q]);
          for (int e = 0; e < epi.n; ++e) {
            if (epi.scalar[e] == 2) {  // a full [M, N] operand (row-major, ld = N): this row's 16 values
              float xe[16];
              const int n = n0 + c0;
              const float* xr = epi.x[e] + (size_t)min(row, M - 1) * N + n;
              if ((N % 4) == 0 && n + 16 <= N && (reinterpret_cast<uintptr_t>(epi.x[e]) & 15) == 0) {
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                  const float4 t = __ldg(reinterpret_cast<const float4*>(xr + q));
                  xe[q] = t.x; xe[q + 1] = t.y; xe[q + 2] = t.z; xe[q + 3] = t.w;
                }
              } else {
#pragma unroll
                for (int q = 0; q < 16; ++q) xe[q] = n + q < N ? __ldg(xr + q) : 0.f;
              }
              epi_apply<16>(vv, epi.op[e], epi.swap[e], xe);
            } else {
              epi_apply<16>(vv, epi.op[e], epi.swap[e], es + e * BN);
            }
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) r[q] = __float_as_uint(vv[q]);
        }
        if (row < M && n0 + c0 < N) {
          float* crow = Cz + (size_t)row * ldc;
          int n = n0 + c0;
          bool vseg = vec;
          int nend = N;
          if (segs.n) {  // column-routed: this chunk's segment (uniform across the warp)
            int sg = 0;
            while (sg + 1 < segs.n && n >= segs.col[sg + 1]) ++sg;
            nend = sg + 1 < segs.n ? segs.col[sg + 1] : N;
            crow = segs.C[sg] + (size_t)row * segs.ldc[sg] - segs.col[sg];
            vseg = (segs.ldc[sg] % 4) == 0 && (reinterpret_cast<uintptr_t>(segs.C[sg]) & 15) == 0 && (segs.col[sg] % 4) == 0;
          }
          if (vseg && n + 16 <= nend) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              *reinterpret_cast<float4*>(crow + n + 4 * q) =
                  make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                              __uint_as_float(r[4 * q + 3]));
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (n + q < nend) crow[n + q] = __uint_as_float(r[q]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (CG == 1 || leader) mbar_arrive(tempty(b));
        else mbar_arrive_cta(tempty(b), 0);
      }
    }
  } else if (GATHER && !cv.tma) {
    // ---------------- warps 10..13: im2col gather of A, one tile row (output pixel) per thread.
    // The (kh, kw, ci) position of the k-slab is advanced incrementally (no
    // per-chunk divisions); with Ci % 32 == 0 a whole slab is one tap: one
    // contiguous 128-byte run of channels per row.
    const int r = threadIdx.x - 320;
    int it = 0;
    for (int u = u_first; u < units; u += u_step) {
      int z, m0, n0, kb0, nk;
      unit(u, z, m0, n0, kb0, nk);
      const int m = m0 + r;
      int n = 0, ho = 0, wo = 0;
      if (m < M) {
        const int hw = cv.Ho * cv.Wo;
        n = m / hw;
        const int q = m - n * hw;
        ho = q / cv.Wo;
        wo = q - ho * cv.Wo;
      }
      const int hb = ho * cv.sh - cv.pt, wb = wo * cv.sw - cv.pl;
      const float* img = cv.x + (size_t)n * cv.H * cv.W * cv.Ci;
      // slab start k0 = kb0 * BK  ->  (kh, kw, ci)
      int k0 = kb0 * BK;
      int tap = k0 / cv.Ci, ci = k0 - tap * cv.Ci;
      int kh = tap / cv.KW, kw = tap - kh * cv.KW;
      const bool row_ok = m < M;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % SA;
        mbar_wait(emptyA(s), ((it / SA) & 1) ^ 1);
        const uint32_t row = sbase + A_BASE + s * TILE_A + r * 128;
        if (raw_hi == 5) {  // measurement probe: no gather (stale A tile)
          mbar_arrive(fullA(s));
          continue;
        }
        if ((cv.Ci & 31) == 0) {  // the slab is 32 channels of one tap
          const int hi = hb + kh, wi = wb + kw;
          const bool ok = row_ok && k0 < K && hi >= 0 && hi < cv.H && wi >= 0 && wi < cv.W;
          const float* src = ok ? img + ((size_t)hi * cv.W + wi) * cv.Ci + ci : cv.x;
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) cp_async16(row + ((jj ^ (r & 7)) << 4), src + (ok ? 4 * jj : 0), ok ? 16u : 0u);
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(fullA(s)) : "memory");
          ci += BK;
          if (ci >= cv.Ci) { ci = 0; if (++kw == cv.KW) { kw = 0; ++kh; } }
          k0 += BK;
        } else if ((cv.Ci & 3) == 0) {  // 4 consecutive k = 4 channels of one tap: one 16-byte async copy
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int hi = hb + kh, wi = wb + kw;
            const bool ok = row_ok && k0 < K && hi >= 0 && hi < cv.H && wi >= 0 && wi < cv.W;
            const float* src = ok ? img + ((size_t)hi * cv.W + wi) * cv.Ci + ci : cv.x;
            cp_async16(row + ((jj ^ (r & 7)) << 4), src, ok ? 16u : 0u);
            ci += 4;
            if (ci >= cv.Ci) { ci = 0; if (++kw == cv.KW) { kw = 0; ++kh; } }
            k0 += 4;
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(fullA(s)) : "memory");
        } else {  // few input channels (e.g. RGB): element-wise gather, 16-byte shared stores
          // all 32 loads in flight before the first store (the stores' memory clobber
          // would otherwise serialise 8 rounds of L2 latency per slab: C5 stem 1.2 ms)
          float e[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int hi = hb + kh, wi = wb + kw;
            const bool ok = row_ok && k0 < K && hi >= 0 && hi < cv.H && wi >= 0 && wi < cv.W;
            e[q] = ok ? __ldg(img + ((size_t)hi * cv.W + wi) * cv.Ci + ci) : 0.f;
            if (++ci == cv.Ci) { ci = 0; if (++kw == cv.KW) { kw = 0; ++kh; } }
            ++k0;
          }
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            sts128(row + ((jj ^ (r & 7)) << 4), make_float4(e[4 * jj], e[4 * jj + 1], e[4 * jj + 2], e[4 * jj + 3]));
          mbar_arrive(fullA(s));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2) cluster_sync();  // the pair's MMAs (which write both TMEMs) are all complete
  else __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

// 2-D fp32 row-major matrix [rows, cols] (cols contiguous), box {32 cols, box_rows}.
// K-major operand tiles use SWIZZLE_128B; MN-major ones the 32-byte-atom variant.
bool make_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int box_rows, bool mn_major) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);
EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeIm2colFn)p;
  });
  return fn;
}

// NHWC input as a rank-4 im2col map {C, W, H, N}: 32 channels x 128 pixels per load,
// SWIZZLE_128B rows (the K-major A tile layout).  Bounding box per spatial dim:
// lower = -pad, upper chosen so the strided traversal visits exactly the Wo (Ho)
// output positions: box = (Wo - 1) * sw + 1.
bool make_im2col_map(CUtensorMap* m, const float* x, int n, int h, int w, int ci, int ho, int wo, int sh, int sw, int pt,
                     int pl, int chans) {
  EncodeIm2colFn fn = encode_im2col_fn();
  if (!fn || ci % chans || (reinterpret_cast<uintptr_t>(x) & 15)) return false;
  const int lw = -pl, lh = -pt;
  const int uw = lw + (wo - 1) * sw + 1 - w, uh = lh + (ho - 1) * sh + 1 - h;
  if (lw < -128 || lh < -128 || uw < -128 || uw > 127 || uh < -128 || uh > 127) return false;
  cuuint64_t dims[4] = {(cuuint64_t)ci, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)ci * 4, (cuuint64_t)w * ci * 4, (cuuint64_t)h * w * ci * 4};
  const int lower[2] = {lw, lh}, upper[2] = {uw, uh};
  cuuint32_t estr[4] = {1, (cuuint32_t)sw, (cuuint32_t)sh, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)x, dims, strides, lower, upper, (cuuint32_t)chans, BM, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, chans == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool dot_tc_supported(int M, int N, int K, int ta, int tb) {
  // TMA: global row pitch must be a multiple of 16 B, i.e. the contiguous extent % 4 == 0
  const int64_t a_cols = ta ? M : K, b_cols = tb ? K : N;
  if (a_cols % 4 || b_cols % 4) return false;
  if (M < 1 || N < 1 || K < 1) return false;
  // skinny products are HBM-bound; they stay on the SIMT path
  return M >= 64 && N >= 32 && K >= 8;
}

// N tile: 256 columns when that wastes no more padding than 128 (halves the
// operand traffic per FLOP: A is re-read per N tile), else 128.
int pick_bn(int M, int N, int num_sms, int K) {
  // narrow outputs (convs with 32 / 64 channels): a matching MMA N instead of padding to 128
  if (N <= 32) return 32;
  if (N <= 64) return 64;
  if (const char* e = getenv("CG_TC_BN")) {  // measurement override: only the instantiated tile widths
    const int v = atoi(e);
    if (v == 32 || v == 64 || v == 128) return v;
  }
  // fewer 128-wide tiles than half the SMs and a short K (C4's batch x 84..400 layers:
  // 64 tiles, K <= 400): 64-wide tiles put twice as many CTAs to work on the
  // latency-bound pipeline (-13 us per C4 iteration); with a long K split-K fills the
  // machine instead (C3's weight gradients, K = 4096: 64-wide was 48 us slower)
  const long long tiles128 = (long long)((M + BM - 1) / BM) * ((N + 127) / 128);
  if (tiles128 < num_sms / 2 && K <= 1024) return 64;
  return 128;  // TMEM: 2 x BN accumulator columns + the A stages fit 512 columns for BN <= 128
}

// CTA pairs (cta_group::2, 256-row tiles) when the problem has at least a wave
// of pair units; BN >= 64 so each CTA's half of B is >= 32 columns.
int pick_cg(int M, int N, int bn, int splits, int num_sms, bool gather) {
  (void)gather;  // implicit-GEMM convs pair too (C5: 36.4 -> 34.4 ms)
  if (getenv("CG_TC_NO_PAIRS") || bn < 64 || M < 256) return 1;
  const long long units2 = (long long)((M + 2 * BM - 1) / (2 * BM)) * ((N + bn - 1) / bn) * splits;
  return units2 >= num_sms / 2 ? 2 : 1;  // at least one full wave of pairs
}

void dot_tc_split(int M, int N, int K, int num_sms, int* splits, int* kb_per_split) {
  const int bn = pick_bn(M, N, num_sms, K);
  const long long tiles = (long long)((M + BM - 1) / BM) * ((N + bn - 1) / bn);
  const int nk = (K + BK - 1) / BK;
  // split-K: minimise (waves x k-blocks per unit) + the partials' HBM round trip
  // (S x M x N x 8 B at ~6.5 TB/s, in units of one k-block ~0.45 us) + the finalize
  int S = 1;
  double best = 1e300;
  for (int s = 1; s <= std::max(1, std::min(16, nk / 4)); ++s) {
    const int per_s = (nk + s - 1) / s;
    const int s_eff = (nk + per_s - 1) / per_s;
    const long long waves = (tiles * s_eff + num_sms - 1) / num_sms;
    // (+4 k-blocks for the finalize launch; a split output also cannot take a fused epilogue)
    const double cost = (double)waves * per_s + (s_eff > 1 ? 4.0 + (double)s_eff * M * N * 8.0 / 2.9e6 : 0.0);
    if (cost < best - 1e-9) best = cost, S = s_eff;
  }
  const int per = (nk + S - 1) / S;
  *kb_per_split = per;
  *splits = (nk + per - 1) / per;
}

size_t dot_tc_ws_floats(int M, int N, int K, int num_sms) {
  int S, per;
  dot_tc_split(M, N, K, num_sms, &S, &per);
  return S > 1 ? (size_t)S * M * N : 0;
}

int dot_tc_prepare(DotTcPlan* p, const float* A, const float* B, float* C, int M, int N, int K, int ta, int tb,
                   float* ws, int num_sms) {
  if (!dot_tc_supported(M, N, K, ta, tb)) return -1;
  std::memset(p, 0, sizeof(*p));
  p->M = M; p->N = N; p->K = K;
  p->num_sms = num_sms;
  p->raw_hi = 1;  // tcgen05 kind::tf32 truncates fp32 operands (tests: test_tf32_truncation_probe)
  if (getenv("CG_PROBE_1XTF32")) p->raw_hi = 2;  // measurement probe only (lower accuracy)
  if (getenv("CG_PROBE_MODE")) p->raw_hi = atoi(getenv("CG_PROBE_MODE"));  // 3: no split, 4: no MMA (wrong results)
  dot_tc_split(M, N, K, num_sms, &p->splits, &p->kb_per_split);
  p->ws = ws;
  if (p->splits > 1 && !ws) return -3;
  p->a_mn = ta; p->b_mn = tb ? 0 : 1;
  p->C = C;
  // A: ta = 0 -> [M, K] (K-major, box 32 k x 128 m); ta = 1 -> [K, M] (M-major, box 32 m x 32 k)
  bool ok = ta ? make_map(reinterpret_cast<CUtensorMap*>(p->mapA), A, K, M, 32, true)
               : make_map(reinterpret_cast<CUtensorMap*>(p->mapA), A, M, K, BM, false);
  // B: tb = 0 -> [K, N] (N-major, box 32 n x 32 k); tb = 1 -> [N, K] (K-major, box 32 k x BN/CG n)
  p->bn = pick_bn(M, N, num_sms, K);
  p->cg = pick_cg(M, N, p->bn, p->splits, num_sms, false);
  ok = ok && (tb ? make_map(reinterpret_cast<CUtensorMap*>(p->mapB), B, N, K, p->bn / p->cg, false)
                 : make_map(reinterpret_cast<CUtensorMap*>(p->mapB), B, K, N, 32, true));
  return ok ? 0 : -2;
}

template <bool G, int BNT, int CG>
cudaError_t launch_tc(const DotTcPlan& p, float* out, cudaStream_t s) {
  using T = TC<BNT, CG, G>;
  const cudaError_t attr_err = smem_attr((const void*)gemm_tc_kernel<G, BNT, CG>, T::SMEM_BYTES);  // per device
  if (attr_err != cudaSuccess) return attr_err;
  const int units = ((p.M + BM * CG - 1) / (BM * CG)) * ((p.N + BNT - 1) / BNT) * p.splits;
  const int grid = std::max(1, std::min(units, p.num_sms / CG)) * CG;
  const CUtensorMap& a = *reinterpret_cast<const CUtensorMap*>(p.mapA);
  const CUtensorMap& b = *reinterpret_cast<const CUtensorMap*>(p.mapB);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(G ? THREADS_GATHER : THREADS);
  cfg.dynamicSmemBytes = T::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<G, BNT, CG>, a, b, out, p.M, p.N, p.K, G ? 0 : p.a_mn, G ? 1 : p.b_mn,
                            p.kb_per_split, p.splits, p.conv, p.raw_hi, p.epi, p.dbg,
                            p.splits > 1 || p.ldc <= 0 ? p.N : p.ldc, p.segs);
}

template <bool G, int BNT>
cudaError_t launch_tc_cg(const DotTcPlan& p, float* out, cudaStream_t s) {
  if constexpr (BNT >= 64) {
    if (p.cg == 2) return launch_tc<G, BNT, 2>(p, out, s);
  }
  return launch_tc<G, BNT, 1>(p, out, s);
}

cudaError_t launch_dot_tc(const DotTcPlan& p, cudaStream_t s) {
  if (p.band == 1) return launch_conv_band(p.conv.x, p.band_w, p.C, p.ldc > 0 ? p.ldc : p.N, p.band_n, p.epi, p.num_sms, s);
  if (p.band >= 2)
    return launch_conv_rows(p.band - 1, p.conv.x, p.band_w, p.C, p.ldc > 0 ? p.ldc : p.N, p.band_n, p.epi, p.num_sms, s);
  float* out = p.splits > 1 ? p.ws : p.C;
  cudaError_t e0;
  switch (p.bn) {
    case 64: e0 = p.conv.x ? launch_tc_cg<true, 64>(p, out, s) : launch_tc_cg<false, 64>(p, out, s); break;
    case 32: e0 = p.conv.x ? launch_tc_cg<true, 32>(p, out, s) : launch_tc_cg<false, 32>(p, out, s); break;
    case 128: e0 = p.conv.x ? launch_tc_cg<true, 128>(p, out, s) : launch_tc_cg<false, 128>(p, out, s); break;
    default: return cudaErrorInvalidValue;  // no instantiation: never launch with a B slot of the wrong size
  }
  if (e0 != cudaSuccess) return e0;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || p.splits == 1) return e;
  return launch_reduce_finalize(p.ws, p.C, (long long)p.M * p.N, p.splits, 0, s);
}

bool conv_tc_supported(int ci, int co, long long m) { return co % 4 == 0 && co >= 16 && m >= 128; }

int conv_tc_prepare(DotTcPlan* p, const float* x, const float* w, float* y, int n, int h, int wd, int ci, int kh, int kw,
                    int co, int ho, int wo, int sh, int sw, int pt, int pl, float* ws, int num_sms) {
  const long long M = (long long)n * ho * wo;
  if (!conv_tc_supported(ci, co, M) || M > INT32_MAX) return -1;
  std::memset(p, 0, sizeof(*p));
  p->M = (int)M; p->N = co; p->K = kh * kw * ci;
  p->num_sms = num_sms;
  p->raw_hi = getenv("CG_PROBE_1XTF32") ? 2 : 1;
  if (getenv("CG_PROBE_MODE")) p->raw_hi = atoi(getenv("CG_PROBE_MODE"));  // 3 no split, 4 no MMA, 5 no gather
  dot_tc_split(p->M, p->N, p->K, num_sms, &p->splits, &p->kb_per_split);
  p->ws = ws;
  if (p->splits > 1 && !ws) return -3;
  p->a_mn = 0; p->b_mn = 1;
  p->C = y;
  p->conv = ConvA{x, h, wd, ci, ho, wo, kw, sh, sw, pt, pl, 0};
  // A by TMA im2col: 32-channel boxes when Ci % 32 == 0, pairs of 16-channel boxes when Ci % 16 == 0
  if (!getenv("CG_CONV_NO_IM2COL_TMA") && sh <= 8 && sw <= 8) {
    CUtensorMap* ma = reinterpret_cast<CUtensorMap*>(p->mapA);
    if (ci % 32 == 0 && make_im2col_map(ma, x, n, h, wd, ci, ho, wo, sh, sw, pt, pl, 32)) p->conv.tma = 1;
    else if (ci % 16 == 0 && make_im2col_map(ma, x, n, h, wd, ci, ho, wo, sh, sw, pt, pl, 16)) p->conv.tma = 2;
  }
  p->bn = pick_bn(p->M, co, num_sms, p->K);
  p->cg = pick_cg(p->M, co, p->bn, p->splits, num_sms, true);
  if (conv_band_supported(n, h, wd, ci, kh, kw, co, ho, wo, sh, sw, pt, pl)) {  // the stem: row bands, no split-K
    p->band = 1;
    p->splits = 1;
    p->band_w = w;
    p->band_n = n;
  } else if (const int kind = conv_rows_kind(h, wd, ci, kh, kw, co, ho, wo, sh, sw, pt, pl)) {  // stem 3x3: row ring
    p->band = 1 + kind;
    p->splits = 1;
    p->band_w = w;
    p->band_n = n;
  }
  // B = weights as a [K, Co] row-major matrix (N-major), like DOT with tb = 0
  return make_map(reinterpret_cast<CUtensorMap*>(p->mapB), w, p->K, co, 32, true) ? 0 : -2;
}

size_t conv_tc_ws_floats(long long M, int co, int K, int num_sms) {
  return M > INT32_MAX ? 0 : dot_tc_ws_floats((int)M, co, K, num_sms);
}

}  // namespace cg

// ---- debug entry (tests/tools only): one DOT on device buffers, optional dump
extern "C" int cgx_dot_tc(const float* A, const float* B, float* C, int M, int N, int K, int ta, int tb, float* dbg,
                          int raw_hi) {
  cg::DotTcPlan p;
  int rc = cg::dot_tc_prepare(&p, A, B, C, M, N, K, ta, tb, nullptr, 1);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p.num_sms = sms;
  if (rc) return rc;
  p.dbg = dbg;
  p.raw_hi = raw_hi;
  cudaError_t e = cg::launch_dot_tc(p, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e == cudaSuccess ? 0 : -100 - (int)e;
}
