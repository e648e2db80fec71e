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
// One CTA computes a BM x BN = 128 x 128 output tile:
//   warp 0      TMA producer: loads the raw fp32 A/B k-slab (BK = 32, one 128-byte
//               swizzle row) of stage s with cp.async.bulk.tensor (OOB -> 0, so
//               ragged M/N/K need no masking on the load side)
//   warp 1      TMEM allocator + MMA issuer (one elected thread): 3 x 4
//               tcgen05.mma.kind::tf32 per stage, tcgen05.commit -> empty[s]
//   warps 2-5   split hi/lo in shared memory (elementwise, layout-preserving, so
//               the swizzle of the TMA tile is the swizzle of the hi and lo
//               tiles), then the epilogue: tcgen05.ld TMEM -> registers -> C.
// Operand majorness comes from the transposes: A is K-major when ta = 0 and
// M-major when ta = 1; B is N-major when tb = 0 and K-major when tb = 1.  Both
// are native UMMA smem layouts for TF32 (instruction-descriptor bits 15/16),
// so transposed operands never take a transpose pass.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "dot_tc.h"
#include "kernels.h"

#include <algorithm>

namespace cg {

namespace {

constexpr int BM = 128, BK = 32;
// Tile configurations (N = 128 or 256 columns per unit).  Decoupled rings: the
// raw operand tiles (TMA / gather destinations, also the hi operands) live in a
// ring that runs ahead of the MMAs; the lo tiles written by the split warps only
// live from the split to the MMA.
template <int BNT, int CG = 1>
struct TC {
  static constexpr int BN = BNT;
  static constexpr int TILE_A = BM * BK * 4;           // 16 KiB
  static constexpr int TILE_B = BNT / CG * BK * 4;     // this CTA's share of the B tile
  static constexpr int STAGE_BYTES = TILE_A + TILE_B;
  static constexpr int LO_BYTES = TILE_A + TILE_B;
  static constexpr int LSTAGES = 2;                    // lo ring
  static constexpr int EPI_BYTES = kEpiMax * BNT * 4;
  static constexpr int STAGES_FIT = (220 * 1024 - LSTAGES * LO_BYTES - EPI_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 6 ? 6 : STAGES_FIT;   // raw ring
  static constexpr int LO_BASE = STAGES * STAGE_BYTES;
  static constexpr int EPI_BASE = LO_BASE + LSTAGES * LO_BYTES;   // fused-epilogue operands [kEpiMax][BN]
  static constexpr int BAR_BASE = EPI_BASE + EPI_BYTES;
  static constexpr int SMEM_BYTES = BAR_BASE + 1024 /*barriers*/ + 1024 /*alignment slack*/;
  static_assert(STAGES >= 2, "pipeline depth");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};
constexpr int THREADS = 320;         // TMA, MMA, 4 split warps, 4 epilogue warps
constexpr int THREADS_GATHER = 448;  // + 4 warps gathering the im2col A tile

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// Blocking wait on an mbarrier phase (try_wait suspends briefly in hardware; an
// explicit suspend-time hint compiled to NANOSLEEP.SYNCS and made waiters
// oversleep the phase flip: measured 45 -> 63 ms on C5 with fused epilogues).
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    // watchdog: a lost arrival must fail the launch (10 s), not hang the GPU
    if (t0 == 0) t0 = globaltimer();
    else if (globaltimer() - t0 > 10000000000ull) __trap();
  }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// UMMA shared-memory descriptor (version 1 = sm_100).  layout: 2 = SWIZZLE_128B
// (16-byte chunks), 1 = SWIZZLE_128B_BASE32B (32-byte chunks; the only swizzled
// MN-major layout TF32 operands have).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)layout << 61;
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

// arrive on the mbarrier at the same shared-memory offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cta(uint32_t bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
// commit of a CTA-pair MMA: arrive on the barrier at this offset in both CTAs
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
               "h"((uint16_t)3)
               : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

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
//   warp 1        TMEM allocator + MMA issuer (one thread); two 128-column
//                 accumulators so the epilogue of unit j overlaps the MMAs of j+1
//   warps 2-5     hi/lo split of each stage (writes lo; the raw tile is the hi operand)
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
                   const __grid_constant__ EpiProg epi, float* __restrict__ dbg) {
  using T = TC<BNT, CG>;
  constexpr int BN = T::BN, STAGES = T::STAGES, LSTAGES = T::LSTAGES, BNH = BNT / CG;
  constexpr int TILE_A = T::TILE_A, TILE_B = T::TILE_B, STAGE_BYTES = T::STAGE_BYTES, LO_BYTES = T::LO_BYTES;
  constexpr int LO_BASE = T::LO_BASE, BAR_BASE = T::BAR_BASE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = (uint64_t*)(smem + BAR_BASE);
  const uint32_t bar0 = smem_u32(bars);
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto conv = [&](int l) { return bar0 + 8u * (2 * STAGES + l); };
  auto lofree = [&](int l) { return bar0 + 8u * (2 * STAGES + LSTAGES + l); };
  auto tfull = [&](int b) { return bar0 + 8u * (2 * STAGES + 2 * LSTAGES + b); };
  auto tempty = [&](int b) { return bar0 + 8u * (2 * STAGES + 2 * LSTAGES + 2 + b); };
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
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), GATHER ? 1 + 128 : 1);
      mbar_init(empty(s), 1);
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
    if (!GATHER) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(2 * BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(2 * BN));
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
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(empty(s), ph ^ 1);
          const uint32_t st = sbase + s * STAGE_BYTES;
          mbar_expect_tx(full(s), GATHER ? TILE_B : TILE_A + TILE_B);  // (this CTA's B share)
          const int nb = n0 + (int)rank * BNH;
          const int k0 = (kb0 + kb) * BK;
          if (GATHER) {
          } else if (a_mn) {
            for (int j = 0; j < BM / 32; ++j) tma_load_2d(st + j * 4096, &mapA, m0 + 32 * j, k0, full(s));
          } else {
            tma_load_2d(st, &mapA, k0, m0, full(s));
          }
          if (b_mn) {
            for (int j = 0; j < BNH / 32; ++j) tma_load_2d(st + TILE_A + j * 4096, &mapB, nb + 32 * j, k0, full(s));
          } else {
            tma_load_2d(st + TILE_A, &mapB, k0, nb, full(s));
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (the leader CTA of a pair)
      // instruction descriptor: D f32, A/B tf32, majors, N>>3, M>>4
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((BM * CG) >> 4) << 24);
      int it = 0, j = 0;
      for (int u = u_first; u < units; u += u_step, ++j) {
        int z, m0, n0, kb0, nk;
        unit(u, z, m0, n0, kb0, nk);
        const int b = j & 1;
        mbar_wait(tempty(b), ((j >> 1) & 1) ^ 1);  // the epilogue has drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(b * BN);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES, l = it % LSTAGES;
          mbar_wait(conv(l), (it / LSTAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = sbase + s * STAGE_BYTES, lo = sbase + LO_BASE + l * LO_BYTES;
          const uint32_t ahi = st, bhi = st + TILE_A, alo = lo, blo = lo + TILE_A;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t acc0 = (kb > 0 || kk > 0) ? 1u : 0u;
            // small terms first, then the leading hi.hi product
            if (CG == 1) {
              if (raw_hi != 2) {
                mma_tf32(d, tile_desc(alo, a_mn, kk), tile_desc(bhi, b_mn, kk), idesc, acc0);
                mma_tf32(d, tile_desc(ahi, a_mn, kk), tile_desc(blo, b_mn, kk), idesc, 1u);
              }
              mma_tf32(d, tile_desc(ahi, a_mn, kk), tile_desc(bhi, b_mn, kk), idesc, raw_hi != 2 ? 1u : acc0);
            } else {
              if (raw_hi != 2) {
                mma_tf32_pair(d, tile_desc(alo, a_mn, kk), tile_desc(bhi, b_mn, kk), idesc, acc0);
                mma_tf32_pair(d, tile_desc(ahi, a_mn, kk), tile_desc(blo, b_mn, kk), idesc, 1u);
              }
              mma_tf32_pair(d, tile_desc(ahi, a_mn, kk), tile_desc(bhi, b_mn, kk), idesc, raw_hi != 2 ? 1u : acc0);
            }
          }
          if (CG == 1) {
            mma_commit(empty(s));   // frees the raw slot once these MMAs have read it
            mma_commit(lofree(l));  // and the lo slot
          } else {
            mma_commit_pair(empty(s));
            mma_commit_pair(lofree(l));
          }
        }
        if (CG == 1) mma_commit(tfull(b));
        else mma_commit_pair(tfull(b));
      }
    }
  } else if (warp < 6) {
    // ---------------- warps 2..5: hi/lo split of each stage
    const int t = threadIdx.x - 64;  // 0..127
    int it = 0;
    for (int u = u_first; u < units; u += u_step) {
      int z, m0, n0, kb0, nk;
      unit(u, z, m0, n0, kb0, nk);
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % STAGES, l = it % LSTAGES;
        mbar_wait(full(s), (it / STAGES) & 1);
        mbar_wait(lofree(l), ((it / LSTAGES) & 1) ^ 1);
        if (dbg && u == 0 && kb == 0 && t < 8) {
          dbg[t] = reinterpret_cast<float*>(smem)[t];                   // A raw
          dbg[8 + t] = reinterpret_cast<float*>(smem + TILE_A)[t];  // B raw
        }
        if (raw_hi == 2) {  // probe only: 1xTF32 (no split) to measure what the split costs
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if (CG == 1 || leader) mbar_arrive(conv(l));
            else mbar_arrive_cta(conv(l), 0);
          }
          continue;
        }
        // 16 float4 per thread: all loads first (ILP), explicit shared-space ops
        const uint32_t hb = sbase + s * STAGE_BYTES + t * 16, lb = sbase + LO_BASE + l * LO_BYTES + t * 16;
        constexpr int PER = STAGE_BYTES / 16 / 128;
        float4 v[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) v[q] = lds128(hb + q * 2048);
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          float4 h, l;
          h.x = __uint_as_float(__float_as_uint(v[q].x) & 0xFFFFE000u);
          h.y = __uint_as_float(__float_as_uint(v[q].y) & 0xFFFFE000u);
          h.z = __uint_as_float(__float_as_uint(v[q].z) & 0xFFFFE000u);
          h.w = __uint_as_float(__float_as_uint(v[q].w) & 0xFFFFE000u);
          l.x = __fsub_rn(v[q].x, h.x);
          l.y = __fsub_rn(v[q].y, h.y);
          l.z = __fsub_rn(v[q].z, h.z);
          l.w = __fsub_rn(v[q].w, h.w);
          // The A tile of a GATHER stage was written by cp.async / st.shared of other
          // threads (generic proxy); rewriting it here, followed by this thread's
          // proxy fence, is what makes it visible to the tensor core.  TMA tiles are
          // async-proxy writes already, so with raw_hi they are read as they are.
          if (!raw_hi || (GATHER && q < TILE_A / 2048)) sts128(hb + q * 2048, h);
          sts128(lb + q * 2048, l);
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
    const bool vec = (N % 4) == 0;
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
          es[i] = epi.op[e] == EPI_RELU ? 0.f : (epi.scalar[e] ? __ldg(epi.x[e]) : (col < N ? __ldg(epi.x[e] + col) : 0.f));
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
          for (int e = 0; e < epi.n; ++e) {
            const int op = epi.op[e], sw = epi.swap[e];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              float v = __uint_as_float(r[q]);
              const float xv = es[e * BN + q];
              const float a = sw ? xv : v, bb = sw ? v : xv;
              switch (op) {
                case EPI_ADD: v = __fadd_rn(a, bb); break;
                case EPI_SUB: v = __fsub_rn(a, bb); break;
                case EPI_MUL: v = __fmul_rn(a, bb); break;
                case EPI_DIV: v = __fdiv_rn(a, bb); break;
                case EPI_RELU: v = v > 0.f ? v : 0.f; break;
                case EPI_MAX: asm("max.NaN.f32 %0, %1, %2;" : "=f"(v) : "f"(a), "f"(bb)); break;
                case EPI_MIN: asm("min.NaN.f32 %0, %1, %2;" : "=f"(v) : "f"(a), "f"(bb)); break;
              }
              r[q] = __float_as_uint(v);
            }
          }
        }
        if (row < M && n0 + c0 < N) {
          float* crow = Cz + (size_t)row * N;
          const int n = n0 + c0;
          if (vec && n + 16 <= N) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              *reinterpret_cast<float4*>(crow + n + 4 * q) =
                  make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                              __uint_as_float(r[4 * q + 3]));
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (n + q < N) crow[n + q] = __uint_as_float(r[q]);
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
  } else if (GATHER) {
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
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(empty(s), ph ^ 1);
        const uint32_t row = sbase + s * STAGE_BYTES + r * 128;
        if ((cv.Ci & 31) == 0) {  // the slab is 32 channels of one tap
          const int hi = hb + kh, wi = wb + kw;
          const bool ok = row_ok && k0 < K && hi >= 0 && hi < cv.H && wi >= 0 && wi < cv.W;
          const float* src = ok ? img + ((size_t)hi * cv.W + wi) * cv.Ci + ci : cv.x;
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) cp_async16(row + ((jj ^ (r & 7)) << 4), src + (ok ? 4 * jj : 0), ok ? 16u : 0u);
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full(s)) : "memory");
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
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full(s)) : "memory");
        } else {  // few input channels (e.g. RGB): element-wise gather, 16-byte shared stores
          for (int jj = 0; jj < 8; ++jj) {
            float e[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int hi = hb + kh, wi = wb + kw;
              const bool ok = row_ok && k0 < K && hi >= 0 && hi < cv.H && wi >= 0 && wi < cv.W;
              e[q] = ok ? __ldg(img + ((size_t)hi * cv.W + wi) * cv.Ci + ci) : 0.f;
              if (++ci == cv.Ci) { ci = 0; if (++kw == cv.KW) { kw = 0; ++kh; } }
              ++k0;
            }
            sts128(row + ((jj ^ (r & 7)) << 4), make_float4(e[0], e[1], e[2], e[3]));
          }
          mbar_arrive(full(s));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2) cluster_sync();  // the pair's MMAs (which write both TMEMs) are all complete
  else __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
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
int pick_bn(int M, int N, int num_sms) {
  // narrow outputs (convs with 32 / 64 channels): a matching MMA N instead of padding to 128
  if (N <= 32) return 32;
  if (N <= 64) return 64;
  const int w128 = (N + 127) / 128 * 128 - N, w256 = (N + 255) / 256 * 256 - N;
  const long long units256 = (long long)((M + BM - 1) / BM) * ((N + 255) / 256);
  // only with enough units for two waves: otherwise the wider tile just idles SMs
  return (N >= 256 && w256 <= w128 && units256 >= 2LL * num_sms) ? 256 : 128;
}

// CTA pairs (cta_group::2, 256-row tiles) when the problem has at least a wave
// of pair units and no split-K; BN >= 64 so each CTA's half of B is >= 32 columns.
// Measured: 8192^3 DOT 200 -> 220 TFLOP/s; C5's gathered convs 43 -> 48 ms (their
// cost is the per-CTA A side, and the pair couples two CTAs' splits), so
// implicit-GEMM convs stay on single CTAs.
int pick_cg(int M, int N, int bn, int splits, int num_sms, bool gather) {
  if (gather || getenv("CG_TC_NO_PAIRS") || splits != 1 || bn < 64 || M < 256) return 1;
  const long long units2 = (long long)((M + 2 * BM - 1) / (2 * BM)) * ((N + bn - 1) / bn);
  return units2 >= num_sms ? 2 : 1;
}

void dot_tc_split(int M, int N, int K, int num_sms, int* splits, int* kb_per_split) {
  const int bn = pick_bn(M, N, num_sms);
  const int tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
  const int nk = (K + BK - 1) / BK;
  int S = 1;
  if (tiles < num_sms) S = std::max(1, std::min((num_sms + tiles - 1) / tiles, nk / 4));
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
  dot_tc_split(M, N, K, num_sms, &p->splits, &p->kb_per_split);
  p->ws = ws;
  if (p->splits > 1 && !ws) return -3;
  p->a_mn = ta; p->b_mn = tb ? 0 : 1;
  p->C = C;
  // A: ta = 0 -> [M, K] (K-major, box 32 k x 128 m); ta = 1 -> [K, M] (M-major, box 32 m x 32 k)
  bool ok = ta ? make_map(reinterpret_cast<CUtensorMap*>(p->mapA), A, K, M, 32, true)
               : make_map(reinterpret_cast<CUtensorMap*>(p->mapA), A, M, K, BM, false);
  // B: tb = 0 -> [K, N] (N-major, box 32 n x 32 k); tb = 1 -> [N, K] (K-major, box 32 k x BN/CG n)
  p->bn = pick_bn(M, N, num_sms);
  p->cg = pick_cg(M, N, p->bn, p->splits, num_sms, false);
  ok = ok && (tb ? make_map(reinterpret_cast<CUtensorMap*>(p->mapB), B, N, K, p->bn / p->cg, false)
                 : make_map(reinterpret_cast<CUtensorMap*>(p->mapB), B, K, N, 32, true));
  return ok ? 0 : -2;
}

template <bool G, int BNT, int CG>
cudaError_t launch_tc(const DotTcPlan& p, float* out, cudaStream_t s) {
  using T = TC<BNT, CG>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_tc_kernel<G, BNT, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM_BYTES);
  });
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
                            p.kb_per_split, p.splits, p.conv, p.raw_hi, p.epi, p.dbg);
}

template <bool G, int BNT>
cudaError_t launch_tc_cg(const DotTcPlan& p, float* out, cudaStream_t s) {
  if constexpr (BNT >= 64) {
    if (p.cg == 2) return launch_tc<G, BNT, 2>(p, out, s);
  }
  return launch_tc<G, BNT, 1>(p, out, s);
}

cudaError_t launch_dot_tc(const DotTcPlan& p, cudaStream_t s) {
  float* out = p.splits > 1 ? p.ws : p.C;
  cudaError_t e0;
  switch (p.bn) {
    case 256: e0 = p.conv.x ? launch_tc_cg<true, 256>(p, out, s) : launch_tc_cg<false, 256>(p, out, s); break;
    case 64: e0 = p.conv.x ? launch_tc_cg<true, 64>(p, out, s) : launch_tc_cg<false, 64>(p, out, s); break;
    case 32: e0 = p.conv.x ? launch_tc_cg<true, 32>(p, out, s) : launch_tc_cg<false, 32>(p, out, s); break;
    default: e0 = p.conv.x ? launch_tc_cg<true, 128>(p, out, s) : launch_tc_cg<false, 128>(p, out, s); break;
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
  dot_tc_split(p->M, p->N, p->K, num_sms, &p->splits, &p->kb_per_split);
  p->ws = ws;
  if (p->splits > 1 && !ws) return -3;
  p->a_mn = 0; p->b_mn = 1;
  p->C = y;
  p->conv = ConvA{x, h, wd, ci, ho, wo, kw, sh, sw, pt, pl};
  p->bn = pick_bn(p->M, co, num_sms);
  p->cg = pick_cg(p->M, co, p->bn, p->splits, num_sms, true);
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
