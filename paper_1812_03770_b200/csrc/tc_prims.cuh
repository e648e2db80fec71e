// tcgen05 / TMEM / mbarrier / TMA device primitives shared by the tensor-core
// kernels (dot_tc.cu, conv_img_tc.cu).  Included inside an anonymous namespace.
#pragma once
#include <cuda.h>
#include <cstdint>

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
// expect more transaction bytes on the current phase without arriving (a later
// arrive.expect_tx of the same phase completes it)
__device__ __forceinline__ void mbar_expect_tx_only(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
#ifndef CG_LAZY_NS
#define CG_LAZY_NS 128
#endif
// optional suspend-time hint (ns) for try_wait (A/B measurement only, see below)
#ifdef CG_MBAR_HINT
#define CG_MBAR_HINT_ARG ", %3"
#define CG_MBAR_HINT_OP , "n"(CG_MBAR_HINT)
#else
#define CG_MBAR_HINT_ARG ""
#define CG_MBAR_HINT_OP
#endif

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
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2" CG_MBAR_HINT_ARG ";\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity) CG_MBAR_HINT_OP
        : "memory");
    if (done) return;
    // watchdog: a lost arrival must fail the launch (10 s), not hang the GPU
    if (t0 == 0) t0 = globaltimer();
    else if (globaltimer() - t0 > 10000000000ull) __trap();
  }
}

// Wait for a role that is known to run ahead (its slack hides a late wake-up):
// back off with nanosleep between polls, so a spinning warp does not take
// shared-memory-pipe slots from the roles on the critical path.
__device__ __forceinline__ void mbar_wait_lazy(uint32_t bar, uint32_t parity) {
  uint64_t t0 = 0;
  while (true) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(CG_LAZY_NS);
    if (t0 == 0) t0 = globaltimer();
    else if (globaltimer() - t0 > 10000000000ull) __trap();
  }
}

// Warp-collective wait: the exit condition is a vote, so code after it stays
// provably warp-uniform (lets the compiler keep MMA operands in uniform registers).
__device__ __forceinline__ void mbar_wait_warp(uint32_t bar, uint32_t parity) {
  uint64_t t0 = 0;
  while (true) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2" CG_MBAR_HINT_ARG ";\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity) CG_MBAR_HINT_OP
        : "memory");
    if (__all_sync(0xffffffffu, done)) return;
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

// 1-D bulk copy global -> shared (TMA engine), completion counted in bytes on `bar`.
// dst, src and bytes must be multiples of 16.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// im2col load of 128 output pixels x 32 channels: TMA walks the pixels from (w, h, n)
// through the map's bounding box (conv strides = traversal strides) and reads channels
// [c, c + 32) at pixel + (off_w, off_h); outside the image -> zero.
__device__ __forceinline__ void tma_load_im2col(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                                uint16_t off_w, uint16_t off_h, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6], "
      "{%7, %8};" ::"r"(dst),
      "l"(map), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bar), "h"(off_w), "h"(off_h)
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

// 32 consecutive columns of this thread's TMEM lane (warp-collective, lane quadrant = warp % 4)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,"
      "%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]),
      "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),
      "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]),
      "r"(r[31])
      : "memory");
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}

// arrive on the mbarrier at the same shared-memory offset in CTA `cta` of the cluster.
// Default (.release.cta) semantics: what the peer consumes after this arrive is
// TMEM / shared memory read by the tensor core, ordered by the tcgen05 and proxy
// fences issued before it.  (.release.cluster compiled to MEMBAR.ALL.GPU + ERRBAR
// and made the follower CTA's split the pair's critical path: ncu, 8192^3 DOT.)
__device__ __forceinline__ void mbar_arrive_cta(uint32_t bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(cta));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Warp-collective forms: every lane computes the (uniform) operands, elect.sync
// picks the one lane that issues.  CG = 2: the pair instruction (leader CTA only)
// and a commit multicast to the barrier at this offset in both CTAs.
template <int CG>
__device__ __forceinline__ void mma_tf32_e(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t accum) {
  if (CG == 1)
    asm volatile(
        "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(accum));
  else
    asm volatile(
        "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(accum));
}
template <int CG>
__device__ __forceinline__ void mma_commit_e(uint32_t bar) {
  if (CG == 1)
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
        : "memory");
  else
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(bar),
        "h"((uint16_t)3)
        : "memory");
}
