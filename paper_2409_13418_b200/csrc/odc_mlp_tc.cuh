// odc_mlp_tc.cuh -- tcgen05/TMEM evaluator of the occupancy MLP (sm_100a).
//
// One persistent CTA per SM evaluates two 128-point tiles at a time through
// all 8 layers.  Roles (384 threads):
//   warp 0      weight producer: streams 16 KB weight chunks (K 64 x N 128,
//               pre-packed on the host in the UMMA K-major SWIZZLE_128B smem
//               image) with cp.async.bulk into an NS-stage ring
//   warp 1      MMA issuer: one thread issues tcgen05.mma (M=128, N=128,
//               K=16, bf16 x bf16 -> f32) for both tiles from every chunk, so
//               each weight byte fetched from L2 feeds 256 points
//   warp 2      TMEM allocator (512 columns: tile t, half nh -> col t*256+nh*128)
//   warps 4-11  epilogue, 128 threads per tile (warp%4 = TMEM lane quarter):
//               positional encoding -> A tile; tcgen05.ld accumulators,
//               bias + ReLU -> bf16 -> next layer's A tile (swizzled st.shared);
//               fp32 head dot product + fp64 prior -> label.
// Layer order per tile pair: for l: for nh in {0,1}: for kc: chunk(l,nh,kc).
// The epilogue drains half 0 while the MMA runs half 1, keeps it in
// registers until the layer's MMAs finished reading A, then writes it; the
// next layer's first two K chunks only need half 0, so the MMA restarts
// before half 1 is written.
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

namespace odc {
namespace tc {

constexpr int kThreads = 384;
constexpr int kStages = 5;
constexpr int kChunkBytes = 16384;        // 128 rows x 128 B
constexpr int kTileABytes = 4 * 16384;    // 128 rows x 256 bf16 (4 K-atoms)
constexpr int kChunksPerPair = 2 + 7 * 8; // layer 0: K=64 (1 kc) x 2 halves; layers 1-7: 4 kc x 2 halves
constexpr uint32_t kIdesc = (1u << 4)      // D f32
                            | (1u << 7)    // A bf16
                            | (1u << 10)   // B bf16
                            | (16u << 17)  // N = 128
                            | (8u << 24);  // M = 128
constexpr size_t kSmemBytes = 1024 + 2 * kTileABytes + kStages * kChunkBytes + 256 + (8 * 256 + 256) * 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Bounded wait: a protocol bug traps (kernel error) after g_mbar_timeout_ns
// (default 4 s; odc_set_param("mbar_timeout_ms"), 0 = wait forever) instead
// of hanging the GPU.
__device__ unsigned long long g_mbar_timeout_ns = 4000000000ull;
__device__ __forceinline__ bool mbar_timed_out(uint64_t& t0) {
  const uint64_t t = globaltimer_ns();
  if (t0 == 0) {
    t0 = t;
    return false;
  }
  const unsigned long long lim = *(volatile unsigned long long*)&g_mbar_timeout_ns;
  return lim != 0 && t - t0 > lim;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t spins = 0;; spins++) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
    if ((spins & 1023) == 0 && mbar_timed_out(t0)) __trap();
  }
}
// mbar_wait with cluster-scope acquire: for data a peer CTA stored into this
// CTA's shared memory before its release.cluster arrive
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t spins = 0;; spins++) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
    if ((spins & 1023) == 0 && mbar_timed_out(t0)) __trap();
  }
}
// Spin on the non-blocking test_wait (no suspend); bounded like mbar_wait.
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t spins = 0;; spins++) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
    if ((spins & 1023) == 0 && mbar_timed_out(t0)) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// one lane of the (converged) warp returns true
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(e));
  return e != 0;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, SBO = 1024 B (8 rows
// x 128 B), LBO = 16 B (unused for swizzled K-major), version 1.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;          // LBO (16 B units)
  d |= (uint64_t)(1024 >> 4) << 32; // SBO
  d |= (uint64_t)1 << 46;          // version
  d |= (uint64_t)2 << 61;          // SWIZZLE_128B
  return d;
}

// Descriptor split: the low word carries the start address (>> 4) and LBO;
// the high word (SBO = 1024 B, version 1, SWIZZLE_128B) is the same for every
// operand, so per-MMA descriptors are a 32-bit add on a base low word.
constexpr uint32_t kDescHi = (uint32_t)(((uint64_t)(1024 >> 4) << 32 | (uint64_t)1 << 46 | (uint64_t)2 << 61) >> 32);
__device__ __forceinline__ uint32_t desc_lo(uint32_t saddr) { return ((saddr >> 4) & 0x3FFF) | (1u << 16); }
__device__ __forceinline__ uint64_t make_desc(uint32_t lo) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "r"(lo), "r"(kDescHi));
  return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#define ODC_TMEM_LD32(taddr, r)                                                                                    \
  asm volatile(                                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19," \
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                                    \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), \
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),     \
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),    \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                 \
      : "r"(taddr))
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
// byte offset of 16-byte chunk c (8 bf16 along K) of row r inside a K-atom
__device__ __forceinline__ uint32_t sw128_off(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

}  // namespace tc
}  // namespace odc
