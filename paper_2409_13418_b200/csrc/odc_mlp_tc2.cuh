// odc_mlp_tc2.cuh -- CTA-pair (cta_group::2) tcgen05 evaluator of the MLP.
//
// A cluster of two CTAs (two SMs of one TPC) evaluates a 256-point tile
// (128 rows per CTA) through the 8 layers with tcgen05.mma.cta_group::2
// (M = 256, N = 128, K = 16):
//   * A (activations) lives in TMEM (TS form): the epilogue writes the next
//     layer's bf16 activations with tcgen05.st, double-buffered, so shared
//     memory carries only weights;
//   * B (weights) is split along N: each CTA streams its 64-row half of every
//     (layer, N half, K half) block of the weights (16 KB, 2 K-atoms) into a
//     12-stage ring with cp.async.bulk; the leader's MMA reads both halves;
//   * D (fp32 accumulators) per CTA: its 128 rows x N, in TMEM.
// Per SM and layer that is 64 KB of weights through shared memory per 2048
// MMA cycles (32 B/clk), against 128 B/clk for the single-CTA SS version.
//
// Roles per CTA (384 threads):
//   warp 0      producer (lane 0): own weight half -> ring stage, local full[s]
//   warp 1      leader only: MMA issuer (lane 0)
//   warp 2      TMEM allocator (cta_group::2, both CTAs)
//   warp 3      peer only: relays local full[s] completion to the leader (fullp[s])
//   warps 4-7   epilogue, accumulator columns 0..127   (warp%4 = lane quarter)
//   warps 8-11  epilogue, accumulator columns 128..255
// TMEM columns: D half 0 [0,128), D half 1 [128,256), A buffer 0 [256,384),
// A buffer 1 [384,512).  Layer l reads A[l%2]; its epilogue writes A[(l+1)%2].
#pragma once
#include <cstdint>

#include "odc_mlp_tc.cuh"

namespace odc {
namespace tc2 {

constexpr int kThreads = 384;
constexpr int kStages = 12;           // ring of weight stages
constexpr int kStageBytes = 16384;    // per CTA: 64 rows x K 128 (2 K-atoms of 8 KB)
constexpr int kStagesPerTile = 30;    // (layer, N half, K half); layer 0 has one K half
constexpr uint32_t kIdesc = (1u << 4)      // D f32
                            | (1u << 7)    // A bf16
                            | (1u << 10)   // B bf16
                            | (16u << 17)  // N = 128
                            | (16u << 24); // M = 256 (CTA pair)
constexpr size_t kSmemBytes = 1024 + kStages * kStageBytes + 1024 + (8 * 256 + 256 + 256) * 4;

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Relaxed remote arrive.  A release.cluster arrive compiles to MEMBAR.ALL.GPU
// + ERRBAR (~600 ns on the critical path).  Use only where the data the
// arrive publishes is already complete in shared memory: bulk-copy data
// observed through complete_tx, or generic stores that their writers fenced
// (fence.proxy.async) and released at CTA scope before this thread acquired
// them -- shared memory is not cached, so a performed store is what the
// peer's tensor-core read sees.
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(kIdesc), "r"(accumulate));
}
// arrive on the barrier at this offset in both CTAs of the pair when all
// previously issued tcgen05 ops of this thread have completed
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          tc::smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

#define ODC_TMEM_ST32(taddr, r)                                                                                     \
  asm volatile(                                                                                                     \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"  \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),                                     \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),  \
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),   \
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),   \
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])                                                                \
      : "memory")
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

}  // namespace tc2
}  // namespace odc
