// Microbenchmark: back-to-back tcgen05.mma throughput for the operand forms
// the MLP kernels use (cycles per instruction per SM, clock64 on the issuing
// thread; one commit + wait at the end).  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o mma_mb mma_microbench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)64 << 32) | (1ull << 46) | (2ull << 61);
}
template <int CG, int M, int N, bool TS>
__global__ void __launch_bounds__(128, 1) kmb(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) base[i] = 0;
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t a = smem_u32(base), b = smem_u32(base + 32768);
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
      const uint32_t ks = (i & 3) * 32;
      const uint32_t acc = i > 0;
      if (TS) {
        if (CG == 1)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(tmem + 256 + (i & 3) * 8), "l"(desc(b + ks)), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(tmem + 256 + (i & 3) * 8), "l"(desc(b + ks)), "r"(idesc), "r"(acc));
      } else {
        if (CG == 1)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(desc(a + ks)), "l"(desc(b + ks)), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(desc(a + ks)), "l"(desc(b + ks)), "r"(idesc), "r"(acc));
      }
    }
    if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    else
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.b32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  if (CG == 2 && threadIdx.x == 0 && rank == 1) {  // peer waits for the multicast commit too
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.b32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  else __syncthreads();
  if (warp == 0) {
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int CG, int M, int N, bool TS>
void run(const char* name) {
  auto k = kmb<CG, M, N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaMemset(d, 0, 148 * 8);
  const int iters = 4096;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 70000;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; rep++) cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; i += CG) mx = h[i] > mx ? h[i] : mx;
  const double macs_per_sm = (double)M * N * 16 / CG;
  printf("%-28s err=%d  cycles/instr %.1f  (ideal at 4096 MAC/clk/SM: %.1f)\n", name, (int)e, (double)mx / iters,
         macs_per_sm / 4096.0);
  cudaFree(d);
}

int main() {
  run<1, 128, 128, false>("cg1 SS M128 N128");
  run<1, 128, 256, false>("cg1 SS M128 N256");
  run<1, 128, 128, true>("cg1 TS M128 N128");
  run<1, 128, 256, true>("cg1 TS M128 N256");
  run<2, 256, 128, true>("cg2 TS M256 N128");
  run<2, 256, 256, true>("cg2 TS M256 N256");
  run<2, 256, 128, false>("cg2 SS M256 N128");
  run<2, 256, 256, false>("cg2 SS M256 N256");
  return 0;
}
