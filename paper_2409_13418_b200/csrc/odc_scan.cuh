// odc_scan.cuh -- hand-written multi-channel exclusive scans (block scans for
// the single-pass look-back scan and the tiled reduce-then-scan, odc_kernels.cu).
//
// Every ordered output of the pipeline (edge rows, instance ids, cell rows,
// partition ids, triangle offsets, fan-vertex ids, repair vertex ids) is an
// exclusive prefix sum of per-element counts, so output order is fixed by
// the index space, never by atomics.
#pragma once
#include <cstdint>

namespace odc {

constexpr int kScanBlock = 256;

// Block-wide exclusive scan of NCH channels; returns per-thread exclusive
// prefix and (to all threads) the block total.
template <int NCH, int BLOCK = kScanBlock>
__device__ __forceinline__ void block_exscan(const uint32_t (&v)[NCH], uint32_t (&excl)[NCH],
                                             uint32_t (&total)[NCH]) {
  static_assert(BLOCK % 32 == 0 && BLOCK <= 1024, "block of whole warps");
  __shared__ uint32_t wsum[NCH][BLOCK / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t incl[NCH];
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    uint32_t x = v[c];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    incl[c] = x;
    if (lane == 31) wsum[c][wid] = x;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      uint32_t x = lane < BLOCK / 32 ? wsum[c][lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane < BLOCK / 32) wsum[c][lane] = x;  // inclusive over warps
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    uint32_t before = wid == 0 ? 0u : wsum[c][wid - 1];
    excl[c] = before + incl[c] - v[c];
    total[c] = wsum[c][BLOCK / 32 - 1];
  }
  __syncthreads();
}

// Single-block exclusive scan of tile sums (NCH channels laid out [c][ntiles]);
// writes offsets in place and the 64-bit totals.  Each thread owns kPer
// consecutive tiles per round (a serial sum in registers), so a round of
// 1024 threads covers 8 K tiles and the block-wide steps run 8x less often.
template <int NCH>
__global__ void __launch_bounds__(1024) k_scan_tiles(uint32_t* sums, int64_t ntiles, unsigned long long* totals) {
  constexpr int kPer = 8;
  __shared__ unsigned long long carry[NCH];
  __shared__ unsigned long long wpart[NCH][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x < NCH) carry[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t base = 0; base < ntiles; base += 1024 * kPer) {
    const int64_t i0 = base + (int64_t)threadIdx.x * kPer;
    unsigned long long tot[NCH], x[NCH];
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      tot[c] = 0;
#pragma unroll
      for (int k = 0; k < kPer; k++) tot[c] += i0 + k < ntiles ? sums[c * ntiles + i0 + k] : 0u;
      x[c] = tot[c];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, x[c], o);
        if (lane >= o) x[c] += y;
      }
      if (lane == 31) wpart[c][wid] = x[c];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
      for (int c = 0; c < NCH; c++) {
        unsigned long long y = wpart[c][lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          unsigned long long z = __shfl_up_sync(0xffffffffu, y, o);
          if (lane >= o) y += z;
        }
        wpart[c][lane] = y;
      }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      unsigned long long run = (wid == 0 ? 0ull : wpart[c][wid - 1]) + carry[c] + x[c] - tot[c];
#pragma unroll
      for (int k = 0; k < kPer; k++) {
        if (i0 + k < ntiles) {
          const uint32_t v = sums[c * ntiles + i0 + k];
          sums[c * ntiles + i0 + k] = (uint32_t)run;
          run += v;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < NCH) carry[threadIdx.x] += wpart[threadIdx.x][31];
    __syncthreads();
  }
  if (threadIdx.x < NCH) totals[threadIdx.x] = carry[threadIdx.x];
}

}  // namespace odc
