// odc_mlp.cu -- MlpField evaluator.  This file holds the SIMT evaluator
// (bf16 operands, fp32 accumulate) used until the tcgen05 path is selected;
// see odc_mlp.h for the field definition.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "odc_mlp.h"

namespace odc {

constexpr int kWidth = 256;
constexpr int kDepth = 8;
constexpr int kDin = 39;
constexpr int kDinPad = 64;
constexpr int kPts = 32;  // points per block (SIMT evaluator)

size_t mlp_packed_weight_elems() { return (size_t)kDinPad * kWidth + (size_t)(kDepth - 1) * kWidth * kWidth; }

static uint16_t f2bf(float f) {  // inputs are already bf16-representable
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16);
}

// row-major W[k][n] per layer; layer 0 zero-padded to K = 64
void mlp_pack_weights(const float* w0, int d_in, const float* w_hidden, uint16_t* out) {
  for (int k = 0; k < kDinPad; k++)
    for (int n = 0; n < kWidth; n++) out[(size_t)k * kWidth + n] = k < d_in ? f2bf(w0[(size_t)k * kWidth + n]) : 0;
  uint16_t* o = out + (size_t)kDinPad * kWidth;
  for (size_t i = 0; i < (size_t)(kDepth - 1) * kWidth * kWidth; i++) o[i] = f2bf(w_hidden[i]);
}

__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

__device__ __forceinline__ void point_of(const PointSrc& s, int64_t i, double p[3]) {
  if (s.pts) {
    p[0] = s.pts[3 * i];
    p[1] = s.pts[3 * i + 1];
    p[2] = s.pts[3 * i + 2];
  } else {
    vposition(s.grid, s.begin + i, p);
  }
}

// positional encoding gamma(p - 0.5): [x(3), sin_0(3), cos_0(3), ..., sin_5(3), cos_5(3)]
__device__ __forceinline__ float pe_feature(const double p[3], int j) {
  if (j >= kDin) return 0.f;
  if (j < 3) return (float)(p[j] - 0.5);
  const int k = (j - 3) / 6, r = (j - 3) % 6, c = r % 3;
  const float x = (float)(p[c] - 0.5);
  float sv, cv;
  sincospif(x * (float)(1 << k), &sv, &cv);
  return r < 3 ? sv : cv;
}

__global__ void __launch_bounds__(kWidth) k_mlp_simt(MlpDev m, PointSrc src, int64_t n, uint8_t* __restrict__ labels,
                                                     double* __restrict__ raw) {
  __shared__ float h[kPts][kWidth];
  __shared__ float red[kPts][kWidth / 32];
  const int64_t p0 = (int64_t)blockIdx.x * kPts;
  const int j = threadIdx.x;
  for (int t = j; t < kPts * kDinPad; t += kWidth) {
    const int pi = t / kDinPad, f = t % kDinPad;
    float v = 0.f;
    if (p0 + pi < n) {
      double p[3];
      point_of(src, p0 + pi, p);
      v = pe_feature(p, f);
    }
    h[pi][f] = bf16r(v);
  }
  __syncthreads();
  const __nv_bfloat16* W = reinterpret_cast<const __nv_bfloat16*>(m.w_packed);
  float acc[kPts];
  for (int layer = 0; layer < kDepth; layer++) {
    const int K = layer == 0 ? kDinPad : kWidth;
    for (int pi = 0; pi < kPts; pi++) acc[pi] = 0.f;
    for (int k = 0; k < K; k++) {
      const float w = __bfloat162float(W[(size_t)k * kWidth + j]);
#pragma unroll
      for (int pi = 0; pi < kPts; pi++) acc[pi] = fmaf(h[pi][k], w, acc[pi]);
    }
    W += (size_t)K * kWidth;
    const float b = m.bias[layer * kWidth + j];
    __syncthreads();
    for (int pi = 0; pi < kPts; pi++) {
      float v = acc[pi] + b;
      v = v > 0.f ? v : 0.f;
      h[pi][j] = layer == kDepth - 1 ? v : bf16r(v);
    }
    __syncthreads();
  }
  // head: fp32 dot product, fixed order (per-warp partials then warps in order)
  const float wh = m.w_head[j];
  for (int pi = 0; pi < kPts; pi++) {
    float v = h[pi][j] * wh;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((j & 31) == 0) red[pi][j >> 5] = v;
  }
  __syncthreads();
  if (j < kPts && p0 + j < n) {
    float s = 0.f;
    for (int w = 0; w < kWidth / 32; w++) s += red[j][w];
    const double mlp = (double)(s + m.b_head);
    double p[3];
    point_of(src, p0 + j, p);
    double d[3] = {p[0] - m.prior_center[0], p[1] - m.prior_center[1], p[2] - m.prior_center[2]};
    const double dist = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    const double logit = m.amplitude * mlp - m.prior_scale * (dist - m.prior_radius);
    const double r = 1.0 / (1.0 + exp(-logit));
    labels[p0 + j] = r > 0.5 ? 1 : 0;
    if (raw) raw[p0 + j] = r;
  }
}

int mlp_eval(const MlpDev& m, const PointSrc& src, int64_t n, uint8_t* labels, double* raw, cudaStream_t s) {
  if (n <= 0) return 0;
  const int64_t blocks = (n + kPts - 1) / kPts;
  k_mlp_simt<<<(unsigned)blocks, kWidth, 0, s>>>(m, src, n, labels, raw);
  return 0;
}

const char* mlp_kernel_name() { return "k_mlp_simt"; }

}  // namespace odc
