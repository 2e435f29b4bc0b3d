// odc_mlp.h -- occupancy MLP evaluator (MlpField, BASELINE config 3).
//
//   gamma(p) = [x, sin(2^k pi x), cos(2^k pi x)]_{k<6},  x = p - 0.5   (39 -> padded 64)
//   h_0 = relu(gamma W_0 + b_0); h_i = relu(h_{i-1} W_i + b_i), i = 1..7 (256 wide)
//   mlp = h_7 . w_head + b_head
//   logit = amplitude*mlp - prior_scale*(|p - c| - r);  raw = sigmoid(logit); label = raw > 0.5
//
// bf16 operands, fp32 accumulation.  Every point's result is independent of
// the batch it is evaluated in (no split-K, fixed K order), which the
// shared-field parity oracle relies on.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "odc_device.cuh"

namespace odc {

struct MlpDev {
  // tensor-core layout (UMMA canonical K-major, see odc_mlp.cu)
  const uint16_t* w_packed;  // 8 layers of bf16 weights, each N=256 x K (K=64 for layer 0, 256 after)
  const float* bias;         // (8, 256)
  const float* w_head;       // (256)
  float b_head;
  double amplitude, prior_scale, prior_radius;
  double prior_center[3];
};

// Points source: explicit (pts != nullptr) or grid vertices [begin, begin+n)
struct PointSrc {
  const double* pts;
  GridP grid;
  int64_t begin;
};

size_t mlp_packed_weight_elems();
// host: pack float32 weights (already bf16-representable) into the device layout
void mlp_pack_weights(const float* w0, int d_in, const float* w_hidden, uint16_t* out);

// labels (u8) and optionally raw = sigmoid(logit) (f64) for n points
int mlp_eval(const MlpDev& m, const PointSrc& src, int64_t n, uint8_t* labels, double* raw, cudaStream_t s);
const char* mlp_kernel_name();

}  // namespace odc
