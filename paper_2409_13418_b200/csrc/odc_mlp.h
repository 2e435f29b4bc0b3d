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
  const uint16_t* w_tc;      // 58 chunks of 128x64 bf16 in the UMMA SWIZZLE_128B smem image (odc_mlp_tc.cuh)
  int debug;                 // timing experiments, odc_profile_mlp only (results are wrong):
                             // 1 no weight refills after the first ring, 8 static round-robin schedule,
                             // 4 every label through fp64, 16 every label decided in fp32
  int has_bias;              // any non-zero bias (selects the bias-add epilogue)
  unsigned long long* trace; // profiling: event timeline of CTA 0 (nullptr = off)
  // dynamic pair schedule: a per-context device counter that only
  // grows; mlp_eval() sets sched_base from *sched_next and advances it
  unsigned long long* sched;
  unsigned long long sched_base;
  const float* bias;         // (8, 256)
  const float* w_head;       // (256)
  float w_head_k[256];       // the same by value: kernel-parameter (constant) space, so the
                             // CTA-pair head's uniform weight reads are FFMA constant operands
  float b_head;
  double amplitude, prior_scale, prior_radius;
  double prior_center[3];
};

// Points source: explicit (pts != nullptr) or grid vertices [begin, begin+n)
struct PointSrc {
  const double* pts;
  GridP grid;
  int64_t begin;
  // grid sources, filled in by mlp_eval: per-axis encoding table (x, sin_k,
  // cos_k of every coordinate index, 16 floats per row) and a fast divisor by S
  const float* petab;
  uint32_t fd_m, fd_s;
  // compacted batches: the point count is read on the
  // device (n is then only the launch's upper bound) and label/raw i goes
  // to out_map[i]
  const int64_t* n_dev;
  const int32_t* out_map;
  // set by mlp_eval (labels only): fp32-undecided labels are written
  // as 2 with their head dot here, and finished in fp64 by k_mlp_fixup
  float* defer_dot;
  // parity hook (odc_eval_mlp_dot): the fp32 head dot of every point
  float* dot_out;
};

// host: pack float32 weights (already bf16-representable) into the device layout
size_t mlp_tc_weight_elems();
void mlp_pack_weights_tc(const float* w0, int d_in, const float* w_hidden, uint16_t* out);

// labels (u8) and optionally raw = sigmoid(logit) (f64) for n points
// (k_mlp_tc4, the CTA-pair tcgen05 evaluator).  Needs m.sched and
// sched_next (the host copy of the counter's value at the next launch,
// advanced here).  Returns the number of kernels it launched (0 for n == 0),
// negative when the counter or the weights are missing.
int mlp_eval(const MlpDev& m, const PointSrc& src, int64_t n, uint8_t* labels, double* raw, cudaStream_t s,
             unsigned long long* sched_next = nullptr);
const char* mlp_kernel_name();
// The evaluator's mbarrier waits trap (a kernel error instead of a hung GPU)
// after this long without progress; 0 waits forever (debuggers, heavy
// preemption).  Default 4 s.  Applies to the current device.
int mlp_set_wait_timeout_ns(unsigned long long ns);

}  // namespace odc
