// odc_mlp.cu -- MlpField evaluator.  This file holds the SIMT evaluator
// (bf16 operands, fp32 accumulate) used until the tcgen05 path is selected;
// see odc_mlp.h for the field definition.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "odc_mlp.h"
#include "odc_mlp_tc.cuh"
#include "odc_mlp_tc2.cuh"  // cluster helpers (mapa, named barriers, pair commits) used by k_mlp_tc4

namespace odc {

// Timeline trace of CTA 0 (profiling hook, odc_profile_mlp): clock64 at
// pipeline events of the first two tiles; slot = ((tile*8 + layer)*16 + event).
#define ODC_TRACE(t, l, e)                                                                   \
  do {                                                                                       \
    if (m.trace && blockIdx.x == 0 && (t) < 2) m.trace[((t) * 8 + (l)) * 16 + (e)] = clock64(); \
  } while (0)

constexpr int kWidth = 256;
constexpr int kDepth = 8;
constexpr int kDin = 39;
static_assert(kDin <= 48, "tc4 skips layer-0 K-step 3 (features 48..63 are padding)");

static uint16_t f2bf(float f) {  // inputs are already bf16-representable
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16);
}

__device__ __forceinline__ void point_of(const PointSrc& s, int64_t i, double p[3]) {
  if (s.pts) {
    p[0] = s.pts[3 * i];
    p[1] = s.pts[3 * i + 1];
    p[2] = s.pts[3 * i + 2];
  } else {
    vposition(s.grid, s.begin + i, p);
  }
}

// ===========================================================================
// tcgen05 / TMEM evaluator (see odc_mlp_tc.cuh for the structure)
// ===========================================================================
size_t mlp_tc_weight_elems() { return (size_t)tc::kChunksPerPair * 128 * 64; }

// chunk order = MMA consumption order: for l: for nh: for kc.  Each chunk is
// the smem image of B rows n = 128 nh + r (K-major), k = 64 kc + j, swizzled.
void mlp_pack_weights_tc(const float* w0, int d_in, const float* w_hidden, uint16_t* out) {
  // 8 x 8 blocks: 8 rows k (8 contiguous n each) in, transposed, 8 contiguous
  // 16-byte units (8 consecutive k of one row n) out
  size_t ci = 0;
  for (int l = 0; l < kDepth; l++) {
    const int nkc = l == 0 ? 1 : 4;
    for (int nh = 0; nh < 2; nh++)
      for (int kc = 0; kc < nkc; kc++, ci++) {
        uint16_t* img = out + ci * 128 * 64;
        for (int g = 0; g < 8; g++)      // k = 64 kc + 8 g + i
          for (int rb = 0; rb < 16; rb++) {  // r = 8 rb + c
            float blk[8][8];  // [i][c]
            for (int i = 0; i < 8; i++) {
              const int k = 64 * kc + 8 * g + i;
              const int n0 = 128 * nh + 8 * rb;
              if (l == 0) {
                for (int c = 0; c < 8; c++) blk[i][c] = k < d_in ? w0[(size_t)k * kWidth + n0 + c] : 0.f;
              } else {
                const float* row = w_hidden + ((size_t)(l - 1) * kWidth + k) * kWidth + n0;
                for (int c = 0; c < 8; c++) blk[i][c] = row[c];
              }
            }
            for (int c = 0; c < 8; c++) {
              const int r = 8 * rb + c;
              uint16_t* unit = img + ((r >> 3) * 1024 + (r & 7) * 128 + ((g ^ (r & 7)) << 4)) / 2;
              for (int i = 0; i < 8; i++) unit[i] = f2bf(blk[i][c]);
            }
          }
      }
  }
}

// Positional encoding of point p packed to 32 bf16x2 words (features 0..63,
// 39..63 zero); one sincospif per (frequency, coordinate) feeds both the sin
// and the cos feature.  Same values as pe_feature().
__device__ __forceinline__ void pe_row_packed(const PointSrc& src, int64_t n, int64_t p, uint32_t (&pk)[32]) {
  double pt[3] = {0.5, 0.5, 0.5};
  const bool ok = p < n;
  if (ok) point_of(src, p, pt);
  float f[40];
  const float x[3] = {(float)(pt[0] - 0.5), (float)(pt[1] - 0.5), (float)(pt[2] - 0.5)};
#pragma unroll
  for (int c = 0; c < 3; c++) f[c] = x[c];
#pragma unroll
  for (int k = 0; k < 6; k++)
#pragma unroll
    for (int c = 0; c < 3; c++) {
      float sv, cv;
      sincospif(x[c] * (float)(1 << k), &sv, &cv);
      f[3 + 6 * k + c] = sv;
      f[3 + 6 * k + 3 + c] = cv;
    }
  f[39] = 0.f;
#pragma unroll
  for (int c = 0; c < 20; c++) pk[c] = ok ? tc::pack_bf16x2(f[2 * c], f[2 * c + 1]) : 0u;
#pragma unroll
  for (int c = 20; c < 32; c++) pk[c] = 0u;
}
__device__ __forceinline__ void store_pe_row(const uint32_t (&pk)[32], uint32_t a_atom0, int r) {
#pragma unroll
  for (int c = 0; c < 8; c++)
    tc::st_shared_v4(a_atom0 + tc::sw128_off(r, c), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
}

// relu(a + b), relu(c + d) -> bf16x2 in one conversion
__device__ __forceinline__ uint32_t relu_pack(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// 32 accumulator columns -> 16 packed bf16x2 words of relu(acc + bias)
template <bool kBias>
__device__ __forceinline__ void relu_pack32(const uint32_t (&v)[32], const float* __restrict__ sb, uint32_t* out) {
#pragma unroll
  for (int j = 0; j < 16; j++) {
    float a = __uint_as_float(v[2 * j]), b = __uint_as_float(v[2 * j + 1]);
    if (kBias) {
      a += sb[2 * j];
      b += sb[2 * j + 1];
    }
    out[j] = relu_pack(a, b);
  }
}
// The CTA-pair evaluator's head: relu(acc) . w over 32 columns with packed
// FFMA2 (even and odd columns in the two lanes of a 64-bit accumulator;
// the head is ALU-issue-bound on the pair boundary's critical path)
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t pack_f2(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ float2 unpack_f2(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return make_float2(lo, hi);
}
// sw: head weights in kernel-parameter space at a compile-time offset (the
// caller branches on the column half), so no shared-memory load competes
// with the tensor core's operand reads
template <bool kBias>
__device__ __forceinline__ uint64_t head32x2(const uint32_t (&v)[32], const float* __restrict__ sb,
                                             const float* sw, uint64_t acc) {
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    float a = __uint_as_float(v[j]), b = __uint_as_float(v[j + 1]);
    if (kBias) {
      a += sb[j];
      b += sb[j + 1];
    }
    a = a > 0.f ? a : 0.f;
    b = b > 0.f ? b : 0.f;
    acc = ffma2(pack_f2(a, b), pack_f2(sw[j], sw[j + 1]), acc);
  }
  return acc;
}

// grid vertex -> (x, y, z) with the precomputed divisor by S (vids < 2^31)
__device__ __forceinline__ void grid_coords_fast(const PointSrc& src, int64_t p, uint32_t c[3]) {
  const uint32_t S = (uint32_t)src.grid.S;
  const uint32_t v = (uint32_t)(src.begin + p);
  const uint32_t q = __umulhi(v, src.fd_m) >> src.fd_s;
  c[0] = v - q * S;
  c[2] = __umulhi(q, src.fd_m) >> src.fd_s;
  c[1] = q - c[2] * S;
}
// fp64 prior + logistic of one point from its fp32 head dot product
// (paper_2409_13418_b200/fields.py MlpField); p < 0 or p >= n: nothing to do
// fp64 label/raw of point p from its fp32 head dot (the reference's
// expression: sigma(A * mlp - P * (|p - c| - R)), fields.py/MlpField)
__device__ __forceinline__ void label_fp64(const MlpDev& m, const PointSrc& src, int64_t p, int64_t o, float dot,
                                           uint8_t* __restrict__ labels, double* __restrict__ raw) {
  const double mlp = (double)(dot + m.b_head);
  double pt[3];
  point_of(src, p, pt);
  const double d[3] = {pt[0] - m.prior_center[0], pt[1] - m.prior_center[1], pt[2] - m.prior_center[2]};
  const double dist = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
  const double logit = m.amplitude * mlp - m.prior_scale * (dist - m.prior_radius);
  if (!raw) {
    // the label of sigma(logit) > 1/2 without exp and the division: logit
    // <= 0 gives exp(-logit) >= 1, 1 + e >= 2 and sigma <= 1/2; logit >
    // 1e-12 keeps exp(-logit) thousands of ulps below 1, so 1 + e rounds
    // below 2 and sigma > 1/2.  Only the sliver in between (and NaN) takes
    // the full expression.
    if (logit <= 0.0) {
      labels[o] = 0;
      return;
    }
    if (logit > 1e-12) {
      labels[o] = 1;
      return;
    }
  }
  const double rv = 1.0 / (1.0 + exp(-logit));
  labels[o] = rv > 0.5 ? 1 : 0;
  if (raw) raw[o] = rv;
}

// Label (and raw) of point p from its fp32 head dot.  Labels only: the sign
// of the logit in fp32.  Against the fp64 logit (same fp32 dot), each fp32
// step rounds within a few ulps of its operand (parameters rounded to fp32
// included), |error| < 4 * 2^-24 * M with M = |A * mlp| + P * (dist + R +
// |x|_1 + |c|_1), so a margin of 1e-6 * M (about 4x that) decides exactly.  Closer points take the fp64 expression -- inline, or, with
// src.defer_dot (CTA-pair evaluator), deferred: label 2 and the dot are
// written and k_mlp_fixup finishes them after the launch, keeping fp64
// latency out of the epilogue (search points sit near the surface, where
// this case is common).
__device__ __forceinline__ void finish_label(const MlpDev& m, const PointSrc& src, int64_t n, int64_t p, float dot,
                                             uint8_t* __restrict__ labels, double* __restrict__ raw) {
  if (p < 0 || p >= n) return;
  const int64_t o = src.out_map ? (int64_t)src.out_map[p] : p;  // output slot
  if (src.dot_out) src.dot_out[o] = dot;  // parity hook: the fp32 head dot of every point
  if (!raw) {
    float xf[3];
    if (src.pts) {
#pragma unroll
      for (int a = 0; a < 3; a++) xf[a] = (float)src.pts[3 * p + a];
    } else {
      int64_t c[3];
      if (src.fd_m) {
        uint32_t cf[3];
        grid_coords_fast(src, p, cf);
        c[0] = cf[0];
        c[1] = cf[1];
        c[2] = cf[2];
      } else {
        vid_coords(src.grid, src.begin + p, c);
      }
#pragma unroll
      for (int a = 0; a < 3; a++) xf[a] = fmaf((float)c[a], (float)src.grid.h[a], (float)src.grid.lo[a]);
    }
    float d2 = 0.f;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const float x = xf[a] - (float)m.prior_center[a];
      d2 = fmaf(x, x, d2);
    }
    const float am = (float)m.amplitude * (dot + m.b_head), dist = sqrtf(d2);
    const float ps = (float)m.prior_scale, pr = (float)m.prior_radius;
    const float lg = am - ps * (dist - pr);
    const float mag = fabsf(am) + fabsf(ps) * (dist + fabsf(pr) + fabsf(xf[0]) + fabsf(xf[1]) + fabsf(xf[2]) +
                                               fabsf((float)m.prior_center[0]) + fabsf((float)m.prior_center[1]) +
                                               fabsf((float)m.prior_center[2]));
    if ((fabsf(lg) > 1e-6f * mag + 1e-30f && !(m.debug & 4)) || (m.debug & 16)) {  // debug 16 / 4: timing only
      labels[o] = lg > 0.f ? 1 : 0;
      return;
    }
    if (src.defer_dot) {
      labels[o] = 2;
      src.defer_dot[p] = dot;
      return;
    }
  }
  label_fp64(m, src, p, o, dot, labels, raw);
}

// the deferred labels of one launch (finish_label with src.defer_dot)
__global__ void k_mlp_fixup(MlpDev m, PointSrc src, int64_t n_launch, uint8_t* __restrict__ labels) {
  const int64_t n = src.n_dev ? *src.n_dev : n_launch;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t o = src.out_map ? (int64_t)src.out_map[p] : p;
  if (labels[o] == 2) label_fp64(m, src, p, o, src.defer_dot[p], labels, nullptr);
}

// Positional encoding built in pieces across the layers of the current tile
// pair (the epilogue's slack after each layer): piece 0 = the fp64 point and
// frequency 0, piece k = frequency k.  The packed words equal
// pe_row_packed's: word c = (feature 2c, feature 2c + 1), features
// [x(3), sin_k(3), cos_k(3), ...]; frequency k's first feature 3 + 6k is the
// high half of word 1 + 3k, whose low half (``pend``) is the previous one.
struct PePiece {
  float x[3];
  float pend;
  bool ok;
};
// encoding row of grid point p from the per-axis table: the same values as
// pe_row_packed (the table holds exactly its per-coordinate features)
__device__ __forceinline__ void pe_from_table(const PointSrc& src, int64_t n, int64_t p, uint32_t (&pk)[32]) {
#pragma unroll
  for (int c = 20; c < 32; c++) pk[c] = 0u;
  if (p >= n) {
#pragma unroll
    for (int c = 0; c < 20; c++) pk[c] = 0u;
    return;
  }
  uint32_t ci[3];
  grid_coords_fast(src, p, ci);
  float T[3][16];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const float4* row = reinterpret_cast<const float4*>(src.petab + ((size_t)a * src.grid.S + ci[a]) * 16);
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const float4 q = __ldg(row + j);
      T[a][4 * j] = q.x;
      T[a][4 * j + 1] = q.y;
      T[a][4 * j + 2] = q.z;
      T[a][4 * j + 3] = q.w;
    }
  }
  float f[40];
#pragma unroll
  for (int a = 0; a < 3; a++) f[a] = T[a][0];
#pragma unroll
  for (int k = 0; k < 6; k++)
#pragma unroll
    for (int a = 0; a < 3; a++) {
      f[3 + 6 * k + a] = T[a][1 + k];
      f[6 + 6 * k + a] = T[a][7 + k];
    }
  f[39] = 0.f;
#pragma unroll
  for (int c = 0; c < 20; c++) pk[c] = tc::pack_bf16x2(f[2 * c], f[2 * c + 1]);
}

// table rows: [x, sin_0..sin_5, cos_0..cos_5, 0, 0, 0] per (axis, coordinate index)
__global__ void k_pe_table(GridP g, float* __restrict__ tab) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * g.S) return;
  const int a = (int)(i / g.S);
  const int64_t c = i % g.S;
  const float x = (float)(gpos(g, a, c) - 0.5);
  float* row = tab + i * 16;
  row[0] = x;
  for (int k = 0; k < 6; k++) {
    float sv, cv;
    sincospif(x * (float)(1 << k), &sv, &cv);
    row[1 + k] = sv;
    row[7 + k] = cv;
  }
  row[13] = row[14] = row[15] = 0.f;
}

template <int K>
__device__ __forceinline__ void pe_piece_k(const PointSrc& src, int64_t n, int64_t p, PePiece& st,
                                           uint32_t (&pk)[32]) {
  if (K == 0) {
    double pt[3] = {0.5, 0.5, 0.5};
    st.ok = p < n;
    if (st.ok) point_of(src, p, pt);
#pragma unroll
    for (int c = 0; c < 3; c++) st.x[c] = (float)(pt[c] - 0.5);
    pk[0] = tc::pack_bf16x2(st.x[0], st.x[1]);
    st.pend = st.x[2];
  }
  float sv[3], cv[3];
#pragma unroll
  for (int c = 0; c < 3; c++) sincospif(st.x[c] * (float)(1 << K), &sv[c], &cv[c]);
  pk[1 + 3 * K] = tc::pack_bf16x2(st.pend, sv[0]);
  pk[2 + 3 * K] = tc::pack_bf16x2(sv[1], sv[2]);
  pk[3 + 3 * K] = tc::pack_bf16x2(cv[0], cv[1]);
  st.pend = cv[2];
  if (K == 5) {
    pk[19] = tc::pack_bf16x2(st.pend, 0.f);
#pragma unroll
    for (int c = 0; c < 20; c++) pk[c] = st.ok ? pk[c] : 0u;
#pragma unroll
    for (int c = 20; c < 32; c++) pk[c] = 0u;
  }
}
// runtime piece index -> compile-time register indices (no local-memory array)
__device__ __forceinline__ void pe_piece(const PointSrc& src, int64_t n, int64_t p, int k, PePiece& st,
                                         uint32_t (&pk)[32]) {
  switch (k) {
    case 0: pe_piece_k<0>(src, n, p, st, pk); break;
    case 1: pe_piece_k<1>(src, n, p, st, pk); break;
    case 2: pe_piece_k<2>(src, n, p, st, pk); break;
    case 3: pe_piece_k<3>(src, n, p, st, pk); break;
    case 4: pe_piece_k<4>(src, n, p, st, pk); break;
    default: pe_piece_k<5>(src, n, p, st, pk); break;
  }
}

// ===========================================================================
// CTA-pair, N = 256, tile ping-pong evaluator (k_mlp_tc4, the MLP evaluator)
//
// A cluster of two CTAs (one TPC) runs 2 x 256 points through the layers.
// Each CTA holds two 128-row activation tiles in shared memory (A, bf16,
// 128 KB) and its 128-row half of every weight K-atom (B split along N:
// CTA r owns output columns 128r .. 128r+127 -- exactly tc1's chunk
// (l, nh = r, kc), so w_tc is reused).  The leader issues
// tcgen05.mma.cta_group::2 M256 N256 K16 (128 cycles): A from each CTA's own
// tile, B from both CTAs' halves, fp32 D of tile t in TMEM columns 256t ..
// 256t+255 of each CTA (its 128 rows).  Tiles alternate: (t0, l), (t1, l),
// (t0, l+1), ... so tile t's epilogue (TMEM -> bias + ReLU -> bf16 -> A(t))
// runs while the other tile's MMAs run, and a weight stage serves both
// tiles of a layer before it is released.  Per SM and layer: A reads 128 KB,
// B reads 128 KB, weight copies 64 KB, activation stores 128 KB of shared
// memory traffic for 4,096 MMA cycles (tc1: 768 KB), so the tensor pipe,
// not shared memory, sets the pace.
//
// Synchronisation rules that the measurements forced:
// * the MMA issuer waits only on named barriers (an mbarrier poll there
//   stalls the tensor pipe ~180 cycles); helper warps turn mbarrier phases
//   into bar.arrive;
// * no epilogue warp issues a release.cluster arrive (MEMBAR.ALL.GPU +
//   ERRBAR, ~1,000 cycles): CTA-scope arrives, and the peer's warp 1
//   forwards them with one relaxed remote arrive;
// * pairs come from a device counter through a 4-slot ring (dynamic
//   schedule), the leader's copy by st.async + complete_tx;
// * at the pair boundary the epilogue is the critical path: the next pair's
//   encoding goes in before the head, the head's weights are kernel
//   parameters, and labels are finished in the slack of layers 2 and 3
//   (fp32-undecided ones deferred to k_mlp_fixup for search batches).
// ===========================================================================
namespace tc4 {
constexpr int kThreads = 384;
constexpr int kStages = 6;
constexpr int kStageBytes = 16384;   // per CTA: 128 N rows x K 64 (one K-atom)
constexpr int kTileABytes = 65536;   // 128 rows x 256 bf16
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (32u << 17) | (16u << 24);  // M256 N256
constexpr size_t kSmemBytes = 1024 + 2 * kTileABytes + kStages * kStageBytes + 48 * 8 + 384 * 4;
constexpr int kSched = 4;  // pair-index ring depth (dynamic schedule)
constexpr uint32_t kSchedReaders = 23;  // warps that read each slot: 12 in the leader, 11 in the peer
constexpr uint32_t kBarW = 2;              // named barriers 2..7: weight stage s ready
constexpr uint32_t kBarA = kBarW + kStages;  // 8..9: A(t) ready
constexpr uint32_t kBarX = kBarA + 2;        // 10: the label exchange's s_part was read
static_assert(kBarX + 1 <= 16, "named barriers");
__device__ __forceinline__ void umma_ss2(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}
}  // namespace tc4

template <bool kBias>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc4::kThreads, 1)
    k_mlp_tc4(MlpDev m, PointSrc src, int64_t n_launch, uint8_t* __restrict__ labels, double* __restrict__ raw) {
  using namespace tc;
  using tc2::cluster_ctarank;
  using tc2::cluster_sync;
  using tc2::mapa;
  using tc2::mbar_arrive_cluster;
  using tc2::mbar_arrive_cluster_relaxed;
  using tc2::named_bar_arrive;
  using tc2::named_bar_sync;
  using tc2::umma_commit_pair;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* A0 = smem;
  uint8_t* Wst = smem + 2 * tc4::kTileABytes;
  uint64_t* bars = (uint64_t*)(Wst + tc4::kStages * tc4::kStageBytes);
  uint64_t* full = bars;                       // [S] local weight half landed
  uint64_t* empty = full + tc4::kStages;       // [S] both tiles done with the stage (commit, both CTAs)
  uint64_t* fullp = empty + tc4::kStages;      // [S] leader: the peer's half landed (relay)
  uint64_t* acc_full = fullp + tc4::kStages;   // [2] tile t's layer done (commit, both CTAs)
  uint64_t* a_ready = acc_full + 2;            // [2] leader: A(t) written and D(t) drained, 8 warps
  uint32_t* tmem_slot = (uint32_t*)(a_ready + 2);
  uint64_t* sched_full = bars + 24;            // [4] pair index of slot s written (scheduler, both CTAs)
  uint64_t* sched_empty = bars + 28;           // [4] peer: all 22 reader warps took slot s
  int64_t* sched_pr = (int64_t*)(bars + 32);   // [4] ring of pair indices (>= npairs: no more work)
  uint64_t* a_loc = bars + 36;                 // [2] peer: its 8 epilogue warps released A(t)
  float* s_part = (float*)(bars + 48) + kWidth;  // (128) head partials of columns 128..255 (the head's
                                                 // weights are kernel parameters, m.w_head_k)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int64_t n = src.n_dev ? *src.n_dev : n_launch;  // compacted batch: count from the producer kernel
  const int64_t npairs = (n + 511) / 512;

  if (m.trace && threadIdx.x == 0 && blockIdx.x < 300) m.trace[400 + 2 * blockIdx.x] = globaltimer_ns();
  if (threadIdx.x == 0) {
    for (int s = 0; s < tc4::kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&fullp[s], 1);
    }
    for (int t = 0; t < 2; t++) {
      mbar_init(&acc_full[t], 1);
      mbar_init(&a_ready[t], 9);  // leader: its 8 epilogue warps + the peer's relay
      mbar_init(&a_loc[t], 8);
    }
    for (int i = 0; i < tc4::kSched; i++) {
      mbar_init(&sched_full[i], 1);
      mbar_init(&sched_empty[i], tc4::kSchedReaders);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Dynamic schedule: the peer's warp 2 takes pair indices from a global
  // counter (m.sched, minus this launch's base) into a 4-slot ring in both
  // CTAs; every role walks the ring, so clusters that run faster take more
  // pairs and all clusters finish within about one pair of each other
  // (static round-robin left a ~4 % spread of cluster end times).
  // Whole-warp call; slot i's reader count is tc4::kSchedReaders.
  auto sched_get = [&](uint32_t i) -> int64_t {
    const uint32_t sl = i % tc4::kSched, ph = (i / tc4::kSched) & 1;
    mbar_wait(&sched_full[sl], ph);  // leader: the slot came by st.async (async proxy, complete_tx)
    const int64_t pr = *(volatile int64_t*)&sched_pr[sl];
    __syncwarp();
    if (lane == 0) {
      if (crank == 1) {
        mbar_arrive(&sched_empty[sl]);
      } else {
        // relaxed: a release.cluster arrive would first drain this thread's
        // outstanding stores (~1,000 cycles); the slot's value is already in
        // a register and the scheduler refills it only kSched pairs later
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                         mapa(smem_u32(&sched_empty[sl]), 1))
                     : "memory");
      }
    }
    return pr;
  };

  if (warp == 0) {  // ---- weight producer: this CTA's N half of every K-atom
    uint32_t g = 0;
    for (uint32_t i = 0; sched_get(i) < npairs; i++)
      for (int l = 0; l < kDepth; l++)
        for (int kc = 0; kc < (l == 0 ? 1 : 4); kc++, g++) {
          const uint32_t s = g % tc4::kStages, ph = (g / tc4::kStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (elect_one()) {
            if ((m.debug & 1) && g >= (uint32_t)tc4::kStages) {
              mbar_arrive(&full[s]);  // experiment (odc_profile_mlp only): stale weights, no L2 traffic
            } else {
              const int ci = l == 0 ? (int)crank : 2 + (l - 1) * 8 + (int)crank * 4 + kc;
              mbar_expect_tx(&full[s], tc4::kStageBytes);
              bulk_g2s(Wst + s * tc4::kStageBytes, m.w_tc + (size_t)ci * 128 * 64, tc4::kStageBytes, &full[s]);
            }
          }
          __syncwarp();
        }
  } else if (warp == 3) {
    // peer: its half landed -> the leader's fullp[s].  leader: both halves
    // landed -> named barrier kBarW + s for the MMA warp (a bar.sync is cheap
    // for the issuer; an mbarrier poll costs it ~180 cycles of tensor-pipe
    // bubble with shared memory saturated by operand reads)
    uint32_t g = 0;
    for (uint32_t i = 0; sched_get(i) < npairs; i++)
      for (int l = 0; l < kDepth; l++)
        for (int kc = 0; kc < (l == 0 ? 1 : 4); kc++, g++) {
          const uint32_t s = g % tc4::kStages, ph = (g / tc4::kStages) & 1;
          mbar_wait(&full[s], ph);
          if (leader) {
            mbar_wait(&fullp[s], ph);
            named_bar_arrive(tc4::kBarW + s, 64);
          } else {
            if (elect_one()) mbar_arrive_cluster_relaxed(mapa(smem_u32(&fullp[s]), 0));
            __syncwarp();
          }
        }
  } else if (warp == 2) {
    if (leader) {  // ---- relay: a_ready[t] -> named barrier kBarA + t for the MMA warp
      uint32_t ra[2] = {0, 0};
      for (uint32_t i = 0; sched_get(i) < npairs; i++)
        for (int l = 0; l < kDepth; l++)
          for (int t = 0; t < 2; t++) {
            mbar_wait(&a_ready[t], ra[t] & 1);
            if (m.trace && blockIdx.x == 0 && lane == 0 && ra[t] < 24) m.trace[750 + 24 * t + ra[t]] = globaltimer_ns();
            ra[t]++;
            named_bar_arrive(tc4::kBarA + t, 64);
          }
    } else if (lane == 0) {  // ---- scheduler: pair indices into both CTAs' rings
      const uint32_t peer_pr = mapa(smem_u32(sched_pr), 0);
      const uint32_t peer_full = mapa(smem_u32(sched_full), 0);
      for (uint32_t i = 0;; i++) {
        const uint32_t sl = i % tc4::kSched, ph = (i / tc4::kSched) & 1;
        mbar_wait(&sched_empty[sl], ph ^ 1);
        int64_t pr = (int64_t)(atomicAdd(m.sched, 1ull) - m.sched_base);
        if (m.debug & 8) {  // experiment (odc_profile_mlp only): static round-robin order
          const int64_t st = (int64_t)(blockIdx.x >> 1) + (int64_t)i * (int64_t)(gridDim.x >> 1);
          pr = st < npairs ? st : npairs;
        }
        *(volatile int64_t*)&sched_pr[sl] = pr;
        mbar_arrive(&sched_full[sl]);
        // the leader's copy: an async-proxy store that completes the leader's
        // barrier transaction (like a bulk copy), so its readers need no
        // cluster-scope acquire (that wait cost ~1,300 cycles per pair)
        asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], 8;" ::"r"(
                         peer_full + 8 * sl)
                     : "memory");
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(peer_pr + 8 * sl),
                     "l"(pr), "r"(peer_full + 8 * sl)
                     : "memory");
        if (pr >= npairs) break;
      }
    }
  } else if (warp == 1 && !leader) {
    // ---- peer relay: its 8 epilogue warps released A(t) (CTA-scope arrives,
    // after fence.proxy.async) -> one relaxed remote arrive on the leader's
    // a_ready[t] (see mbar_arrive_cluster_relaxed: a release.cluster arrive
    // costs ~600 ns of MEMBAR.GPU on this path)
    const uint32_t leader_ready[2] = {mapa(smem_u32(&a_ready[0]), 0), mapa(smem_u32(&a_ready[1]), 0)};
    uint32_t ra[2] = {0, 0};
    auto forward = [&](int t) {
      mbar_wait(&a_loc[t], ra[t] & 1);
      if (m.trace && blockIdx.x == 1 && lane == 0 && ra[t] < 24) m.trace[700 + 24 * t + ra[t]] = globaltimer_ns();
      ra[t]++;
      if (elect_one()) mbar_arrive_cluster_relaxed(leader_ready[t]);
      __syncwarp();
    };
    int64_t pr = sched_get(0);
    if (pr < npairs) {
      forward(0);
      forward(1);
    }
    for (uint32_t i = 0; pr < npairs; i++) {
      const int64_t next = sched_get(i + 1);
      for (int l = 0; l < kDepth; l++) {
        forward(0);
        forward(1);
      }
      pr = next;
    }
  } else if (warp == 1) {
    {  // ---- MMA issuer (leader; whole warp walks, one elected lane issues)
      const uint32_t a_lo = desc_lo(smem_u32(A0));
      const uint32_t w_lo = desc_lo(smem_u32(Wst));
      // one tile's layer: NST K-atoms of NKS K-steps each, fully unrolled so
      // that each MMA is two immediate adds on the descriptor words (the
      // issue rate is what keeps the tensor pipe fed between tiles)
      auto tile = [&](auto tc, auto nstc, auto nksc, int ti, int l, uint32_t s0) {
        constexpr int t = decltype(tc)::value, NST = decltype(nstc)::value, NKS = decltype(nksc)::value;
        if (lane == 0) ODC_TRACE(ti, l, 2 * t);
        named_bar_sync(tc4::kBarA + t, 64);  // a_ready[t] (relayed by warp 2)
        tc_fence_after();
        if (lane == 0) ODC_TRACE(ti, l, 2 * t + 1);
        const uint32_t a_t = a_lo + (uint32_t)((t * tc4::kTileABytes) >> 4);
        uint32_t s = s0;
#pragma unroll
        for (int k = 0; k < NST; k++) {
          if (t == 0) {  // both weight halves of stage s landed (relayed by warp 3)
            const long long w0 = m.trace ? clock64() : 0;
            named_bar_sync(tc4::kBarW + s, 64);
            if (m.trace && lane == 0 && blockIdx.x == 0 && ti < 2)
              m.trace[256 + (ti * 8 + l) * 4 + k] = (unsigned long long)(clock64() - w0);
          }
          const uint32_t b_lo = w_lo + s * (tc4::kStageBytes >> 4);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < NKS; ks++)
              tc4::umma_ss2(tmem + t * 256, make_desc(a_t + (uint32_t)((k * 16384) >> 4) + ks * 2),
                            make_desc(b_lo + ks * 2), (k | ks) != 0);
            if (t == 1) umma_commit_pair(&empty[s]);
          }
          __syncwarp();
          s = s + 1 == (uint32_t)tc4::kStages ? 0 : s + 1;
        }
        if (elect_one()) umma_commit_pair(&acc_full[t]);
        __syncwarp();
        if (lane == 0) ODC_TRACE(ti, l, 4 + t);
      };
      using I0 = std::integral_constant<int, 0>;
      using I1 = std::integral_constant<int, 1>;
      uint32_t s0 = 0;
      for (int ti = 0; sched_get((uint32_t)ti) < npairs; ti++) {
        // layer 0: one K-atom; the encoding has 39 features, so K-step 3
        // (features 48..63, all zero) is skipped -- the sum is unchanged
        tile(I0{}, I1{}, std::integral_constant<int, 3>{}, ti, 0, s0);
        tile(I1{}, I1{}, std::integral_constant<int, 3>{}, ti, 0, s0);
        s0 = s0 + 1 == (uint32_t)tc4::kStages ? 0 : s0 + 1;
        for (int l = 1; l < kDepth; l++) {
          tile(I0{}, std::integral_constant<int, 4>{}, std::integral_constant<int, 4>{}, ti, l, s0);
          tile(I1{}, std::integral_constant<int, 4>{}, std::integral_constant<int, 4>{}, ti, l, s0);
          s0 = (s0 + 4) % tc4::kStages;
        }
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue: all 8 warps work on one tile at a time (tiles alternate),
    // warp%4 = TMEM lane quarter, (warp-4)/4 = column half of the 256 outputs
    const int q = warp & 3;
    const int hc = (warp - 4) >> 2;
    const int r = 32 * q + lane;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    int nrel = 0;
    auto release = [&](int t) {  // A(t) written / D(t) drained -> the leader's a_ready[t]
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      // CTA-scope releases only: the leader's MMA warp acquires a_ready[t]
      // directly; the peer's a_loc[t] is forwarded at cluster scope by its
      // warp 1 (release -> acquire -> release.cluster -> acquire.cluster)
      if (lane == 0) mbar_arrive(leader ? &a_ready[t] : &a_loc[t]);
      if (m.trace && blockIdx.x < 2 && lane == 0 && t == 0 && nrel < 24)
        m.trace[800 + blockIdx.x * 200 + (warp - 4) * 24 + nrel] = globaltimer_ns();
      if (t == 0) nrel++;
    };
    // this warp's encoding row: tile hc, row r (column half 0 stores tile 0, half 1 tile 1)
    const uint32_t a_pe = smem_u32(A0 + hc * tc4::kTileABytes);
    uint32_t af[2] = {0, 0};
    uint32_t pe[32];
    PePiece pes;
    // The previous pair's labels are finished in the slack of layers 2 (tile
    // 0) and 3 (tile 1) of the next pair: the column halves' head partials
    // meet in s_part there, away from the pair boundary where the epilogue is
    // the critical path.  dot = partial(cols 0..127) + partial(cols 128..255).
    int64_t p_prev = -1;
    float part_prev[2] = {0.f, 0.f};
    // tile t's labels are finished by column half t (the other half hands its
    // partial over), so each warp finishes one label per pair.  The second
    // barrier only waits for the finisher's read of s_part (bar.arrive), not
    // for its label.  fp32 addition commutes: dot = d0 + d1 either way.
    auto finish_tile = [&](int t) {
      if (hc != t) s_part[r] = part_prev[t];
      named_bar_sync(1, 256);
      float dot = 0.f;
      if (hc == t) {
        dot = t == 0 ? part_prev[0] + s_part[r] : s_part[r] + part_prev[1];
        named_bar_arrive(tc4::kBarX, 256);  // s_part read
        finish_label(m, src, n, p_prev + 256 * t, dot, labels, raw);
      } else {
        named_bar_sync(tc4::kBarX, 256);  // s_part reusable
      }
    };
    const bool tr = r == 0 && crank == 0 && hc == 0;
    int64_t pr = sched_get(0);
    if (pr < npairs) {
      if (src.petab) pe_from_table(src, n, pr * 512 + hc * 256 + crank * 128 + r, pe);
      else pe_row_packed(src, n, pr * 512 + hc * 256 + crank * 128 + r, pe);
      store_pe_row(pe, a_pe, r);
      release(0);
      release(1);
    }
    for (int ti = 0; pr < npairs; ti++) {
      int64_t next = npairs;  // the following pair: taken from the ring in layer 1's slack
      float part[2] = {0.f, 0.f};
      for (int l = 0; l < kDepth; l++) {
        const float* bl = m.bias + l * kWidth + hc * 128;
#pragma unroll
        for (int t = 0; t < 2; t++) {
          const uint32_t a_t = smem_u32(A0 + t * tc4::kTileABytes);
          const uint32_t dcol = tmem + lane_base + t * 256 + hc * 128;
          if (tr) ODC_TRACE(ti, l, 6 + t);
          mbar_wait(&acc_full[t], af[t] & 1);
          af[t]++;
          tc_fence_after();
          if (tr) ODC_TRACE(ti, l, 8 + t);
          if (l < kDepth - 1) {
#pragma unroll
            for (int gk = 0; gk < 2; gk++) {  // 64 columns = one K-atom of the next layer's A
              uint32_t v0[32], v1[32], w[32];
              ODC_TMEM_LD32(dcol + 64 * gk, v0);
              ODC_TMEM_LD32(dcol + 64 * gk + 32, v1);
              tmem_ld_wait();
              relu_pack32<kBias>(v0, bl + 64 * gk, w);
              relu_pack32<kBias>(v1, bl + 64 * gk + 32, w + 16);
              const uint32_t atom = a_t + (2 * hc + gk) * 16384;
#pragma unroll
              for (int c = 0; c < 8; c++)
                st_shared_v4(atom + sw128_off(r, c), w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
            }
            release(t);
            if (tr) ODC_TRACE(ti, l, 10 + t);
            // slack until the next layer's tile 0
            if (t == 1) {
              if (l == 1) {
                const long long sg0 = m.trace ? clock64() : 0;
                next = sched_get((uint32_t)ti + 1);
                if (m.trace && tr && ti < 8) m.trace[320 + ti] = (unsigned long long)(clock64() - sg0);
              }
              if (l == 2 && p_prev >= 0) finish_tile(0);
              if (l == 3 && p_prev >= 0) finish_tile(1);
              if (l >= 1 && next < npairs) {  // one piece of the next pair's encoding
                const int64_t pn = next * 512 + hc * 256 + crank * 128 + r;
                if (src.petab) {  // grid points: table lookups, in one layer's slack
                  if (l == kDepth - 2) pe_from_table(src, n, pn, pe);
                } else {  // explicit points: one frequency per layer
                  pe_piece(src, n, pn, l - 1, pes, pe);
                }
              }
              if (tr) ODC_TRACE(ti, l, 14);
            }
          } else {
            // layer 7 consumed A(t): the next pair's encoding of tile t goes in
            // first (half t's rows), then the head drains D(t)
            if (next < npairs && hc == t) store_pe_row(pe, a_pe, r);
            auto head = [&](auto hcc) {
              constexpr int H = decltype(hcc)::value;
              uint64_t acc = 0;  // (+0.f, +0.f)
#pragma unroll
              for (int gk = 0; gk < 4; gk += 2) {
                uint32_t v0[32], v1[32];
                ODC_TMEM_LD32(dcol + 32 * gk, v0);
                ODC_TMEM_LD32(dcol + 32 * gk + 32, v1);
                tmem_ld_wait();
                acc = head32x2<kBias>(v0, bl + 32 * gk, m.w_head_k + H * 128 + 32 * gk, acc);
                acc = head32x2<kBias>(v1, bl + 32 * gk + 32, m.w_head_k + H * 128 + 32 * gk + 32, acc);
              }
              const float2 e = unpack_f2(acc);
              return e.x + e.y;
            };
            part[t] = hc == 0 ? head(std::integral_constant<int, 0>{}) : head(std::integral_constant<int, 1>{});
            if (tr) ODC_TRACE(ti, l, 12 + t);
            release(t);
            if (tr) ODC_TRACE(ti, l, 10 + t);
          }
        }
      }
      p_prev = pr * 512 + crank * 128 + r;  // tile 0 row; tile 1 row = +256
      part_prev[0] = part[0];
      part_prev[1] = part[1];
      pr = next;
    }
    if (p_prev >= 0) {
      finish_tile(0);
      finish_tile(1);
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (m.trace && threadIdx.x == 0 && blockIdx.x < 300) m.trace[401 + 2 * blockIdx.x] = globaltimer_ns();
}

int mlp_eval(const MlpDev& m_in, const PointSrc& src, int64_t n, uint8_t* labels, double* raw, cudaStream_t s,
             unsigned long long* sched_next) {
  MlpDev m = m_in;
  if (n <= 0) return 0;
  // kernel attributes and the SM count, once per device (thread-safe: the
  // batch mode drives one context per host thread)
  static std::once_flag once[64];
  static int num_sms[64];
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  std::call_once(once[dev], [dev]() {
    cudaFuncSetAttribute(k_mlp_tc4<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc4::kSmemBytes);
    cudaFuncSetAttribute(k_mlp_tc4<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc4::kSmemBytes);
    cudaDeviceGetAttribute(&num_sms[dev], cudaDevAttrMultiProcessorCount, dev);
  });
  const int g_num_sms = num_sms[dev];
  const int64_t np4 = (n + 511) / 512;
  const int64_t pairs = (g_num_sms / 2) < np4 ? (g_num_sms / 2) : np4;
  if (!m.sched || !sched_next || !m.w_tc) return -1;  // the dynamic schedule needs the context's counter
  // every cluster takes indices until one is >= np4: np4 + clusters fetches
  m.sched_base = *sched_next;
  *sched_next += (unsigned long long)(np4 + pairs);
  PointSrc sp = src;
  sp.petab = nullptr;
  sp.fd_m = sp.fd_s = 0;
  float* tab = nullptr;
  if (!src.pts && src.begin + n <= INT32_MAX && src.grid.S >= 2) {
    // grid points: per-axis encoding table + divisor by S (CUTLASS-style
    // round-up multiplier, exact for dividends < 2^31)
    uint32_t l2 = 0;
    while ((1u << l2) < (uint32_t)src.grid.S) l2++;
    const uint32_t pw = 31 + l2;
    sp.fd_m = (uint32_t)(((1ull << pw) + (uint64_t)src.grid.S - 1) / (uint64_t)src.grid.S);
    sp.fd_s = pw - 32;
    if (cudaMallocAsync((void**)&tab, sizeof(float) * 16 * 3 * src.grid.S, s) == cudaSuccess) {
      k_pe_table<<<(unsigned)((3 * src.grid.S + 127) / 128), 128, 0, s>>>(src.grid, tab);
      sp.petab = tab;
    } else {
      cudaGetLastError();
    }
  }
  // labels of explicit (search) points: undecided fp32 labels are finished
  // by k_mlp_fixup after the launch (stream-ordered scratch for their
  // dots).  Grid points rarely sit within the margin of the surface, so
  // the grid pass keeps the inline fp64 path and needs no scratch.
  float* defer = nullptr;
  if (!raw && src.pts && !src.dot_out) {
    if (cudaMallocAsync((void**)&defer, sizeof(float) * n, s) == cudaSuccess) sp.defer_dot = defer;
    else cudaGetLastError();
  }
  if (m.has_bias)
    k_mlp_tc4<true><<<(unsigned)(2 * pairs), tc4::kThreads, tc4::kSmemBytes, s>>>(m, sp, n, labels, raw);
  else
    k_mlp_tc4<false><<<(unsigned)(2 * pairs), tc4::kThreads, tc4::kSmemBytes, s>>>(m, sp, n, labels, raw);
  if (defer) {
    k_mlp_fixup<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(m, sp, n, labels);
    cudaFreeAsync(defer, s);
  }
  if (tab) cudaFreeAsync(tab, s);
  return 1 + (defer ? 1 : 0) + (tab ? 1 : 0);  // kernels launched
}

const char* mlp_kernel_name() { return "k_mlp_tc4"; }

int mlp_set_wait_timeout_ns(unsigned long long ns) {
  return cudaMemcpyToSymbol(tc::g_mbar_timeout_ns, &ns, sizeof ns) == cudaSuccess ? 0 : -1;
}

}  // namespace odc
