// odc_kernels.cu -- sm_100a kernels of the ODC extraction path (fp64 part).
//
// Compiled with --fmad=false: every fp64 expression keeps numpy's rounding
// (one rounding per ufunc); see odc_device.cuh.
//
// Data layout in HBM (per extraction):
//   L       bit-packed vertex labels, rows (y,z) of W words         S^2 W x 4 B
//   occ     per 32 words: active-word bitmap + active words before    S^2 W / 4 B
//   rec     WordRec per ACTIVE word: edge/face/4-face/centre/cell
//           bitmaps + exclusive ranks (edges, instances, cells)     A x 64 B
//   lists   edge keys (K), instance keys (Q), cell ids (C) as int64, in
//           the reference's ascending key order
//   stage   t/pos1d (K), pos2/pos3/status (Q), vertices (P + fans), ...
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "odc_kernels.h"
#include "odc_eigh3.cuh"
#include "odc_scan.cuh"

namespace odc {

namespace {
inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }
// Statistics counters: one atomic per warp (the sum over the active lanes)
// instead of one per thread -- a million same-address atomics serialise in
// L2 (k_s2_finish spent 0.7 ms on them).  Call with the warp converged.
// PEER: lanes are grouped by target address (a batch warp can straddle two
// shapes, whose counters differ).
template <bool PEER = false>
__device__ __forceinline__ void warp_count(unsigned long long* p, unsigned v) {
  const unsigned m = __activemask();
  const unsigned peers = PEER ? __match_any_sync(m, (unsigned long long)p) : m;
  const unsigned s = __reduce_add_sync(peers, v);
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1 && s) atomicAdd(p, (unsigned long long)s);
}
// bins[b] += 1 for this lane's bin b (0..3) when on
template <bool PEER = false>
__device__ __forceinline__ void warp_count4(unsigned long long* bins, int b, bool on) {
#pragma unroll
  for (int v = 0; v < 4; v++) warp_count<PEER>(&bins[v], on && b == v ? 1u : 0u);
}
// max over the active lanes of non-negative doubles (ordered as bits)
template <bool PEER = false>
__device__ __forceinline__ void warp_max_nonneg_double(unsigned long long* p, double v) {
  const unsigned m = PEER ? __match_any_sync(__activemask(), (unsigned long long)p) : __activemask();
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const unsigned hi = (unsigned)(bits >> 32);
  const unsigned top = __reduce_max_sync(m, hi);
  const unsigned m2 = __ballot_sync(m, hi == top);
  if (hi == top) {
    const unsigned lo = __reduce_max_sync(m2, (unsigned)bits);
    if ((int)(threadIdx.x & 31) == __ffs(m2) - 1 && (top | lo)) atomicMax(p, ((unsigned long long)top << 32) | lo);
  }
}
// bits of word wx that lie below coordinate `limit` (valid x of the row)
__device__ __forceinline__ uint32_t bits_below(int64_t limit, int64_t wx) {
  int64_t n = limit - wx * 32;
  if (n <= 0) return 0u;
  if (n >= 32) return 0xffffffffu;
  return 0xffffffffu >> (32 - n);
}
}  // namespace

// ===========================================================================
// K1: grid labels (grid.py:109-126).  One thread per (row, x) bit, ballot
// packs 32 consecutive x into one word.  label = raw > iso (fields.py:47).
// ===========================================================================
// Grid: blockIdx.x = label row (z, y) of the window, blockIdx.y = 256-bit
// chunk of the row -- the row's coordinates are block-uniform, so no
// per-thread division.
// Label words decided in bulk: each lane bounds the field over the ball
// around its word's (up to) 32 vertices (field_label_ball); the warp then
// evaluates every vertex of each undecided word, 32 lanes per word.  Far
// from the surface one evaluation decides 32 labels.
template <bool B, int EV>
__global__ void __launch_bounds__(256, 4) k_labels_analytic(GridP g, FieldP f, uint32_t* __restrict__ L) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int dec = 2;  // nothing to do
  int64_t y = 0, z = 0, wx = 0;
  if (w < g.NW) {
    word_coords(g, w, y, z, wx);
    GridP gl = g;
    const int b = localize<B>(gl, z);
    const int64_t xa = wx * 32, xb = (xa + 31 < g.S - 1) ? xa + 31 : g.S - 1;
    const double pa = gpos(gl, 0, xa), pb = gpos(gl, 0, xb);
    const double pc[3] = {__dmul_rn(__dadd_rn(pa, pb), 0.5), gpos(gl, 1, y), gpos(gl, 2, z)};
    const double rad = __dmul_rn(__dsub_rn(pb, pa), 0.5) * (1.0 + 1e-12) + 1e-300;
    if constexpr (B) dec = field_label_ball(f.batch[b], pc, rad);
    else if constexpr (EV == EV_BOX2F) dec = field_label_ball_box2f(f, pc, rad);
    else dec = field_label_ball(f, pc, rad);
    if (dec >= 0) L[w] = dec ? bits_below(g.S, wx) : 0u;
  }
  unsigned und = __ballot_sync(0xffffffffu, dec == -1);
  while (und) {
    const int j = __ffs(und) - 1;
    und &= und - 1;
    const int64_t wj = __shfl_sync(0xffffffffu, w, j), yj = __shfl_sync(0xffffffffu, y, j),
                  zj = __shfl_sync(0xffffffffu, z, j), wxj = __shfl_sync(0xffffffffu, wx, j);
    const int64_t x = wxj * 32 + lane;
    uint32_t lab = 0;
    if (x < g.S) {
      GridP gl = g;
      const int b = localize<B>(gl, zj);
      const double p[3] = {gpos(gl, 0, x), gpos(gl, 1, yj), gpos(gl, 2, zj)};
      if constexpr (B) {  // the shape's specialised evaluation (warp-uniform: one word)
        const FieldP& fb = f.batch[b];
        switch (fb.ev) {
          case EV_SPHERE: lab = field_label_t<EV_SPHERE>(fb, p); break;
          case EV_BOX: lab = field_label_t<EV_BOX>(fb, p); break;
          case EV_TORUS: lab = field_label_t<EV_TORUS>(fb, p); break;
          default: lab = field_label_t<EV_SEL>(fb, p); break;
        }
      } else {
        lab = field_label_t<EV>(f, p);
      }
    }
    const uint32_t word = __ballot_sync(0xffffffffu, lab);
    if (lane == 0) L[wj] = word;
  }
}

void launch_labels_analytic(const GridP& g, const FieldP& f, uint32_t* L, cudaStream_t s) {
  if (!g.NW) return;
  const unsigned grid = grid_for(g.NW, 256);
  if (g.nb) {
    k_labels_analytic<true, EV_SEL><<<grid, 256, 0, s>>>(g, f, L);
    return;
  }
  switch (ev_mode_of(f)) {  // the per-vertex evaluations of undecided words, specialised
    case EV_SPHERE: k_labels_analytic<false, EV_SPHERE><<<grid, 256, 0, s>>>(g, f, L); break;
    case EV_BOX: k_labels_analytic<false, EV_BOX><<<grid, 256, 0, s>>>(g, f, L); break;
    case EV_TORUS: k_labels_analytic<false, EV_TORUS><<<grid, 256, 0, s>>>(g, f, L); break;
    case EV_SPHERE2: k_labels_analytic<false, EV_SPHERE2><<<grid, 256, 0, s>>>(g, f, L); break;
    case EV_BOX2F: k_labels_analytic<false, EV_BOX2F><<<grid, 256, 0, s>>>(g, f, L); break;
    default: k_labels_analytic<false, EV_PARAM><<<grid, 256, 0, s>>>(g, f, L); break;
  }
}

// one warp per label row: lane j of word w reads byte 32 w + j (coalesced),
// a ballot makes the word -- no per-element 64-bit division
__global__ void __launch_bounds__(256) k_pack_labels(GridP g, const uint8_t* __restrict__ bytes,
                                                     uint32_t* __restrict__ L) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= g.nz * g.S) return;
  const int lane = threadIdx.x & 31;
  const uint8_t* src = bytes + row * g.S;
  uint32_t* dst = L + row * g.W;
  const int S = (int)g.S;
  for (int w = 0; w < (int)g.W; w++) {
    const int x = 32 * w + lane;
    const uint32_t lab = x < S ? (uint32_t)(src[x] != 0) : 0u;
    const uint32_t bits = __ballot_sync(0xffffffffu, lab);
    if (lane == 0) dst[w] = bits;
  }
}
void launch_pack_labels(const GridP& g, const uint8_t* bytes, uint32_t* L, cudaStream_t s) {
  const int64_t rows = g.nz * g.S;
  if (rows) k_pack_labels<<<grid_for(rows, 8), 256, 0, s>>>(g, bytes, L);
}

__global__ void k_unpack_labels(GridP g, const uint32_t* __restrict__ L, uint8_t* __restrict__ bytes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.nz * g.S2) return;
  bytes[i] = (uint8_t)label_at(L, g, g.z0 * g.S2 + i);
}
void launch_unpack_labels(const GridP& g, const uint32_t* L, uint8_t* bytes, cudaStream_t s) {
  k_unpack_labels<<<grid_for(g.nz * g.S2, 256), 256, 0, s>>>(g, L, bytes);
}

__global__ void k_grid_points(GridP g, int64_t begin, int64_t n, double* __restrict__ pts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3];
  vposition(g, begin + i, p);
  pts[3 * i] = p[0];
  pts[3 * i + 1] = p[1];
  pts[3 * i + 2] = p[2];
}
void launch_grid_points(const GridP& g, int64_t begin, int64_t n, double* pts, cudaStream_t s) {
  k_grid_points<<<grid_for(n, 256), 256, 0, s>>>(g, begin, n, pts);
}

// ===========================================================================
// K2: active sets (grid.py:171-296) from four neighbouring label rows.
//   edge (v,a) crosses  <=> L(v) != L(v + step_a)          (grid.py:185-195)
//   face (v,n) crosses  <=> >= 2 of its 4 cyclic edges cross (grid.py:212-260)
//   cell crosses        <=> its corner labels are not all equal (grid.py:263-278)
// Channels of the rank scan: 0 edges, 1 instances (faces + 4-faces),
// 2 cells, 3 faces, 4 4-crossing faces.
// ===========================================================================
constexpr int kActiveBlock = kScanBlock;
constexpr int kActiveCh = 6;
// A tile (one block, one tile-sum per channel) is kActiveGroups occupancy
// groups of 32 words: pass 1 walks it word by word (kActiveSub sub-tiles of
// kActiveBlock words), pass 2 group by group (a warp per group).
constexpr int kActiveGroups = 64;
constexpr int64_t kActiveTile = (int64_t)kActiveGroups * 32;
constexpr int kActiveSub = (int)(kActiveTile / kActiveBlock);
constexpr int64_t kActiveWarpGroups = 65536;  // pass 2: warp per group below this many groups


struct ActiveBits {
  uint32_t e[3], f[3], f4[3], cell;
};

__device__ __forceinline__ ActiveBits compute_active(const GridP& g, const uint32_t* __restrict__ L, int64_t y,
                                                     int64_t z, int64_t wx) {
  const int64_t W = g.W, S = g.S, R = g.R;
  const int64_t ztop = g.z0 + g.nz - 1;  // last layer held
  const int64_t zl = g.nb ? z - idiv(z, S) * S : z;  // layer within its shape (batch)
  const bool yin = y < R, zin = zl < R && z < ztop;
  auto ld = [&](int64_t yy, int64_t zz, int64_t ww) -> uint32_t {
    if (yy > R || zz > ztop || ww >= W) return 0u;
    return L[((zz - g.z0) * S + yy) * W + ww];
  };
  const uint32_t a00 = ld(y, z, wx), a10 = ld(y + 1, z, wx), a01 = ld(y, z + 1, wx), a11 = ld(y + 1, z + 1, wx);
  const uint32_t n00 = ld(y, z, wx + 1), n10 = ld(y + 1, z, wx + 1), n01 = ld(y, z + 1, wx + 1),
                 n11 = ld(y + 1, z + 1, wx + 1);
  ActiveBits b;
  {  // uniform neighbourhood (all 0 or all 1 labels): nothing crosses
    const uint32_t o = a00 | a10 | a01 | a11 | n00 | n10 | n01 | n11;
    const uint32_t n = a00 & a10 & a01 & a11 & n00 & n10 & n01 & n11;
    if (o == 0u || n == 0xffffffffu) {
#pragma unroll
      for (int a = 0; a < 3; a++) b.e[a] = b.f[a] = b.f4[a] = 0u;
      b.cell = 0u;
      return b;
    }
  }
  // label at x+1
  const uint32_t s00 = (a00 >> 1) | (n00 << 31), s10 = (a10 >> 1) | (n10 << 31);
  const uint32_t s01 = (a01 >> 1) | (n01 << 31), s11 = (a11 >> 1) | (n11 << 31);
  const uint32_t mS = bits_below(S, wx), mR = bits_below(R, wx);
  b.e[0] = (a00 ^ s00) & mR;
  b.e[1] = yin ? ((a00 ^ a10) & mS) : 0u;
  b.e[2] = zin ? ((a00 ^ a01) & mS) : 0u;
  // x-normal face at v: edges EY(v), EZ(v+Sy), EY(v+Sz), EZ(v)
  {
    uint32_t e01 = a00 ^ a10, e12 = a10 ^ a11, e23 = a01 ^ a11, e30 = a00 ^ a01;
    uint32_t m = (yin && zin) ? mS : 0u;
    b.f[0] = (e01 | e12 | e23 | e30) & m;
    b.f4[0] = (e01 & e12 & e23 & e30) & m;
  }
  // y-normal face (b=z, c=x): EZ(v), EX(v+Sz), EZ(v+1), EX(v)
  {
    uint32_t e01 = a00 ^ a01, e12 = a01 ^ s01, e23 = s00 ^ s01, e30 = a00 ^ s00;
    uint32_t m = zin ? mR : 0u;
    b.f[1] = (e01 | e12 | e23 | e30) & m;
    b.f4[1] = (e01 & e12 & e23 & e30) & m;
  }
  // z-normal face (b=x, c=y): EX(v), EY(v+1), EX(v+Sy), EY(v)
  {
    uint32_t e01 = a00 ^ s00, e12 = s00 ^ s10, e23 = a10 ^ s10, e30 = a00 ^ a10;
    uint32_t m = yin ? mR : 0u;
    b.f[2] = (e01 | e12 | e23 | e30) & m;
    b.f4[2] = (e01 & e12 & e23 & e30) & m;
  }
  {
    uint32_t d = (a00 ^ s00) | (a00 ^ a10) | (a00 ^ s10) | (a00 ^ a01) | (a00 ^ s01) | (a00 ^ a11) | (a00 ^ s11);
    b.cell = (yin && zin) ? (d & mR) : 0u;
  }
  return b;
}

__device__ __forceinline__ void active_counts(const ActiveBits& b, uint32_t (&c)[kActiveCh]) {
  uint32_t nf = __popc(b.f[0]) + __popc(b.f[1]) + __popc(b.f[2]);
  uint32_t n4 = __popc(b.f4[0]) + __popc(b.f4[1]) + __popc(b.f4[2]);
  c[0] = __popc(b.e[0]) + __popc(b.e[1]) + __popc(b.e[2]);
  c[1] = nf + n4;
  c[2] = __popc(b.cell);
  c[3] = nf;
  c[4] = n4;
}

// Pass 1: per-tile counts only (6 channels: edges, instances, cells, faces,
// 4-crossing faces, active words); nothing per word is written.
__device__ __forceinline__ bool word_active(const ActiveBits& b) {
  return (b.e[0] | b.e[1] | b.e[2] | b.f[0] | b.f[1] | b.f[2] | b.cell) != 0u;  // f4 is a subset of f
}

template <bool B>
__global__ void __launch_bounds__(kActiveBlock) k_active_bits(GridP g, const uint32_t* __restrict__ L,
                                                              uint2* __restrict__ occ, uint32_t* __restrict__ sums,
                                                              int64_t ntiles, DevStats* st) {
  __shared__ uint32_t part[kActiveBlock / 32][kActiveCh];
  uint32_t c[kActiveCh] = {0, 0, 0, 0, 0, 0};
  uint32_t shell = 0;
  for (int j = 0; j < kActiveSub; j++) {
    const int64_t idx = (int64_t)blockIdx.x * kActiveTile + j * kActiveBlock + threadIdx.x;
    if (idx >= g.NW) break;
    int64_t y, z, wx;
    word_coords(g, idx, y, z, wx);
    const ActiveBits b = compute_active(g, L, y, z, wx);
    uint32_t cw[kActiveCh];
    active_counts(b, cw);
    cw[5] = word_active(b) ? 1u : 0u;
    // occupancy bitmap of the warp's 32 consecutive words
    const uint32_t act = __ballot_sync(__activemask(), cw[5] != 0u);
    if ((threadIdx.x & 31) == 0) occ[idx >> 5].x = act;
#pragma unroll
    for (int ch = 0; ch < kActiveCh; ch++) c[ch] += cw[ch];
    // boundary_inside_count (grid.py:102-106)
    const uint32_t lab = (z >= g.own0 && z < g.own1) ? (L[idx] & bits_below(g.S, wx)) : 0u;
    const int64_t zl = z - (int64_t)shape_of_z(g, z) * g.S;
    uint32_t sh;
    if (y == 0 || y == g.R || zl == 0 || zl == g.R) {
      sh = __popc(lab);
    } else {
      uint32_t m = 0u;
      if (wx == 0) m |= 1u;
      if ((g.R >> 5) == wx) m |= 1u << (g.R & 31);
      sh = __popc(lab & m);
    }
    if constexpr (B) warp_count<true>(&st[shape_of_z(g, z)].boundary_inside, sh);  // per shape
    else shell += sh;
  }
  // tile totals: warp sums, then one thread over the warps (no scan needed)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int ch = 0; ch < kActiveCh; ch++) {
    const uint32_t v = __reduce_add_sync(0xffffffffu, c[ch]);
    if (lane == 0) part[wid][ch] = v;
  }
  shell = __reduce_add_sync(0xffffffffu, shell);
  if (lane == 0 && shell) atomicAdd(&st->boundary_inside, (unsigned long long)shell);
  __syncthreads();
  if (threadIdx.x < kActiveCh) {
    uint32_t t = 0;
    for (int w = 0; w < kActiveBlock / 32; w++) t += part[w][threadIdx.x];
    sums[threadIdx.x * ntiles + blockIdx.x] = t;
  }
}

int64_t active_tiles(const GridP& g) { return (g.NW + kActiveTile - 1) / kActiveTile; }
int64_t occ_words(const GridP& g) { return (g.NW + 31) / 32; }

void launch_active_bits(const GridP& g, const uint32_t* L, uint2* occ, uint32_t* tile_sums, DevStats* st,
                        cudaStream_t s) {
  int64_t nt = active_tiles(g);
  if (g.nb) k_active_bits<true><<<(unsigned)nt, kActiveBlock, 0, s>>>(g, L, occ, tile_sums, nt, st);
  else k_active_bits<false><<<(unsigned)nt, kActiveBlock, 0, s>>>(g, L, occ, tile_sums, nt, st);
}

void launch_scan_tiles(uint32_t* sums, int64_t ntiles, int nch, unsigned long long* totals, cudaStream_t s) {
  switch (nch) {
    case 1: k_scan_tiles<1><<<1, 1024, 0, s>>>(sums, ntiles, totals); break;
    case 2: k_scan_tiles<2><<<1, 1024, 0, s>>>(sums, ntiles, totals); break;
    case 6: k_scan_tiles<6><<<1, 1024, 0, s>>>(sums, ntiles, totals); break;
    default: k_scan_tiles<5><<<1, 1024, 0, s>>>(sums, ntiles, totals); break;
  }
}

// Pass 2, per tile of kActiveGroups occupancy groups (32 words each, pass 1
// wrote their bitmaps): (a) a warp per group sums the counts of its active
// words (one lane per word), (b) six warps scan the groups' totals (one
// channel each), (c) a warp per non-empty group recomputes its active words,
// scans them across lanes and writes the records, the group prefix and the
// key lists.  Inactive words -- most of the grid -- cost one bitmap read.
__device__ __forceinline__ ActiveBits active_word(const GridP& g, const uint32_t* __restrict__ L, int64_t w,
                                                  int64_t& y, int64_t& z, int64_t& wx) {
  word_coords(g, w, y, z, wx);
  return compute_active(g, L, y, z, wx);
}

// write the record of active word (y, z, wx) and its keys at positions pos
__device__ __forceinline__ void emit_word(const GridP& g, const ActiveBits& b, int64_t y, int64_t z, int64_t wx,
                                          const uint32_t (&pos)[kActiveCh], WordRec* __restrict__ recs,
                                          int64_t* __restrict__ edge_key, int64_t* __restrict__ inst_key,
                                          int64_t* __restrict__ cell_id, int64_t* __restrict__ f4_key,
                                          int64_t* __restrict__ face_key, int64_t* __restrict__ face_nc) {
  WordRec r;
  for (int a = 0; a < 3; a++) {
    r.e[a] = b.e[a];
    r.f[a] = b.f[a];
    r.f4[a] = b.f4[a];
    r.cf[a] = 0u;
  }
  r.cell = b.cell;
  r.pe = pos[0];
  r.pq = pos[1];
  r.pc = pos[2];
  recs[pos[5]] = r;
  const int64_t vbase = (z * g.S + y) * g.S + wx * 32;  // global vertex id of bit 0 (x = 32 wx)
  // edges: ascending vertex, then axis (edge key = vid*3 + axis)
  uint32_t any = b.e[0] | b.e[1] | b.e[2];
  uint32_t pe = pos[0];
  while (any) {
    int bit = __ffs(any) - 1;
    any &= any - 1;
    int64_t vid = vbase + bit;
    for (int a = 0; a < 3; a++)
      if ((b.e[a] >> bit) & 1u) edge_key[pe++] = vid * 3 + a;
  }
  uint32_t anyf = b.f[0] | b.f[1] | b.f[2];
  uint32_t pq = pos[1], pf = pos[3], p4 = pos[4];
  while (anyf) {
    int bit = __ffs(anyf) - 1;
    anyf &= anyf - 1;
    int64_t vid = vbase + bit;
    for (int n = 0; n < 3; n++) {
      if (!((b.f[n] >> bit) & 1u)) continue;
      const int64_t fk = vid * 3 + n;
      const bool four = (b.f4[n] >> bit) & 1u;
      inst_key[pq++] = fk * 2;
      if (four) {
        inst_key[pq++] = fk * 2 + 1;
        f4_key[p4++] = fk;
      }
      if (face_key) {
        face_key[pf] = fk;
        face_nc[pf] = four ? 4 : 2;
      }
      pf++;
    }
  }
  uint32_t cl = b.cell;
  uint32_t pc = pos[2];
  while (cl) {
    int bit = __ffs(cl) - 1;
    cl &= cl - 1;
    int64_t x = wx * 32 + bit;
    cell_id[pc++] = x + y * g.R + z * g.R * g.R;
  }
}

__global__ void __launch_bounds__(kActiveBlock) k_active_compact_wpg(GridP g, const uint32_t* __restrict__ L,
                                                                 uint2* __restrict__ occ, WordRec* __restrict__ recs,
                                                                 const uint32_t* __restrict__ sums, int64_t ntiles,
                                                                 int64_t* __restrict__ edge_key,
                                                                 int64_t* __restrict__ inst_key,
                                                                 int64_t* __restrict__ cell_id,
                                                                 int64_t* __restrict__ f4_key,
                                                                 int64_t* __restrict__ face_key,
                                                                 int64_t* __restrict__ face_nc) {
  static_assert(kActiveGroups == 64 && kActiveCh <= kActiveBlock / 32, "tile scan: 2 groups per lane, a warp per channel");
  __shared__ uint32_t gt[kActiveGroups][kActiveCh];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int kWarps = kActiveBlock / 32;
  const int64_t ngrp = (g.NW + 31) >> 5;
  const int64_t g0 = (int64_t)blockIdx.x * kActiveGroups;
  // (a) group totals
  for (int i = wid; i < kActiveGroups; i += kWarps) {
    const int64_t grp = g0 + i;
    const uint32_t bits = grp < ngrp ? occ[grp].x : 0u;
    uint32_t c[kActiveCh] = {0, 0, 0, 0, 0, 0};
    if (bits) {  // warp-uniform
      if ((bits >> lane) & 1u) {
        int64_t y, z, wx;
        active_counts(active_word(g, L, grp * 32 + lane, y, z, wx), c);
        c[5] = 1u;
      }
#pragma unroll
      for (int ch = 0; ch < kActiveCh; ch++) c[ch] = __reduce_add_sync(0xffffffffu, c[ch]);
    }
    if (lane == 0)
#pragma unroll
      for (int ch = 0; ch < kActiveCh; ch++) gt[i][ch] = c[ch];
  }
  __syncthreads();
  // (b) exclusive group prefixes (tile offset included), one warp per channel
  if (wid < kActiveCh) {
    const uint32_t v0 = gt[2 * lane][wid], v1 = gt[2 * lane + 1][wid];
    uint32_t x = v0 + v1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    const uint32_t ex = x - v0 - v1 + sums[wid * ntiles + blockIdx.x];
    gt[2 * lane][wid] = ex;
    gt[2 * lane + 1][wid] = ex + v0;
  }
  __syncthreads();
  // (c) records and keys
  for (int i = wid; i < kActiveGroups; i += kWarps) {
    const int64_t grp = g0 + i;
    if (grp >= ngrp) break;  // warp-uniform
    const uint32_t bits = occ[grp].x;
    if (lane == 0) occ[grp].y = gt[i][5];
    if (!bits) continue;
    const bool act = (bits >> lane) & 1u;
    ActiveBits b{};
    uint32_t c[kActiveCh] = {0, 0, 0, 0, 0, 0};
    int64_t y = 0, z = 0, wx = 0;
    if (act) {
      b = active_word(g, L, grp * 32 + lane, y, z, wx);
      active_counts(b, c);
      c[5] = 1u;
    }
    uint32_t pos[kActiveCh];
#pragma unroll
    for (int ch = 0; ch < kActiveCh; ch++) {
      uint32_t x = c[ch];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      pos[ch] = gt[i][ch] + x - c[ch];
    }
    if (!act) continue;
    emit_word(g, b, y, z, wx, pos, recs, edge_key, inst_key, cell_id, f4_key, face_key, face_nc);
  }
}

// Thread per group (large grids: many groups, few active words each)
__global__ void __launch_bounds__(kActiveGroups) k_active_compact_tpg(GridP g, const uint32_t* __restrict__ L,
                                                                      uint2* __restrict__ occ,
                                                                      WordRec* __restrict__ recs,
                                                                      const uint32_t* __restrict__ sums,
                                                                      int64_t ntiles, int64_t* __restrict__ edge_key,
                                                                      int64_t* __restrict__ inst_key,
                                                                      int64_t* __restrict__ cell_id,
                                                                      int64_t* __restrict__ f4_key,
                                                                      int64_t* __restrict__ face_key,
                                                                      int64_t* __restrict__ face_nc) {
  const int64_t grp = (int64_t)blockIdx.x * kActiveGroups + threadIdx.x;
  const int64_t ngrp = (g.NW + 31) >> 5;
  const uint32_t bits = grp < ngrp ? occ[grp].x : 0u;
  uint32_t c[kActiveCh] = {0, 0, 0, 0, 0, 0};
  for (uint32_t m = bits; m; m &= m - 1) {
    int64_t y, z, wx;
    uint32_t cw[kActiveCh];
    active_counts(active_word(g, L, grp * 32 + __ffs(m) - 1, y, z, wx), cw);
#pragma unroll
    for (int ch = 0; ch < 5; ch++) c[ch] += cw[ch];
  }
  c[5] = __popc(bits);
  uint32_t ex[kActiveCh], tot[kActiveCh];
  block_exscan<kActiveCh, kActiveGroups>(c, ex, tot);
  if (grp >= ngrp) return;
  uint32_t pos[kActiveCh];
#pragma unroll
  for (int ch = 0; ch < kActiveCh; ch++) pos[ch] = sums[ch * ntiles + blockIdx.x] + ex[ch];
  occ[grp].y = pos[5];
  for (uint32_t m = bits; m; m &= m - 1) {
    int64_t y, z, wx;
    const ActiveBits b = active_word(g, L, grp * 32 + __ffs(m) - 1, y, z, wx);
    uint32_t cw[kActiveCh];
    active_counts(b, cw);
    cw[5] = 1u;
    emit_word(g, b, y, z, wx, pos, recs, edge_key, inst_key, cell_id, f4_key, face_key, face_nc);
#pragma unroll
    for (int ch = 0; ch < kActiveCh; ch++) pos[ch] += cw[ch];
  }
}

void launch_active_compact(const GridP& g, const uint32_t* L, RecView rec, const uint32_t* tile_sums,
                           int64_t* edge_key, int64_t* inst_key, int64_t* cell_id, int64_t* f4_key, int64_t* face_key,
                           int64_t* face_nc, cudaStream_t s) {
  int64_t nt = active_tiles(g);
  // a warp per group while groups are few (latency: a thread would walk its
  // group's active words serially), a thread per group on large grids
  if ((g.NW + 31) / 32 < kActiveWarpGroups)
    k_active_compact_wpg<<<(unsigned)nt, kActiveBlock, 0, s>>>(g, L, const_cast<uint2*>(rec.occ), rec.rec, tile_sums,
                                                                nt, edge_key, inst_key, cell_id, f4_key, face_key,
                                                                face_nc);
  else
    k_active_compact_tpg<<<(unsigned)nt, kActiveGroups, 0, s>>>(g, L, const_cast<uint2*>(rec.occ), rec.rec, tile_sums,
                                                                 nt, edge_key, inst_key, cell_id, f4_key, face_key,
                                                                 face_nc);
}

// exclusive element prefixes (edges, instances, cells) at word w: the ranks
// stored in the first active record at or after w, else the totals
__global__ void k_prefix_at(RecView rv, int64_t w, int64_t A, const unsigned long long* __restrict__ totals,
                            unsigned long long* __restrict__ out) {
  const uint2 o = rv.occ[w >> 5];
  const int64_t a = (int64_t)o.y + __popc(o.x & lowmask((int)(w & 31)));
  if (a < A) {
    out[0] = rv.rec[a].pe;
    out[1] = rv.rec[a].pq;
    out[2] = rv.rec[a].pc;
  } else {
    out[0] = totals[0];
    out[1] = totals[1];
    out[2] = totals[2];
  }
}
void launch_prefix_at(RecView rv, int64_t w, int64_t A, const unsigned long long* totals, unsigned long long* out,
                      cudaStream_t s) {
  k_prefix_at<<<1, 1, 0, s>>>(rv, w, A, totals, out);
}

// first partition of the window's owned cells and the end of them: pbase at
// the owned cell rows c_lo = pre[2], c_hi = pre[5] (or C without a top
// bound), P = the partition total past the last cell
__global__ void k_part_bounds(const uint32_t* __restrict__ pbase, int64_t C, const unsigned long long* __restrict__ pre,
                              int has_hi, const unsigned long long* __restrict__ totals, unsigned long long* out) {
  const unsigned long long P = totals[0];
  const int64_t clo = (int64_t)pre[2], chi = has_hi ? (int64_t)pre[5] : C;
  out[0] = clo < C ? (unsigned long long)pbase[clo] : P;
  out[1] = chi < C ? (unsigned long long)pbase[chi] : P;
}
void launch_part_bounds(const uint32_t* pbase, int64_t C, const unsigned long long* pre, bool has_hi,
                        const unsigned long long* totals, unsigned long long* out, cudaStream_t s) {
  k_part_bounds<<<1, 1, 0, s>>>(pbase, C, pre, has_hi ? 1 : 0, totals, out);
}

// ===========================================================================
// face-centre probes (dualize.py:59-70): corner + 0.5 h along both in-plane axes
// ===========================================================================
__device__ __forceinline__ void face_center(const GridP& g, int64_t fk, double p[3]) {
  int64_t vid = fk / 3;
  int n = (int)(fk % 3), b = (n + 1) % 3, c = (n + 2) % 3;
  vposition(g, vid, p);
  p[b] = p[b] + 0.5 * g.h[b];
  p[c] = p[c] + 0.5 * g.h[c];
}
__device__ __forceinline__ void set_center_bit(const GridP& g, const RecView& rec, int64_t fk) {
  int64_t vid = fk / 3;
  int n = (int)(fk % 3);
  int64_t c[3];
  vid_coords(g, vid, c);
  atomicOr(&rec_find(rec, word_of(g, c[0], c[1], c[2]))->cf[n], 1u << (c[0] & 31));  // a 4-crossing face's word is active
}

__global__ void k_face_center_points(GridP g, const int64_t* __restrict__ f4, int64_t n, double* __restrict__ pts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3];
  face_center(g, f4[i], p);
  pts[3 * i] = p[0];
  pts[3 * i + 1] = p[1];
  pts[3 * i + 2] = p[2];
}
void launch_face_center_points(const GridP& g, const int64_t* f4_key, int64_t n, double* pts, cudaStream_t s) {
  if (n) k_face_center_points<<<grid_for(n, 128), 128, 0, s>>>(g, f4_key, n, pts);
}

template <bool B>
__global__ void k_face_center_analytic(GridP g, FieldP f, const int64_t* __restrict__ f4, int64_t n,
                                       RecView rec) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3];
  GridP gl = g;
  int b = 0;
  if constexpr (B) b = localize<B>(gl, idiv(f4[i] / 3, g.S2));
  face_center(gl, f4[i], p);
  uint32_t lab;
  if constexpr (B) lab = field_label_t<true>(f.batch[b], p);
  else lab = field_label(f, p);
  if (lab) set_center_bit(g, rec, f4[i]);
}
void launch_face_center_analytic(const GridP& g, const FieldP& f, const int64_t* f4_key, int64_t n, RecView rec,
                                 cudaStream_t s) {
  if (!n) return;
  if (g.nb) k_face_center_analytic<true><<<grid_for(n, 128), 128, 0, s>>>(g, f, f4_key, n, rec);
  else k_face_center_analytic<false><<<grid_for(n, 128), 128, 0, s>>>(g, f, f4_key, n, rec);
}

__global__ void k_face_center_scatter(GridP g, const int64_t* __restrict__ f4, const uint8_t* __restrict__ lab,
                                      int64_t n, RecView rec) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (lab[i]) set_center_bit(g, rec, f4[i]);
}
void launch_face_center_scatter(const GridP& g, const int64_t* f4_key, const uint8_t* labels, int64_t n,
                                RecView rec, cudaStream_t s) {
  if (n) k_face_center_scatter<<<grid_for(n, 128), 128, 0, s>>>(g, f4_key, labels, n, rec);
}

// ===========================================================================
// K3: 1D points (search.py:71-94, pipeline.py:94-123)
// ===========================================================================
struct EdgeGeom {
  int64_t vin, vout;
  double pin[3], span[3];
};
__device__ __forceinline__ EdgeGeom edge_geom(const GridP& g, const uint32_t* L, int64_t key) {
  EdgeGeom e;
  int64_t vid = key / 3;
  int a = (int)(key % 3);
  int64_t other = vid + vstep(g, a);
  bool base_in = label_at(L, g, vid) == 1u;
  e.vin = base_in ? vid : other;
  e.vout = base_in ? other : vid;
  double po[3];
  vposition(g, e.vin, e.pin);
  vposition(g, e.vout, po);
  for (int j = 0; j < 3; j++) e.span[j] = po[j] - e.pin[j];
  return e;
}

__device__ __forceinline__ double clip_t(double t, int iters) {
  double eps = ldexp(1.0, -iters);
  double upper = 1.0 - eps;
  t = t < eps ? eps : t;
  t = t > upper ? upper : t;
  return t;
}

__device__ __forceinline__ double linear_t(double ri, double ro, double iso) {
  double pi = ri - iso, po = ro - iso;
  double den = pi - po;
  double t = fabs(den) < 1e-300 ? 0.5 : pi / (den == 0.0 ? 1.0 : den);
  t = t < 0.0 ? 0.0 : t;
  return t > 1.0 ? 1.0 : t;
}

template <int SEL>
__device__ __forceinline__ void search1d_one(const GridP& g, const FieldP& f, const OptP& o,
                                             const uint32_t* __restrict__ L, const int64_t* __restrict__ edge_key,
                                             int64_t k, double* __restrict__ tout, double* __restrict__ pos,
                                             int64_t* __restrict__ vin_out) {
  EdgeGeom e = edge_geom(g, L, edge_key[k]);
  double t;
  if (o.one_d == ODC_ONE_D_BINARY) {
    double lo = 0.0, hi = 1.0;
    for (int it = 0; it < o.iters_1d; it++) {
      double tm = 0.5 * (lo + hi);
      double q[3];
      for (int j = 0; j < 3; j++) q[j] = e.pin[j] + tm * e.span[j];
      if (field_label_t<SEL>(f, q)) lo = tm; else hi = tm;  // bracket: label(lo)=1, label(hi)=0
    }
    t = clip_t(0.5 * (lo + hi), o.iters_1d);
  } else if (o.one_d == ODC_ONE_D_MIDPOINT) {
    t = 0.5;
  } else {
    double ri, ro;
    if (o.continuous) {
      double po[3];
      vposition(g, e.vout, po);
      ri = field_raw_t<SEL>(f, e.pin);
      ro = field_raw_t<SEL>(f, po);
    } else {
      ri = 1.0;
      ro = 0.0;
    }
    t = linear_t(ri, ro, f.iso);
  }
  tout[k] = t;
  for (int j = 0; j < 3; j++) pos[3 * k + j] = e.pin[j] + t * e.span[j];
  if (vin_out) vin_out[k] = e.vin;
}

template <bool B, int EV>
__global__ void __launch_bounds__(128) k_search1d_analytic(GridP g, FieldP f, OptP o, const uint32_t* __restrict__ L,
                                                           const int64_t* __restrict__ edge_key, int64_t K,
                                                           double* __restrict__ tout, double* __restrict__ pos,
                                                           int64_t* __restrict__ vin_out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  if constexpr (B) {
    GridP gl = g;
    const int sb = localize<B>(gl, idiv(edge_key[k] / 3, g.S2));
    const FieldP& fb = f.batch[sb];
    switch (fb.ev) {  // the shape's specialised evaluation (elements are in shape order)
      case EV_SPHERE: search1d_one<EV_SPHERE>(gl, fb, o, L, edge_key, k, tout, pos, vin_out); break;
      case EV_BOX: search1d_one<EV_BOX>(gl, fb, o, L, edge_key, k, tout, pos, vin_out); break;
      case EV_TORUS: search1d_one<EV_TORUS>(gl, fb, o, L, edge_key, k, tout, pos, vin_out); break;
      default: search1d_one<EV_SEL>(gl, fb, o, L, edge_key, k, tout, pos, vin_out); break;
    }
  } else {
    search1d_one<EV>(g, f, o, L, edge_key, k, tout, pos, vin_out);
  }
}

void launch_search1d_analytic(const GridP& g, const FieldP& f, const OptP& o, const uint32_t* L,
                              const int64_t* edge_key, int64_t K, double* t, double* pos, int64_t* v_in,
                              cudaStream_t s) {
  if (!K) return;
  const unsigned grid = grid_for(K, 128);
#define S1A(BB, EVV) k_search1d_analytic<BB, EVV><<<grid, 128, 0, s>>>(g, f, o, L, edge_key, K, t, pos, v_in)
  if (g.nb) {
    S1A(true, EV_SEL);
    return;
  }
  switch (ev_mode_of(f)) {
    case EV_SPHERE: S1A(false, EV_SPHERE); break;
    case EV_BOX: S1A(false, EV_BOX); break;
    case EV_TORUS: S1A(false, EV_TORUS); break;
    case EV_SPHERE2: S1A(false, EV_SPHERE2); break;
    case EV_BOX2F: S1A(false, EV_BOX2F); break;
    default: S1A(false, EV_PARAM); break;
  }
#undef S1A
}

// lock-step form (batched fields): lo/hi state, points, update, finish
__global__ void k_search1d_init(int64_t K, double* lo, double* hi) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  lo[k] = 0.0;
  hi[k] = 1.0;
}
void launch_search1d_init(const GridP&, const uint32_t*, const int64_t*, int64_t K, double* lo, double* hi,
                          cudaStream_t s) {
  if (K) k_search1d_init<<<grid_for(K, 256), 256, 0, s>>>(K, lo, hi);
}
__global__ void k_search1d_points(GridP g, const uint32_t* __restrict__ L, const int64_t* __restrict__ edge_key,
                                  int64_t K, const double* __restrict__ lo, const double* __restrict__ hi,
                                  double* __restrict__ pts) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  EdgeGeom e = edge_geom(g, L, edge_key[k]);
  double tm = 0.5 * (lo[k] + hi[k]);
  for (int j = 0; j < 3; j++) pts[3 * k + j] = e.pin[j] + tm * e.span[j];
}
void launch_search1d_points(const GridP& g, const uint32_t* L, const int64_t* edge_key, int64_t K, const double* lo,
                            const double* hi, double* pts, cudaStream_t s) {
  if (K) k_search1d_points<<<grid_for(K, 256), 256, 0, s>>>(g, L, edge_key, K, lo, hi, pts);
}
__global__ void k_search1d_update(int64_t K, const uint8_t* __restrict__ lab, double* lo, double* hi) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double tm = 0.5 * (lo[k] + hi[k]);
  if (lab[k] == 1) lo[k] = tm; else hi[k] = tm;
}
void launch_search1d_update(int64_t K, const uint8_t* lab, double* lo, double* hi, cudaStream_t s) {
  if (K) k_search1d_update<<<grid_for(K, 256), 256, 0, s>>>(K, lab, lo, hi);
}
__global__ void k_search1d_finish(GridP g, OptP o, double iso, const uint32_t* __restrict__ L,
                                  const int64_t* __restrict__ edge_key, int64_t K, const double* __restrict__ lo,
                                  const double* __restrict__ hi, const double* __restrict__ raw_in,
                                  const double* __restrict__ raw_out, double* __restrict__ tout,
                                  double* __restrict__ pos, int64_t* __restrict__ vin_out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  EdgeGeom e = edge_geom(g, L, edge_key[k]);
  double t;
  if (o.one_d == ODC_ONE_D_BINARY) t = clip_t(0.5 * (lo[k] + hi[k]), o.iters_1d);
  else if (o.one_d == ODC_ONE_D_MIDPOINT) t = 0.5;
  else t = raw_in ? linear_t(raw_in[k], raw_out[k], iso) : linear_t(1.0, 0.0, iso);
  tout[k] = t;
  for (int j = 0; j < 3; j++) pos[3 * k + j] = e.pin[j] + t * e.span[j];
  if (vin_out) vin_out[k] = e.vin;
}
void launch_search1d_finish(const GridP& g, const OptP& o, const uint32_t* L, const int64_t* edge_key, int64_t K,
                            const double* lo, const double* hi, const double* raw_in, const double* raw_out,
                            double* t, double* pos, int64_t* v_in, cudaStream_t s) {
  if (K)
    k_search1d_finish<<<grid_for(K, 256), 256, 0, s>>>(g, o, 0.5, L, edge_key, K, lo, hi, raw_in, raw_out, t, pos,
                                                       v_in);
}

__global__ void k_edge_endpoints(GridP g, const uint32_t* __restrict__ L, const int64_t* __restrict__ edge_key,
                                 int64_t K, int which, double* __restrict__ pts) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  EdgeGeom e = edge_geom(g, L, edge_key[k]);
  vposition(g, which ? e.vout : e.vin, pts + 3 * k);
}
void launch_edge_endpoints(const GridP& g, const uint32_t* L, const int64_t* edge_key, int64_t K, int which,
                           double* pts, cudaStream_t s) {
  if (K) k_edge_endpoints<<<grid_for(K, 256), 256, 0, s>>>(g, L, edge_key, K, which, pts);
}

// ===========================================================================
// K5: 2D points -- build_face_batch (dualize.py:97-129) + find_2d_points
// (search.py:194-322) + line_binary_search_batch (search.py:97-133).
// One instance = (face, edge pair).  In-plane axes u = (n+1)%3, v = (n+2)%3;
// lift(u,v) = origin with origin[u] += u, origin[v] += v (search.py:172-177).
// ===========================================================================
struct Inst2D {
  double org[3];
  int bu, bv;
  double hu, hv, hmin;
  double p1[2], p2[2];
  uint32_t cl[4];  // corner labels w0..w3
};

// Decode an instance key (face_key*2 + slot): corner labels, the slot's edge
// pair (dualize.py:37-48, :72-88) and the two 1D points in face coordinates.
__device__ __forceinline__ bool decode_instance(const GridP& g, const uint32_t* L, RecView rec,
                                                int64_t ikey, const double* pos1d, Inst2D& I, int64_t pair[2]) {
  const int64_t fk = ikey >> 1;
  const int slot = (int)(ikey & 1);
  const int64_t vid = fk / 3;
  const int n = (int)(fk % 3), b = (n + 1) % 3, c = (n + 2) % 3;
  const int64_t w0 = vid, w1 = vid + vstep(g, b), w3 = vid + vstep(g, c), w2 = w1 + vstep(g, c);
  I.cl[0] = label_at(L, g, w0);
  I.cl[1] = label_at(L, g, w1);
  I.cl[2] = label_at(L, g, w2);
  I.cl[3] = label_at(L, g, w3);
  const int64_t ek[4] = {w0 * 3 + b, w1 * 3 + c, w3 * 3 + b, w0 * 3 + c};
  const bool cr[4] = {I.cl[0] != I.cl[1], I.cl[1] != I.cl[2], I.cl[3] != I.cl[2], I.cl[0] != I.cl[3]};
  const int ncross = (int)cr[0] + (int)cr[1] + (int)cr[2] + (int)cr[3];
  int64_t a0, a1;
  if (ncross == 2) {  // the two crossing edges in j order (no dynamic index: registers)
    bool have = false;
    a0 = a1 = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (cr[j] && !have) {
        a0 = ek[j];
        have = true;
      } else if (cr[j]) {
        a1 = ek[j];
      }
    }
  } else {
    int64_t cc[3];
    vid_coords(g, vid, cc);
    const uint32_t centre = (rec_find(rec, word_of(g, cc[0], cc[1], cc[2]))->cf[n] >> (cc[0] & 31)) & 1u;
    if (centre == I.cl[0]) {
      a0 = slot ? ek[2] : ek[0];
      a1 = slot ? ek[3] : ek[1];
    } else {
      a0 = slot ? ek[1] : ek[3];
      a1 = slot ? ek[2] : ek[0];
    }
  }
  if (a1 < a0) { int64_t t = a0; a0 = a1; a1 = t; }
  pair[0] = a0;
  pair[1] = a1;
  vposition(g, vid, I.org);
  I.bu = b;
  I.bv = c;
  I.hu = b == 0 ? g.h[0] : b == 1 ? g.h[1] : g.h[2];
  I.hv = c == 0 ? g.h[0] : c == 1 ? g.h[1] : g.h[2];
  I.hmin = I.hu < I.hv ? I.hu : I.hv;
  const double ob = b == 0 ? I.org[0] : b == 1 ? I.org[1] : I.org[2];
  const double oc = c == 0 ? I.org[0] : c == 1 ? I.org[1] : I.org[2];
  const int64_t r0 = edge_rank(rec, g, a0 / 3, (int)(a0 % 3));
  const int64_t r1 = edge_rank(rec, g, a1 / 3, (int)(a1 % 3));
  I.p1[0] = pos1d[3 * r0 + b] - ob;
  I.p1[1] = pos1d[3 * r0 + c] - oc;
  I.p2[0] = pos1d[3 * r1 + b] - ob;
  I.p2[1] = pos1d[3 * r1 + c] - oc;
  return true;
}

__device__ __forceinline__ void lift(const Inst2D& I, double u, double v, double p[3]) {
  // the addend is selected, not the slot (p[I.bu] = ... is a dynamic index
  // and puts p in local memory).  org + 0.0 == org: grid positions are
  // lo + c*h rounded to nearest, never -0.0.
#pragma unroll
  for (int a = 0; a < 3; a++) p[a] = I.org[a] + (a == I.bu ? u : a == I.bv ? v : 0.0);
}

// Geometry derived from the chord, before any evaluation (search.py:213-219)
struct Chord {
  double mid[2], dl[2];
  bool degen;
};
__device__ __forceinline__ Chord make_chord(const Inst2D& I) {
  Chord ch;
  ch.mid[0] = 0.5 * (I.p1[0] + I.p2[0]);
  ch.mid[1] = 0.5 * (I.p1[1] + I.p2[1]);
  const double c0 = I.p2[0] - I.p1[0], c1 = I.p2[1] - I.p1[1];
  const double clen = sqrt(c0 * c0 + c1 * c1);
  ch.degen = clen < 1e-12 * I.hmin;
  const double safe = ch.degen ? 1.0 : clen;
  ch.dl[0] = c0 / safe;
  ch.dl[1] = c1 / safe;
  return ch;
}

// Ray side toward the nearest corner whose label differs from the midpoint
// label (search.py:222-239).  Returns false when no corner differs.
__device__ __forceinline__ bool ray_direction(const Inst2D& I, const Chord& ch, uint32_t mid_label, double ray[2]) {
  const double perp0 = -ch.dl[1], perp1 = ch.dl[0];
  const double cu[4] = {0.0, I.hu, I.hu, 0.0}, cv[4] = {0.0, 0.0, I.hv, I.hv};
  double plus_d = INFINITY, minus_d = INFINITY;
#pragma unroll
  for (int c = 0; c < 4; c++) {
    const double r0 = cu[c] - ch.mid[0], r1 = cv[c] - ch.mid[1];
    const double side = r0 * perp0 + r1 * perp1;
    const double dist = sqrt(r0 * r0 + r1 * r1);
    if (I.cl[c] == mid_label) continue;
    if (side > 0 && dist < plus_d) plus_d = dist;
    if (side < 0 && dist < minus_d) minus_d = dist;
  }
  if (isinf(plus_d) && isinf(minus_d)) return false;
  if (plus_d <= minus_d) {
    ray[0] = perp0;
    ray[1] = perp1;
  } else {
    ray[0] = -perp0;
    ray[1] = -perp1;
  }
  return true;
}

// Final step: line intersection, clamp, status (search.py:278-322)
__device__ __forceinline__ void finish2d(const Inst2D& I, const Chord& ch, double dist_r, bool found_r,
                                         const double qa[2], bool found_a, const double qb[2], bool found_b,
                                         double out2[2], uint8_t& status) {
  const double a1[2] = {qa[0] - I.p1[0], qa[1] - I.p1[1]};
  const double a2[2] = {qb[0] - I.p2[0], qb[1] - I.p2[1]};
  const double l1 = sqrt(a1[0] * a1[0] + a1[1] * a1[1]);
  const double l2 = sqrt(a2[0] * a2[0] + a2[1] * a2[1]);
  const double cr = a1[0] * a2[1] - a1[1] * a2[0];
  const bool exact = dist_r <= 1e-4 * I.hmin;
  const bool parallel = (fabs(cr) <= 1e-6 * l1 * l2) || (l1 < 1e-12 * I.hmin) || (l2 < 1e-12 * I.hmin) || ch.degen;
  const double sc = parallel ? 1.0 : cr;
  const double d21[2] = {I.p2[0] - I.p1[0], I.p2[1] - I.p1[1]};
  const double tpar = (d21[0] * a2[1] - d21[1] * a2[0]) / sc;
  double pos[2];
  if (exact || parallel) {
    pos[0] = ch.mid[0];
    pos[1] = ch.mid[1];
  } else {
    pos[0] = I.p1[0] + tpar * a1[0];
    pos[1] = I.p1[1] + tpar * a1[1];
  }
  const double lov[2] = {-0.5 * I.hu, -0.5 * I.hv}, hiv[2] = {1.5 * I.hu, 1.5 * I.hv};
  const double delta[2] = {pos[0] - ch.mid[0], pos[1] - ch.mid[1]};
  double smin = INFINITY;
#pragma unroll
  for (int i = 0; i < 2; i++) {
    const double shi = delta[i] > 0 ? (hiv[i] - ch.mid[i]) / delta[i] : INFINITY;
    const double slo = delta[i] < 0 ? (lov[i] - ch.mid[i]) / delta[i] : INFINITY;
    const double m2 = shi < slo ? shi : slo;
    if (m2 < smin) smin = m2;
  }
  const double s = smin < 1.0 ? smin : 1.0;
  const bool clamped = s < 1.0;
  out2[0] = ch.mid[0] + s * delta[0];
  out2[1] = ch.mid[1] + s * delta[1];
  uint8_t st = 0;
  if (!(found_r && found_a && found_b)) st = 3;
  if (clamped) st = 2;
  if (parallel && !exact) st = 1;
  if (exact) st = 0;
  status = st;
}

// Fused per-instance search for analytic fields.  Evaluations happen in the
// same per-element order as the lock-step batches; skipping the samples
// after the first flip of a linear scan does not change any result, and the
// eval accounting reports the reference's logical counts.
template <int SEL>
__device__ __forceinline__ void line_binary(const FieldP& f, const Inst2D& I, const double o2[2], const double d2[2],
                                            uint32_t ref, double max_range, int nlin, int nbin, double& a_out,
                                            bool& found) {
  int first = nlin;
  found = false;
  for (int i = 1; i <= nlin; i++) {
    const double s = max_range * ((double)i / (double)nlin);
    double p[3];
    lift(I, o2[0] + s * d2[0], o2[1] + s * d2[1], p);
    if (field_label_t<SEL>(f, p) != ref) {
      first = i;
      found = true;
      break;
    }
  }
  double a = max_range * ((double)(first - 1) / (double)nlin);
  double b = max_range * ((double)first / (double)nlin);
  for (int it = 0; it < nbin; it++) {
    const double m = 0.5 * (a + b);
    double p[3];
    lift(I, o2[0] + m * d2[0], o2[1] + m * d2[1], p);
    if (field_label_t<SEL>(f, p) == ref) a = m; else b = m;
  }
  a_out = a;
}

// The two step-2 rays (search.py:266-276: -dl and +dl from the same point,
// same budget) searched side by side: each ray's samples and bisection are
// line_binary's, in the same order; interleaving the two independent
// evaluation chains gives the scheduler two fp64 chains per thread.
template <int SEL>
__device__ __forceinline__ void line_binary2(const FieldP& f, const Inst2D& I, const double o2[2],
                                             const double da2[2], const double db2[2], uint32_t ref, double max_range,
                                             int nlin, int nbin, double& a_out, bool& found_a, double& b_out,
                                             bool& found_b) {
  int fa = nlin, fb = nlin;
  found_a = found_b = false;
  for (int i = 1; i <= nlin && !(found_a && found_b); i++) {
    const double s = max_range * ((double)i / (double)nlin);
    if (!found_a) {
      double p[3];
      lift(I, o2[0] + s * da2[0], o2[1] + s * da2[1], p);
      if (field_label_t<SEL>(f, p) != ref) {
        fa = i;
        found_a = true;
      }
    }
    if (!found_b) {
      double p[3];
      lift(I, o2[0] + s * db2[0], o2[1] + s * db2[1], p);
      if (field_label_t<SEL>(f, p) != ref) {
        fb = i;
        found_b = true;
      }
    }
  }
  double aa = max_range * ((double)(fa - 1) / (double)nlin), ba = max_range * ((double)fa / (double)nlin);
  double ab = max_range * ((double)(fb - 1) / (double)nlin), bb = max_range * ((double)fb / (double)nlin);
  for (int it = 0; it < nbin; it++) {
    const double ma = 0.5 * (aa + ba), mb = 0.5 * (ab + bb);
    double pa[3], pb[3];
    lift(I, o2[0] + ma * da2[0], o2[1] + ma * da2[1], pa);
    lift(I, o2[0] + mb * db2[0], o2[1] + mb * db2[1], pb);
    const bool sa = field_label_t<SEL>(f, pa) == ref, sb = field_label_t<SEL>(f, pb) == ref;
    if (sa) aa = ma; else ba = ma;
    if (sb) ab = mb; else bb = mb;
  }
  a_out = aa;
  b_out = ab;
}

template <bool B, int EV>
__device__ __forceinline__ void search2d_one(const GridP& g, const FieldP& f, const OptP& o,
                                             const uint32_t* __restrict__ L, const RecView& rec,
                                             const int64_t* __restrict__ inst_key, int64_t q,
                                             const double* __restrict__ pos1d, const Stage2D& out,
                                             int64_t* __restrict__ inst_edges, DevStats* st, DevStatus* dst,
                                             int64_t st_lo, int64_t st_hi) {
  Inst2D I;
  int64_t pair[2];
  decode_instance(g, L, rec, inst_key[q], pos1d, I, pair);
  if (inst_edges) {
    inst_edges[2 * q] = pair[0];
    inst_edges[2 * q + 1] = pair[1];
  }
  const Chord ch = make_chord(I);
  double pm[3];
  lift(I, ch.mid[0], ch.mid[1], pm);
  const uint32_t mid_label = field_label_t<EV>(f, pm);
  double ray[2];
  if (!ray_direction(I, ch, mid_label, ray)) {
    raise_status(dst, ODC_E_ASSERT, q);
    return;
  }
  double dist_r;
  bool found_r;
  line_binary<EV>(f, I, ch.mid, ray, mid_label, o.s1_range * I.hmin, o.s1_lin, o.s1_bin, dist_r, found_r);
  const double q2[2] = {ch.mid[0] + dist_r * ray[0], ch.mid[1] + dist_r * ray[1]};
  const double r2 = o.s2_range * I.hmin;
  const double dneg[2] = {-ch.dl[0], -ch.dl[1]};
  double da, db;
  bool fa, fb;
  line_binary2<EV>(f, I, q2, dneg, ch.dl, mid_label, r2, o.s2_lin, o.s2_bin, da, fa, db, fb);
  const double qa[2] = {q2[0] + da * dneg[0], q2[1] + da * dneg[1]};
  const double qb[2] = {q2[0] + db * ch.dl[0], q2[1] + db * ch.dl[1]};
  double p2d[2];
  uint8_t status;
  finish2d(I, ch, dist_r, found_r, qa, fa, qb, fb, p2d, status);
  double p3[3];
  lift(I, p2d[0], p2d[1], p3);
  out.pos3[3 * q] = p3[0];
  out.pos3[3 * q + 1] = p3[1];
  out.pos3[3 * q + 2] = p3[2];
  if (out.pos2) {
    out.pos2[2 * q] = p2d[0];
    out.pos2[2 * q + 1] = p2d[1];
  }
  if (out.status) out.status[q] = status;
  if (out.mid) out.mid[q] = (uint8_t)mid_label;
  warp_count4<B>(st->status, status, q >= st_lo && q < st_hi);
}

template <bool B, int EV>
__global__ void __launch_bounds__(128) k_search2d_analytic(GridP g, FieldP f, OptP o, const uint32_t* __restrict__ L,
                                                           RecView rec,
                                                           const int64_t* __restrict__ inst_key, int64_t Q,
                                                           const double* __restrict__ pos1d, Stage2D out,
                                                           int64_t* __restrict__ inst_edges, DevStats* st,
                                                           DevStatus* dst, int64_t st_lo, int64_t st_hi) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  if constexpr (B) {
    GridP gl = g;
    const int sb = localize<B>(gl, idiv((inst_key[q] >> 1) / 3, g.S2));
    const FieldP& fb = f.batch[sb];
#define S2O(EVV) search2d_one<B, EVV>(gl, fb, o, L, rec, inst_key, q, pos1d, out, inst_edges, st + sb, dst, st_lo, st_hi)
    switch (fb.ev) {  // the shape's specialised evaluation (elements are in shape order)
      case EV_SPHERE: S2O(EV_SPHERE); break;
      case EV_BOX: S2O(EV_BOX); break;
      case EV_TORUS: S2O(EV_TORUS); break;
      default: S2O(EV_SEL); break;
    }
#undef S2O
  } else {
    search2d_one<B, EV>(g, f, o, L, rec, inst_key, q, pos1d, out, inst_edges, st, dst, st_lo, st_hi);
  }
}

void launch_search2d_analytic(const GridP& g, const FieldP& f, const OptP& o, const uint32_t* L,
                              RecView rec, const int64_t* inst_key, int64_t Q, const double* pos1d,
                              Stage2D out, int64_t* inst_edges, DevStats* st, DevStatus* dst, int64_t st_lo,
                              int64_t st_hi, cudaStream_t s) {
  if (!Q) return;
  const dim3 grid(grid_for(Q, 128));
#define S2A(BB, EVV) k_search2d_analytic<BB, EVV><<<grid, 128, 0, s>>>(g, f, o, L, rec, inst_key, Q, pos1d, out, \
                                                                      inst_edges, st, dst, st_lo, st_hi)
  if (g.nb) {
    S2A(true, EV_SEL);
    return;
  }
  switch (ev_mode_of(f)) {  // kernels specialised for the commonest fast paths
    case EV_SPHERE: S2A(false, EV_SPHERE); break;
    case EV_BOX: S2A(false, EV_BOX); break;
    case EV_TORUS: S2A(false, EV_TORUS); break;
    case EV_SPHERE2: S2A(false, EV_SPHERE2); break;
    case EV_BOX2F: S2A(false, EV_BOX2F); break;
    default: S2A(false, EV_PARAM); break;
  }
#undef S2A
}

// ---- lock-step 2D search (batched fields) --------------------------------
// Batch sequence per instance (search.py:220, :244-276): step 0 midpoint
// probe (Q points), steps 1..s1_lin+s1_bin the step-1 ray (Q points), then
// s2_lin+s2_bin steps of both step-2 rays in one batch of 2Q points.
struct Search2DState {
  double mid[2], dl[2], ray[2];
  double a1, b1;          // step-1 bracket
  double q2[2];
  double a2[2], b2[2];    // step-2 brackets (ray -dl, ray +dl)
  int32_t first1, first2[2];
  uint8_t mid_label, found1, found2[2], degen;
};

// In HBM the state is structure-of-arrays (14 double fields, then 4 int32
// fields, each Q long) so that every field access of a warp is one coalesced
// 256-/128-byte line; the step kernels load and store only the fields their
// phase touches.
namespace {
enum { F_MID = 0, F_DL = 2, F_RAY = 4, F_A1 = 6, F_B1 = 7, F_Q2 = 8, F_A2 = 10, F_B2 = 12, F_N = 14 };
enum { I_FIRST1 = 0, I_FIRST2 = 1, I_FLAGS = 3, I_N = 4 };
// store masks
enum : unsigned { W_GEOM = 1, W_RAY = 2, W_S1 = 4, W_Q2 = 8, W_S2 = 16, W_INT = 32, W_ALL = 63 };
struct S2View {
  double* d;
  int32_t* i;
  int64_t Q;
};
__host__ __device__ __forceinline__ S2View s2_view(void* base, int64_t Q) {
  return {(double*)base, (int32_t*)((double*)base + F_N * Q), Q};
}
__device__ __forceinline__ Search2DState s2_load(const S2View& v, int64_t q) {
  Search2DState s;
  const double* __restrict__ d = v.d;
  const int32_t* __restrict__ iw = v.i;
  const int64_t Q = v.Q;
  s.mid[0] = d[(F_MID + 0) * Q + q];
  s.mid[1] = d[(F_MID + 1) * Q + q];
  s.dl[0] = d[(F_DL + 0) * Q + q];
  s.dl[1] = d[(F_DL + 1) * Q + q];
  s.ray[0] = d[(F_RAY + 0) * Q + q];
  s.ray[1] = d[(F_RAY + 1) * Q + q];
  s.a1 = d[F_A1 * Q + q];
  s.b1 = d[F_B1 * Q + q];
  s.q2[0] = d[(F_Q2 + 0) * Q + q];
  s.q2[1] = d[(F_Q2 + 1) * Q + q];
  s.a2[0] = d[(F_A2 + 0) * Q + q];
  s.a2[1] = d[(F_A2 + 1) * Q + q];
  s.b2[0] = d[(F_B2 + 0) * Q + q];
  s.b2[1] = d[(F_B2 + 1) * Q + q];
  s.first1 = iw[I_FIRST1 * Q + q];
  s.first2[0] = iw[(I_FIRST2 + 0) * Q + q];
  s.first2[1] = iw[(I_FIRST2 + 1) * Q + q];
  const uint32_t f = (uint32_t)iw[I_FLAGS * Q + q];
  s.mid_label = (uint8_t)(f & 255u);
  s.found1 = (uint8_t)((f >> 8) & 1u);
  s.found2[0] = (uint8_t)((f >> 9) & 1u);
  s.found2[1] = (uint8_t)((f >> 10) & 1u);
  s.degen = (uint8_t)((f >> 16) & 255u);
  return s;
}
__device__ __forceinline__ void s2_store(const S2View& v, int64_t q, const Search2DState& s, unsigned w) {
  double* __restrict__ d = v.d;
  int32_t* __restrict__ iw = v.i;
  const int64_t Q = v.Q;
  if (w & W_GEOM) {
    d[(F_MID + 0) * Q + q] = s.mid[0];
    d[(F_MID + 1) * Q + q] = s.mid[1];
    d[(F_DL + 0) * Q + q] = s.dl[0];
    d[(F_DL + 1) * Q + q] = s.dl[1];
  }
  if (w & W_RAY) {
    d[(F_RAY + 0) * Q + q] = s.ray[0];
    d[(F_RAY + 1) * Q + q] = s.ray[1];
  }
  if (w & W_S1) {
    d[F_A1 * Q + q] = s.a1;
    d[F_B1 * Q + q] = s.b1;
  }
  if (w & W_Q2) {
    d[(F_Q2 + 0) * Q + q] = s.q2[0];
    d[(F_Q2 + 1) * Q + q] = s.q2[1];
  }
  if (w & W_S2) {
    d[(F_A2 + 0) * Q + q] = s.a2[0];
    d[(F_A2 + 1) * Q + q] = s.a2[1];
    d[(F_B2 + 0) * Q + q] = s.b2[0];
    d[(F_B2 + 1) * Q + q] = s.b2[1];
  }
  if (w & W_INT) {
    iw[I_FIRST1 * Q + q] = s.first1;
    iw[(I_FIRST2 + 0) * Q + q] = s.first2[0];
    iw[(I_FIRST2 + 1) * Q + q] = s.first2[1];
    iw[I_FLAGS * Q + q] = (int32_t)((uint32_t)s.mid_label | ((uint32_t)s.found1 << 8) |
                                    ((uint32_t)s.found2[0] << 9) | ((uint32_t)s.found2[1] << 10) |
                                    ((uint32_t)s.degen << 16));
  }
}
}  // namespace

size_t search2d_state_bytes(int64_t Q) { return (size_t)Q * (F_N * sizeof(double) + I_N * sizeof(int32_t)); }
int search2d_num_steps(const OptP& o) { return 1 + o.s1_lin + o.s1_bin + o.s2_lin + o.s2_bin; }

// instance pairs only (face_pairings, dualize.py:72-88) -- the fd-gradient
// mode has no 2D search to write them
__global__ void k_instance_edges(GridP g, const uint32_t* __restrict__ L, RecView rec,
                                 const int64_t* __restrict__ inst_key, int64_t Q, const double* __restrict__ pos1d,
                                 int64_t* __restrict__ inst_edges) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  Inst2D I;
  int64_t pair[2];
  decode_instance(g, L, rec, inst_key[q], pos1d, I, pair);
  inst_edges[2 * q] = pair[0];
  inst_edges[2 * q + 1] = pair[1];
}
void launch_instance_edges(const GridP& g, const uint32_t* L, RecView rec, const int64_t* inst_key, int64_t Q,
                           const double* pos1d, int64_t* inst_edges, cudaStream_t s) {
  if (Q) k_instance_edges<<<grid_for(Q, 128), 128, 0, s>>>(g, L, rec, inst_key, Q, pos1d, inst_edges);
}

__global__ void k_s2_init(GridP g, const uint32_t* __restrict__ L, RecView rec,
                          const int64_t* __restrict__ inst_key, int64_t Q, const double* __restrict__ pos1d,
                          S2View S, int64_t* __restrict__ inst_edges) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  Inst2D I;
  int64_t pair[2];
  decode_instance(g, L, rec, inst_key[q], pos1d, I, pair);
  if (inst_edges) {
    inst_edges[2 * q] = pair[0];
    inst_edges[2 * q + 1] = pair[1];
  }
  Chord ch = make_chord(I);
  Search2DState s = {};
  s.mid[0] = ch.mid[0];
  s.mid[1] = ch.mid[1];
  s.dl[0] = ch.dl[0];
  s.dl[1] = ch.dl[1];
  s.degen = ch.degen;
  s2_store(S, q, s, W_ALL);
}

// Per-instance geometry needed to lift points: recomputed from the key.
__device__ __forceinline__ void inst_frame(const GridP& g, int64_t ikey, Inst2D& I) {
  const int64_t fk = ikey >> 1;
  const int64_t vid = fk / 3;
  const int n = (int)(fk - 3 * vid);
  I.bu = n == 2 ? 0 : n + 1;
  I.bv = n == 0 ? 2 : n - 1;
  vposition(g, vid, I.org);
}

// query point of instance (I, s) at lock-step ``step`` (ray r of the two
// step-2 rays), in face coordinates (search.py:244-276)
__device__ __forceinline__ void s2_point_uv(const OptP& o, const Inst2D& I, const Search2DState& s, int step, int r,
                                            double& u, double& v) {
  const int n1 = o.s1_lin + o.s1_bin;
  if (step == 0) {
    u = s.mid[0];
    v = s.mid[1];
  } else if (step <= n1) {
    const double mr = o.s1_range * I.hmin;
    double d;
    if (step <= o.s1_lin) d = mr * ((double)step / (double)o.s1_lin);
    else d = 0.5 * (s.a1 + s.b1);
    u = s.mid[0] + d * s.ray[0];
    v = s.mid[1] + d * s.ray[1];
  } else {
    const double dir0 = r == 0 ? -s.dl[0] : s.dl[0], dir1 = r == 0 ? -s.dl[1] : s.dl[1];
    const double mr = o.s2_range * I.hmin;
    const int k = step - n1;
    double d;
    if (k <= o.s2_lin) d = mr * ((double)k / (double)o.s2_lin);
    else d = 0.5 * (r == 0 ? s.a2[0] + s.b2[0] : s.a2[1] + s.b2[1]);
    u = s.q2[0] + d * dir0;
    v = s.q2[1] + d * dir1;
  }
}
__device__ __forceinline__ void s2_frame(const GridP& g, int64_t ikey, Inst2D& I) {
  inst_frame(g, ikey, I);
  I.hu = I.bu == 0 ? g.h[0] : I.bu == 1 ? g.h[1] : g.h[2];
  I.hv = I.bv == 0 ? g.h[0] : I.bv == 1 ? g.h[1] : g.h[2];
  I.hmin = I.hu < I.hv ? I.hu : I.hv;
}

__global__ void k_s2_points(GridP g, OptP o, const int64_t* __restrict__ inst_key, int64_t Q, int step, S2View S,
                            double* __restrict__ pts) {
  int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n1 = o.s1_lin + o.s1_bin;
  const bool two = step > n1;
  const int64_t M = two ? 2 * Q : Q;
  if (m >= M) return;
  const int64_t q = two ? (m < Q ? m : m - Q) : m;
  Inst2D I;
  s2_frame(g, inst_key[q], I);
  double u, v, p[3];
  s2_point_uv(o, I, s2_load(S, q), step, m < Q ? 0 : 1, u, v);
  lift(I, u, v, p);
  pts[3 * m] = p[0];
  pts[3 * m + 1] = p[1];
  pts[3 * m + 2] = p[2];
}

// fold the labels of lock-step ``step`` into the search state (search.py:220-276);
// returns the store mask of the fields it changed.  PH: the phase of
// ``step`` when known at compile time (0, 1, 2), -1 to branch at run time.
template <int PH>
__device__ __forceinline__ unsigned s2_apply(const GridP& g, const OptP& o, const uint32_t* __restrict__ L,
                                             const int64_t* __restrict__ inst_key, int64_t Q, int64_t q, int step,
                                             const uint8_t* __restrict__ lab, Inst2D& I, Search2DState& s,
                                             DevStatus* dst, int64_t q_base) {
  const int n1 = o.s1_lin + o.s1_bin;
  if (PH == 0 || (PH < 0 && step == 0)) {
    s.mid_label = lab[q];
    // corner labels for the ray side
    const int64_t fk = inst_key[q] >> 1;
    const int64_t vid = fk / 3;
    const int64_t w1 = vid + vstep(g, I.bu), w3 = vid + vstep(g, I.bv), w2 = w1 + vstep(g, I.bv);
    I.cl[0] = label_at(L, g, vid);
    I.cl[1] = label_at(L, g, w1);
    I.cl[2] = label_at(L, g, w2);
    I.cl[3] = label_at(L, g, w3);
    Chord ch;
    ch.mid[0] = s.mid[0];
    ch.mid[1] = s.mid[1];
    ch.dl[0] = s.dl[0];
    ch.dl[1] = s.dl[1];
    ch.degen = s.degen;
    if (!ray_direction(I, ch, s.mid_label, s.ray)) raise_status(dst, ODC_E_ASSERT, q + q_base);
    s.first1 = o.s1_lin;
    s.found1 = 0;
    return W_RAY | W_INT;
  } else if (PH == 1 || (PH < 0 && step <= n1)) {
    unsigned w = W_INT;
    const double mr = o.s1_range * I.hmin;
    if (step <= o.s1_lin) {
      if (lab[q] != s.mid_label && !s.found1) {
        s.first1 = step;
        s.found1 = 1;
      }
      if (step == o.s1_lin) {
        s.a1 = mr * ((double)(s.first1 - 1) / (double)o.s1_lin);
        s.b1 = mr * ((double)s.first1 / (double)o.s1_lin);
        w |= W_S1;
      }
    } else {
      const double mm = 0.5 * (s.a1 + s.b1);
      if (lab[q] == s.mid_label) s.a1 = mm; else s.b1 = mm;
      w |= W_S1;
    }
    if (step == n1) {
      s.q2[0] = s.mid[0] + s.a1 * s.ray[0];
      s.q2[1] = s.mid[1] + s.a1 * s.ray[1];
      s.first2[0] = s.first2[1] = o.s2_lin;
      s.found2[0] = s.found2[1] = 0;
      w |= W_Q2;
    }
    return w;
  } else {
    const double mr = o.s2_range * I.hmin;
    const int k = step - n1;
#pragma unroll
    for (int r = 0; r < 2; r++) {
      const uint8_t l = lab[q + r * Q];
      if (k <= o.s2_lin) {
        if (l != s.mid_label && !s.found2[r]) {
          s.first2[r] = k;
          s.found2[r] = 1;
        }
        if (k == o.s2_lin) {
          s.a2[r] = mr * ((double)(s.first2[r] - 1) / (double)o.s2_lin);
          s.b2[r] = mr * ((double)s.first2[r] / (double)o.s2_lin);
        }
      } else {
        const double mm = 0.5 * (s.a2[r] + s.b2[r]);
        if (l == s.mid_label) s.a2[r] = mm; else s.b2[r] = mm;
      }
    }
    return (k >= o.s2_lin ? W_S2 : 0u) | (k <= o.s2_lin ? W_INT : 0u);
  }
}

__global__ void k_s2_update(GridP g, OptP o, const uint32_t* __restrict__ L, const int64_t* __restrict__ inst_key,
                            int64_t Q, int step, const uint8_t* __restrict__ lab, S2View S, DevStatus* dst,
                            int64_t q_base) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  Search2DState s = s2_load(S, q);
  Inst2D I;
  s2_frame(g, inst_key[q], I);
  s2_store(S, q, s, s2_apply<-1>(g, o, L, inst_key, Q, q, step, lab, I, s, dst, q_base));
}

// update with the labels of ``step`` and emit the query points of step + 1
// (one thread per instance, both rays in step 2): one pass over the state
// per lock-step instead of two.  PH = phase of ``step`` (0 midpoint probe,
// 1 step-1 ray, 2 step-2 rays), so the loads of fields the phase never reads
// compile away.
//
// Compacted next step (cmp.map != nullptr; the next step is a linear scan):
// an instance (ray) whose scan already flipped cannot change its state, so
// only the others get a query point -- packed at slots taken from cmp.cnt
// (one atomic per warp), with map[slot] = its label slot.  The evaluator
// reads the count on the device (PointSrc::n_dev) and writes labels through
// the map; the eval accounting keeps the reference's logical counts.
struct S2Compact {
  int32_t* map;
  int64_t* cnt;                 // count of the step being produced (zero on entry)
  int64_t* cnt_clear;           // the previous step's count: reset here for the step after
  unsigned long long* sched;    // the evaluator's pair counter for compacted batches: reset here
};
template <int PH>
__global__ void __launch_bounds__(256) k_s2_step(GridP g, OptP o, const uint32_t* __restrict__ L,
                                                 const int64_t* __restrict__ inst_key, int64_t Q, int step,
                                                 const uint8_t* __restrict__ lab, S2View S, DevStatus* dst,
                                                 double* __restrict__ pts, S2Compact cmp, int64_t q_base) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (cmp.map && q == 0) {
    *cmp.cnt_clear = 0;
    *cmp.sched = 0ull;
  }
  if (q >= Q) return;
  Search2DState s = s2_load(S, q);
  if (PH == 0) {  // fields not yet written (init leaves them zero); keep them out of the load
    s.ray[0] = s.ray[1] = s.a1 = s.b1 = s.q2[0] = s.q2[1] = 0.0;
    s.a2[0] = s.a2[1] = s.b2[0] = s.b2[1] = 0.0;
  } else if (PH == 2) {  // step-1 state is final
    s.ray[0] = s.ray[1] = s.a1 = s.b1 = 0.0;
    s.mid[0] = s.mid[1] = 0.0;
  }
  Inst2D I;
  s2_frame(g, inst_key[q], I);
  s2_store(S, q, s, s2_apply<PH>(g, o, L, inst_key, Q, q, step, lab, I, s, dst, q_base));
  const int next = step + 1;
  const int nr = next > o.s1_lin + o.s1_bin ? 2 : 1;
#pragma unroll
  for (int r = 0; r < 2; r++) {
    if (r < nr) {
      double u, v, p[3];
      s2_point_uv(o, I, s, next, r, u, v);
      lift(I, u, v, p);
      int64_t m = q + r * Q;
      if (cmp.map) {
        const bool act = nr == 1 ? !s.found1 : !(r == 0 ? s.found2[0] : s.found2[1]);
        const unsigned am = __activemask();
        const unsigned b = __ballot_sync(am, act);
        const int lane = threadIdx.x & 31, lead = __ffs(am) - 1;
        int64_t base = 0;
        if (lane == lead && b) base = (int64_t)atomicAdd((unsigned long long*)cmp.cnt, (unsigned long long)__popc(b));
        base = __shfl_sync(am, base, lead);
        if (!act) continue;
        const int64_t slot = base + __popc(b & ((1u << lane) - 1u));
        cmp.map[slot] = (int32_t)m;
        m = slot;
      }
      pts[3 * m] = p[0];
      pts[3 * m + 1] = p[1];
      pts[3 * m + 2] = p[2];
    }
  }
}

__global__ void k_s2_finish(GridP g, OptP o, const uint32_t* __restrict__ L, RecView rec,
                            const int64_t* __restrict__ inst_key, int64_t Q, const double* __restrict__ pos1d,
                            S2View S, Stage2D out, DevStats* st, int64_t st_lo, int64_t st_hi) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= Q) return;
  Inst2D I;
  int64_t pair[2];
  decode_instance(g, L, rec, inst_key[q], pos1d, I, pair);
  const Search2DState s = s2_load(S, q);
  Chord ch;
  ch.mid[0] = s.mid[0];
  ch.mid[1] = s.mid[1];
  ch.dl[0] = s.dl[0];
  ch.dl[1] = s.dl[1];
  ch.degen = s.degen;
  const double qa[2] = {s.q2[0] + s.a2[0] * -s.dl[0], s.q2[1] + s.a2[0] * -s.dl[1]};
  const double qb[2] = {s.q2[0] + s.a2[1] * s.dl[0], s.q2[1] + s.a2[1] * s.dl[1]};
  double p2d[2];
  uint8_t status;
  finish2d(I, ch, s.a1, s.found1, qa, s.found2[0], qb, s.found2[1], p2d, status);
  double p3[3];
  lift(I, p2d[0], p2d[1], p3);
  out.pos3[3 * q] = p3[0];
  out.pos3[3 * q + 1] = p3[1];
  out.pos3[3 * q + 2] = p3[2];
  if (out.pos2) {
    out.pos2[2 * q] = p2d[0];
    out.pos2[2 * q + 1] = p2d[1];
  }
  if (out.status) out.status[q] = status;
  if (out.mid) out.mid[q] = s.mid_label;
  warp_count4(st->status, status, q >= st_lo && q < st_hi);
}

void launch_search2d_lockstep_init(const GridP& g, const OptP& o, const uint32_t* L, RecView rec,
                                   const int64_t* inst_key, int64_t Q, const double* pos1d, void* state,
                                   int64_t* inst_edges, cudaStream_t s) {
  (void)o;
  if (Q) k_s2_init<<<grid_for(Q, 128), 128, 0, s>>>(g, L, rec, inst_key, Q, pos1d, s2_view(state, Q), inst_edges);
}
int64_t launch_search2d_lockstep_points(const GridP& g, const OptP& o, const int64_t* inst_key, int64_t Q, int step,
                                        const void* state, double* pts, cudaStream_t s) {
  const int n1 = o.s1_lin + o.s1_bin;
  int64_t M = step > n1 ? 2 * Q : Q;
  if (M) k_s2_points<<<grid_for(M, 128), 128, 0, s>>>(g, o, inst_key, Q, step, s2_view((void*)state, Q), pts);
  return M;
}
void launch_search2d_lockstep_update(const GridP& g, const OptP& o, const uint32_t* L, const int64_t* inst_key,
                                     int64_t Q, int step, const uint8_t* lab, void* state, DevStatus* dst,
                                     cudaStream_t s, int64_t q_base) {
  if (Q)
    k_s2_update<<<grid_for(Q, 128), 128, 0, s>>>(g, o, L, inst_key, Q, step, lab, s2_view(state, Q), dst, q_base);
}
bool search2d_step_is_linear(const OptP& o, int step) {
  const int n1 = o.s1_lin + o.s1_bin;
  return (step >= 1 && step <= o.s1_lin) || (step > n1 && step - n1 <= o.s2_lin);
}
int64_t launch_search2d_lockstep_step(const GridP& g, const OptP& o, const uint32_t* L, const int64_t* inst_key,
                                      int64_t Q, int step, const uint8_t* lab, void* state, DevStatus* dst,
                                      double* pts, cudaStream_t s, int32_t* map, int64_t* cnt2,
                                      unsigned long long* sched, int64_t q_base) {
  if (Q) {
    const int ph = step == 0 ? 0 : step <= o.s1_lin + o.s1_bin ? 1 : 2;
    const S2View v = s2_view(state, Q);
    S2Compact cmp{};
    if (map) cmp = S2Compact{map, cnt2 + ((step + 1) & 1), cnt2 + (step & 1), sched};
    if (ph == 0) k_s2_step<0><<<grid_for(Q, 256), 256, 0, s>>>(g, o, L, inst_key, Q, step, lab, v, dst, pts, cmp, q_base);
    else if (ph == 1)
      k_s2_step<1><<<grid_for(Q, 256), 256, 0, s>>>(g, o, L, inst_key, Q, step, lab, v, dst, pts, cmp, q_base);
    else k_s2_step<2><<<grid_for(Q, 256), 256, 0, s>>>(g, o, L, inst_key, Q, step, lab, v, dst, pts, cmp, q_base);
  }
  return step + 1 > o.s1_lin + o.s1_bin ? 2 * Q : Q;
}
void launch_search2d_lockstep_finish(const GridP& g, const OptP& o, const uint32_t* L, RecView rec,
                                     const int64_t* inst_key, int64_t Q, const double* pos1d, const void* state,
                                     Stage2D out, DevStats* st, int64_t st_lo, int64_t st_hi, cudaStream_t s) {
  if (Q)
    k_s2_finish<<<grid_for(Q, 128), 128, 0, s>>>(g, o, L, rec, inst_key, Q, pos1d, s2_view((void*)state, Q), out,
                                                 st, st_lo, st_hi);
}

// ===========================================================================
// fd-gradient normals (pipeline.py:126-151), ablation path
// ===========================================================================
__global__ void k_fd_points(GridP g, double step, const double* __restrict__ pos1d, int64_t K,
                            double* __restrict__ pts) {
  int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= 6 * K) return;
  const int i = (int)(m / K);
  const int64_t k = m - (int64_t)i * K;
  for (int c = 0; c < 3; c++) {
    const double e = (c == i % 3) ? step : 0.0;
    pts[3 * m + c] = i < 3 ? pos1d[3 * k + c] + e : pos1d[3 * k + c] - e;
  }
}
void launch_fd_points(const GridP& g, const OptP& o, const double* pos1d, int64_t K, double* pts, cudaStream_t s) {
  double hmin = g.h[0] < g.h[1] ? g.h[0] : g.h[1];
  hmin = hmin < g.h[2] ? hmin : g.h[2];
  if (K) k_fd_points<<<grid_for(6 * K, 256), 256, 0, s>>>(g, o.fd_step * hmin, pos1d, K, pts);
}
__global__ void k_eval_raw(FieldP f, const double* __restrict__ pts, int64_t n, double* __restrict__ raw,
                           uint8_t* __restrict__ lab) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  const double r = field_raw(f, p);
  if (raw) raw[i] = r;
  if (lab) lab[i] = r > f.iso ? 1 : 0;
}
void launch_fd_raw_analytic(const FieldP& f, const double* pts, int64_t n, double* raw, cudaStream_t s) {
  if (n) k_eval_raw<<<grid_for(n, 128), 128, 0, s>>>(f, pts, n, raw, nullptr);
}
void launch_eval_raw_analytic(const FieldP& f, const double* pts, int64_t n, double* raw, uint8_t* lab,
                              cudaStream_t s) {
  if (n) k_eval_raw<<<grid_for(n, 128), 128, 0, s>>>(f, pts, n, raw, lab);
}
__global__ void k_fd_normals(GridP g, double step, const uint32_t* __restrict__ L,
                             const int64_t* __restrict__ edge_key, int64_t K, const double* __restrict__ raw,
                             double* __restrict__ nrm, DevStats* st, int64_t st_lo, int64_t st_hi) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double gr[3], n[3];
  for (int i = 0; i < 3; i++) gr[i] = (raw[i * K + k] - raw[(i + 3) * K + k]) / (2.0 * step);
  const double nr = norm3(gr);
  EdgeGeom e = edge_geom(g, L, edge_key[k]);
  const double el = norm3(e.span);
  const bool bad = nr < 1e-30;
  const double sn = bad ? 1.0 : nr;
  for (int c = 0; c < 3; c++) n[c] = bad ? e.span[c] / el : -gr[c] / sn;
  if (einsum3(n, e.span) < 0.0)
    for (int c = 0; c < 3; c++) n[c] = -n[c];
  for (int c = 0; c < 3; c++) nrm[3 * k + c] = n[c];
  warp_count(&st->normal_fallbacks, bad && k >= st_lo && k < st_hi ? 1u : 0u);
}
void launch_fd_normals(const GridP& g, const OptP& o, const uint32_t* L, const int64_t* edge_key, int64_t K,
                       const double* raw, double* edge_normals, DevStats* st, int64_t st_lo, int64_t st_hi,
                       cudaStream_t s) {
  double hmin = g.h[0] < g.h[1] ? g.h[0] : g.h[1];
  hmin = hmin < g.h[2] ? hmin : g.h[2];
  if (K) k_fd_normals<<<grid_for(K, 128), 128, 0, s>>>(g, o.fd_step * hmin, L, edge_key, K, raw, edge_normals, st,
                                                           st_lo, st_hi);
}

// ===========================================================================
// K6: per-cell partitions (dualize.py:194-238 via the cycle table), plane
// samples + normals (dualize.py:299-317, :402-429), QEF (dualize.py:332-372)
// ===========================================================================
__constant__ int c_LE_CORNER[12] = {0, 0, 0, 1, 1, 2, 2, 3, 4, 4, 5, 6};
__constant__ int c_LE_AXIS[12] = {0, 1, 2, 1, 2, 0, 2, 2, 0, 1, 1, 0};
__constant__ int c_LF_CORNER[6] = {0, 0, 0, 1, 2, 4};
__constant__ int c_LF_NORMAL[6] = {0, 1, 2, 0, 1, 2};

__device__ __forceinline__ int64_t cell_base_vid(const GridP& g, int64_t cell) {
  const int64_t x = imod(cell, g.R), y = imod(idiv(cell, g.R), g.R), z = idiv(cell, g.R * g.R);
  return x + y * g.S + z * g.S2;
}
__device__ __forceinline__ int64_t corner_off(const GridP& g, int c) {
  return (int64_t)(c & 1) + ((c >> 1) & 1) * g.S + ((c >> 2) & 1) * g.S2;
}

__global__ void k_cell_config(GridP g, const uint32_t* __restrict__ L, RecView rec,
                              const int64_t* __restrict__ cell_id, int64_t C, const CellTabEntry* __restrict__ table,
                              uint16_t* __restrict__ cfg_out, uint32_t* __restrict__ ncyc,
                              uint32_t* __restrict__ nsamp) {
  int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ci >= C) return;
  const int64_t cell = cell_id[ci];
  const int64_t x = imod(cell, g.R), y = imod(idiv(cell, g.R), g.R), z = idiv(cell, g.R * g.R);
  uint32_t cfg = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) cfg |= label_c(L, g, x + (i & 1), y + ((i >> 1) & 1), z + ((i >> 2) & 1)) << i;
  uint32_t cm = 0;
#pragma unroll
  for (int f = 0; f < 6; f++) {
    const int fc = f < 3 ? 0 : (f == 3 ? 1 : (f == 4 ? 2 : 4));  // c_LF_CORNER
    const int64_t cx = x + (fc & 1);
    const WordRec* r = rec_find(rec, word_of(g, cx, y + ((fc >> 1) & 1), z + ((fc >> 2) & 1)));
    if (r) cm |= ((r->cf[f % 3] >> (cx & 31)) & 1u) << f;  // inactive word: no 4-crossing face
  }
  const uint32_t idx = (cfg << 6) | cm;
  const CellTabEntry& T = table[idx];
  cfg_out[ci] = (uint16_t)idx;
  ncyc[ci] = T.ncyc;
  nsamp[ci] = T.nedge;
}

void launch_cell_config(const GridP& g, const uint32_t* L, RecView rec, const int64_t* cell_id, int64_t C,
                        const CellTabEntry* table, uint16_t* cfg, uint32_t* ncyc, uint32_t* nsamp, cudaStream_t s) {
  if (C) k_cell_config<<<grid_for(C, 128), 128, 0, s>>>(g, L, rec, cell_id, C, table, cfg, ncyc, nsamp);
}

constexpr int kSolveBlock = 128;
// K6 runs in two kernels.  k_cell_samples (one thread per cell) walks the
// cell's cycles through the table and writes every plane sample's normal
// (dualize.py:299-317) and 1D-point row, in sample order, plus each
// partition's first sample; k_part_solve (one thread per partition) sums
// its samples and solves the QEF (dualize.py:332-372).  One kernel holding a
// cycle's samples in per-thread arrays kept them in local memory (≈3.9 GB of
// DRAM traffic at 1024³) and the LAPACK restatement's divergence behind
// them; here each sample is written once and re-read from L1/L2, and the
// solve runs one partition per thread with no per-thread arrays.
template <bool B>
__global__ void __launch_bounds__(kSolveBlock) k_cell_samples(GridP g, OptP o, const uint32_t* __restrict__ L,
                                                      RecView rec, const int64_t* __restrict__ cell_id, int64_t C,
                                                      const CellTabEntry* __restrict__ table,
                                                      const uint16_t* __restrict__ cfg,
                                                      const uint32_t* __restrict__ part_base,
                                                      const uint32_t* __restrict__ samp_base,
                                                      const double* __restrict__ pos1d,
                                                      const double* __restrict__ pos3,
                                                      const double* __restrict__ edge_normals, CellOut out,
                                                      double* __restrict__ snorm, int32_t* __restrict__ srow,
                                                      uint32_t* __restrict__ psoff, DevStats* st, int64_t st_lo,
                                                      int64_t st_hi) {
  int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ci >= C) return;
  const int64_t cell = cell_id[ci];
  const int64_t cc[3] = {imod(cell, g.R), imod(idiv(cell, g.R), g.R), idiv(cell, g.R * g.R)};
  if constexpr (B) st += localize<B>(g, cc[2]);  // batch: this cell's shape geometry (g is the kernel's copy)
  const CellTabEntry T = table[cfg[ci]];
  const int64_t pbase = part_base[ci];
  const int64_t sbase = samp_base[ci];
  out.pinfo[ci] = ((uint64_t)pbase << 24) | T.cyc_of_edge;
  double hmin = g.h[0] < g.h[1] ? g.h[0] : g.h[1];
  hmin = hmin < g.h[2] ? hmin : g.h[2];
  uint32_t nfb = 0;
  int slot = 0;
  // instance id of the cycle's j-th instance (instance j joins edge j and j+1)
  auto iid = [&](int j) -> int64_t {
    const int code = (int)((T.insts >> (4 * (slot + j))) & 15);
    const int f = code >> 1, s = code & 1;
    const int fc = c_LF_CORNER[f];
    return inst_rank_c(rec, g, cc[0] + (fc & 1), cc[1] + ((fc >> 1) & 1), cc[2] + ((fc >> 2) & 1), c_LF_NORMAL[f]) +
           s;
  };
  for (int k = 0; k < T.ncyc; k++) {
    const int len = (T.lens >> (4 * k)) & 15;
    const int64_t pid = pbase + k;
    psoff[pid] = (uint32_t)(sbase + slot);
    out.part_cell[pid] = cell;
    out.part_index[pid] = k;
    if (out.cyc_len) out.cyc_len[pid] = len;
    int64_t ia = len > 0 ? iid(len - 1) : 0;  // instance before edge 0 (cyclic)
    for (int j = 0; j < len; j++) {
      const int64_t ib = iid(j);
      const int le = (int)((T.edges >> (4 * (slot + j))) & 15);
      const int ec = c_LE_CORNER[le];
      const int ax = c_LE_AXIS[le];
      const int64_t ex = cc[0] + (ec & 1), ey = cc[1] + ((ec >> 1) & 1), ez = cc[2] + ((ec >> 2) & 1);
      const int64_t row = edge_rank_c(rec, g, ex, ey, ez, ax);
      const int64_t sj = sbase + slot + j;
      srow[sj] = (int32_t)row;
      if (out.cyc_edges) {
        out.cyc_edges[sj] = (ex + ey * g.S + ez * g.S2) * 3 + ax;
        out.cyc_insts[sj] = ib;
      }
      double n[3];
      if (o.normals == ODC_NORMALS_2D) {
        // estimate_normals (dualize.py:299-317), edge direction p_out - p_in (dualize.py:421-423)
        double pj[3], pi[3], po[3], ed[3];
        for (int c = 0; c < 3; c++) pj[c] = pos1d[3 * row + c];
        const bool base_in = label_c(L, g, ex, ey, ez) == 1u;
        const int64_t ox = ex + (ax == 0), oy = ey + (ax == 1), oz = ez + (ax == 2);  // the edge's other end
        vposition_c(g, base_in ? ex : ox, base_in ? ey : oy, base_in ? ez : oz, pi);
        vposition_c(g, base_in ? ox : ex, base_in ? oy : ey, base_in ? oz : ez, po);
        for (int c = 0; c < 3; c++) ed[c] = po[c] - pi[c];
        double da[3], db[3];
        for (int c = 0; c < 3; c++) {
          da[c] = pos3[3 * ia + c] - pj[c];
          db[c] = pos3[3 * ib + c] - pj[c];
        }
        cross3(da, db, n);
        const double nr = norm3(n);
        const bool fb = nr <= 1e-9 * hmin * hmin;
        const double el = norm3(ed);
        const double safe = fb ? 1.0 : nr;
        for (int c = 0; c < 3; c++) n[c] = n[c] / safe;
        if (fb) {
          for (int c = 0; c < 3; c++) n[c] = ed[c] / el;
          nfb++;
        }
        if (einsum3(n, ed) < 0.0)
          for (int c = 0; c < 3; c++) n[c] = -n[c];
      } else {
        for (int c = 0; c < 3; c++) n[c] = edge_normals[3 * row + c];
      }
      for (int c = 0; c < 3; c++) snorm[3 * sj + c] = n[c];
      ia = ib;
    }
    slot += len;
  }
  if (ci == C - 1) psoff[pbase + T.ncyc] = (uint32_t)(sbase + slot);  // psoff[P] = Ns
  warp_count<B>(&st->normal_fallbacks, ci >= st_lo && ci < st_hi ? (unsigned)nfb : 0u);
}

// solve_qef_batch (dualize.py:332-372) of partition pid: sums sequential in
// cycle order, then np.linalg.eigh (LAPACK dsyevd bit for bit), the
// truncated pseudo-inverse, the clip to the cell, the residual
template <bool B>
__global__ void __launch_bounds__(kSolveBlock, 8) k_part_solve(GridP g, OptP o, int64_t P,
                                                    const double* __restrict__ pos1d,
                                                    const double* __restrict__ snorm,
                                                    const int32_t* __restrict__ srow,
                                                    const uint32_t* __restrict__ psoff, CellOut out, DevStats* st,
                                                    int64_t own_lo, int64_t own_hi) {
  const int64_t pid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pid >= P) return;
  const int64_t s0 = psoff[pid];
  const int len = (int)(psoff[pid + 1] - s0);
  const int64_t cell = out.part_cell[pid];
  const int64_t cc[3] = {imod(cell, g.R), imod(idiv(cell, g.R), g.R), idiv(cell, g.R * g.R)};
  if constexpr (B) st += localize<B>(g, cc[2]);
#define PE(j, c) __ldg(pos1d + 3 * (int64_t)srow[s0 + (j)] + (c))
#define NN(j, c) snorm[3 * (s0 + (j)) + (c)]
  const double cnt = (double)(len < 1 ? 1 : len);
  double cen[3] = {0.0, 0.0, 0.0};
#pragma unroll 4
  for (int j = 0; j < len; j++)
    for (int c = 0; c < 3; c++) cen[c] += PE(j, c);
  for (int c = 0; c < 3; c++) cen[c] /= cnt;
  double A[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, b[3] = {0.0, 0.0, 0.0};
#pragma unroll 4
  for (int j = 0; j < len; j++) {  // A and b accumulate independently, each in cycle order
    const double nj[3] = {NN(j, 0), NN(j, 1), NN(j, 2)};
    for (int r = 0; r < 3; r++)
      for (int c = 0; c < 3; c++) A[3 * r + c] += nj[r] * nj[c];
    const double d[3] = {PE(j, 0) - cen[0], PE(j, 1) - cen[1], PE(j, 2) - cen[2]};
    const double off = einsum3(nj, d);
    for (int c = 0; c < 3; c++) b[c] += nj[c] * off;
  }
  double w[3], V[9];
  odc_eigh3(A, w, V);  // np.linalg.eigh (dualize.py:358), LAPACK dsyevd bit for bit
  double sv[3];
  for (int kk = 0; kk < 3; kk++) sv[kk] = sqrt(w[kk] > 0.0 ? w[kk] : 0.0);
  const double smax = sv[2];
  const double thr = o.qef_trunc * (smax > 1e-300 ? smax : 1e-300);
  bool keep[3];
  int rank = 0;
  for (int kk = 0; kk < 3; kk++) {
    keep[kk] = (sv[kk] >= thr) && (smax > 0.0);
    rank += keep[kk];
  }
  double coef[3], y[3], sol[3];
  for (int j = 0; j < 3; j++) coef[j] = (V[j] * b[0] + V[3 + j] * b[1]) + V[6 + j] * b[2];
  for (int j = 0; j < 3; j++) y[j] = keep[j] ? coef[j] / w[j] : 0.0;
  for (int i = 0; i < 3; i++) sol[i] = (V[3 * i] * y[0] + V[3 * i + 2] * y[2]) + V[3 * i + 1] * y[1];
  double pos[3];
  for (int c = 0; c < 3; c++) {
    const double blo = gpos(g, c, cc[c]);  // cell_bounds (grid.py:89-91): lo + i h
    const double bhi = blo + g.h[c];
    double x = cen[c] + sol[c];
    x = x > blo ? x : blo;  // np.clip
    x = x < bhi ? x : bhi;
    pos[c] = x;
  }
  double res = 0.0;
#pragma unroll 4
  for (int j = 0; j < len; j++) {
    const double nj[3] = {NN(j, 0), NN(j, 1), NN(j, 2)};
    const double d[3] = {pos[0] - PE(j, 0), pos[1] - PE(j, 1), pos[2] - PE(j, 2)};
    const double e = einsum3(nj, d);
    res += e * e;
  }
#undef PE
#undef NN
  for (int c = 0; c < 3; c++) out.verts[3 * pid + c] = pos[c];
  if (out.rank) out.rank[pid] = rank;
  if (out.resid) out.resid[pid] = res;
  const bool own = pid >= own_lo && pid < own_hi;
  warp_count4<B>(st->rank, rank, own);
  warp_max_nonneg_double<B>(&st->max_resid_bits, own && !(res <= 0.0) ? res : 0.0);  // NaN wins
}

void launch_cell_solve(const GridP& g, const OptP& o, const uint32_t* L, RecView rec, const int64_t* cell_id,
                       int64_t C, const CellTabEntry* table, const uint16_t* cfg, const uint32_t* part_base,
                       const uint32_t* samp_base, const double* pos1d, const double* pos3, const double* edge_normals,
                       CellOut out, double* snorm, int32_t* srow, uint32_t* psoff, int64_t P, DevStats* st,
                       int64_t st_lo, int64_t st_hi, int64_t own_lo, int64_t own_hi, cudaStream_t s) {
  if (!C) return;
  if (g.nb) {
    k_cell_samples<true><<<grid_for(C, kSolveBlock), kSolveBlock, 0, s>>>(
        g, o, L, rec, cell_id, C, table, cfg, part_base, samp_base, pos1d, pos3, edge_normals, out, snorm, srow,
        psoff, st, st_lo, st_hi);
    if (P) k_part_solve<true><<<grid_for(P, kSolveBlock), kSolveBlock, 0, s>>>(g, o, P, pos1d, snorm, srow, psoff,
                                                                              out, st, own_lo, own_hi);
  } else {
    k_cell_samples<false><<<grid_for(C, kSolveBlock), kSolveBlock, 0, s>>>(
        g, o, L, rec, cell_id, C, table, cfg, part_base, samp_base, pos1d, pos3, edge_normals, out, snorm, srow,
        psoff, st, st_lo, st_hi);
    if (P) k_part_solve<false><<<grid_for(P, kSolveBlock), kSolveBlock, 0, s>>>(g, o, P, pos1d, snorm, srow, psoff,
                                                                               out, st, own_lo, own_hi);
  }
}

// generic multi-channel exclusive scan over u32 arrays (<= 2 channels)
struct ScanPtrs {
  const uint32_t* in[2];
  uint32_t* out[2];
};
// Reduce-then-scan over tiles of kScanPer x kScanBlock elements: each
// thread owns kScanPer consecutive elements (a serial prefix in registers),
// so the single-block tile scan sees 8x fewer tiles.
constexpr int kScanPer = 8;
constexpr int64_t kScanTile = (int64_t)kScanBlock * kScanPer;
template <int NCH>
__global__ void __launch_bounds__(kScanBlock) k_reduce_u32(ScanPtrs p, int64_t n, uint32_t* sums, int64_t ntiles) {
  __shared__ uint32_t part[NCH][kScanBlock / 32];
  const int64_t i0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPer;
  uint32_t v[NCH];
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    v[c] = 0u;
#pragma unroll
    for (int k = 0; k < kScanPer; k++) v[c] += i0 + k < n ? p.in[c][i0 + k] : 0u;
    v[c] = __reduce_add_sync(0xffffffffu, v[c]);
    if ((threadIdx.x & 31) == 0) part[c][threadIdx.x >> 5] = v[c];
  }
  __syncthreads();
  if (threadIdx.x < NCH) {
    uint32_t t = 0;
    for (int w = 0; w < kScanBlock / 32; w++) t += part[threadIdx.x][w];
    sums[threadIdx.x * ntiles + blockIdx.x] = t;
  }
}
template <int NCH>
__global__ void __launch_bounds__(kScanBlock) k_apply_u32(ScanPtrs p, int64_t n, const uint32_t* sums,
                                                          int64_t ntiles) {
  const int64_t i0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPer;
  uint32_t x[NCH][kScanPer], v[NCH], ex[NCH], tot[NCH];
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    v[c] = 0u;
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
      x[c][k] = i0 + k < n ? p.in[c][i0 + k] : 0u;
      v[c] += x[c][k];
    }
  }
  block_exscan<NCH>(v, ex, tot);
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    uint32_t run = sums[c * ntiles + blockIdx.x] + ex[c];
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
      if (i0 + k < n) p.out[c][i0 + k] = run;
      run += x[c][k];
    }
  }
}
// Small arrays (<= kScanSmallMax = one pass of 1,024 threads x 8): one block,
// one launch instead of three -- what dominates the scans of a small grid is
// launch latency, not bandwidth.  A single block walking more tiles with a
// running carry is slower than the three launches (63 K elements: 48-90 us
// against ~15 us), so larger arrays take the tiled path.
constexpr int kScanSmallBlock = 1024;
constexpr int64_t kScanSmallMax = (int64_t)kScanSmallBlock * kScanPer;
template <int NCH>
__global__ void __launch_bounds__(kScanSmallBlock) k_scan_small(ScanPtrs p, int64_t n, unsigned long long* totals) {
  unsigned long long carry[NCH];
#pragma unroll
  for (int c = 0; c < NCH; c++) carry[c] = 0ull;
  for (int64_t base = 0; base < n; base += (int64_t)kScanSmallBlock * kScanPer) {
    const int64_t i0 = base + (int64_t)threadIdx.x * kScanPer;
    uint32_t x[NCH][kScanPer], v[NCH], ex[NCH], tot[NCH];
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      v[c] = 0u;
#pragma unroll
      for (int k = 0; k < kScanPer; k++) {
        x[c][k] = i0 + k < n ? p.in[c][i0 + k] : 0u;
        v[c] += x[c][k];
      }
    }
    block_exscan<NCH, kScanSmallBlock>(v, ex, tot);
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      uint32_t run = (uint32_t)carry[c] + ex[c];
#pragma unroll
      for (int k = 0; k < kScanPer; k++) {
        if (i0 + k < n) p.out[c][i0 + k] = run;
        run += x[c][k];
      }
      carry[c] += tot[c];
    }
  }
  if (threadIdx.x < NCH) totals[threadIdx.x] = carry[threadIdx.x];
}

// Single-pass scan with decoupled look-back: each tile publishes its
// aggregate, then one warp per channel walks back over its predecessors'
// published words, 32 at a time, until one carries an inclusive prefix, and
// publishes its own (a one-thread walk serialises long tile chains: 2,000
// tiles took longer than the three-launch scan).  One word per
// (channel, tile): epoch (30 bits) | flag (2 bits: 1 aggregate, 2 inclusive)
// | value (32 bits -- the outputs are u32 prefixes).  The epoch is a
// per-context counter bumped every scan, so the status array is never
// cleared: a word from an earlier scan has another epoch and reads as "not
// yet published".  Tiles wait only on lower-indexed tiles, which the
// hardware dispatches first.
template <int NCH>
__global__ void __launch_bounds__(kScanBlock) k_scan_lookback(ScanPtrs p, int64_t n,
                                                              unsigned long long* __restrict__ status,
                                                              int64_t ntiles, uint32_t epoch,
                                                              unsigned long long* __restrict__ totals) {
  __shared__ uint32_t s_excl[NCH];
  const int64_t t = blockIdx.x;
  const int64_t i0 = t * kScanTile + (int64_t)threadIdx.x * kScanPer;
  uint32_t x[NCH][kScanPer], v[NCH], ex[NCH], tot[NCH];
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    v[c] = 0u;
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
      x[c][k] = i0 + k < n ? p.in[c][i0 + k] : 0u;
      v[c] += x[c][k];
    }
  }
  block_exscan<NCH>(v, ex, tot);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < NCH) {  // warp c publishes channel c and looks back 32 tiles per step
    const int c = warp;
    volatile unsigned long long* st = status + (int64_t)c * ntiles;
    const unsigned long long tag = (unsigned long long)epoch << 34;
    if (lane == 0) st[t] = tag | ((t == 0 ? 2ull : 1ull) << 32) | tot[c];  // aggregate (tile 0: inclusive)
    uint32_t excl = 0;
    if (t > 0) {
      int64_t base = t - 1;  // the predecessor lane 0 reads
      while (true) {
        const int64_t j = base - lane;
        // before tile 0: an inclusive prefix of 0
        const unsigned long long w = j >= 0 ? st[j] : (tag | (2ull << 32));
        const unsigned flag = (w >> 34) == epoch ? (unsigned)((w >> 32) & 3ull) : 0u;
        const unsigned pub = __ballot_sync(0xffffffffu, flag != 0u);
        const unsigned inc = __ballot_sync(0xffffffffu, flag == 2u);
        const int k = inc ? __ffs(inc) - 1 : 31;  // lanes 0..k are needed
        const unsigned need = k == 31 ? 0xffffffffu : ((2u << k) - 1u);
        if ((pub & need) != need) continue;  // a needed predecessor has not published yet
        uint32_t val = lane <= k ? (uint32_t)w : 0u;
        val = __reduce_add_sync(0xffffffffu, val);
        excl += val;
        if (inc) break;
        base -= 32;
      }
      if (lane == 0) st[t] = tag | (2ull << 32) | (uint32_t)(excl + tot[c]);
    }
    if (lane == 0) {
      s_excl[c] = excl;
      if (t == ntiles - 1) totals[c] = (unsigned long long)excl + tot[c];
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    uint32_t run = s_excl[c] + ex[c];
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
      if (i0 + k < n) p.out[c][i0 + k] = run;
      run += x[c][k];
    }
  }
}

int launch_scan_lookback(const uint32_t* const* in, uint32_t* const* out, int nch, int64_t n,
                         unsigned long long* status, uint32_t epoch, unsigned long long* totals, cudaStream_t s) {
  ScanPtrs p{};
  for (int c = 0; c < nch; c++) {
    p.in[c] = in[c];
    p.out[c] = out[c];
  }
  const int64_t nt = (n + kScanTile - 1) / kScanTile;
  if (nt == 0) {
    cudaMemsetAsync(totals, 0, sizeof(unsigned long long) * nch, s);
    return 0;
  }
  if (n <= kScanSmallMax) {
    if (nch == 1) k_scan_small<1><<<1, kScanSmallBlock, 0, s>>>(p, n, totals);
    else k_scan_small<2><<<1, kScanSmallBlock, 0, s>>>(p, n, totals);
    return 1;
  }
  if (nch == 1) k_scan_lookback<1><<<(unsigned)nt, kScanBlock, 0, s>>>(p, n, status, nt, epoch, totals);
  else k_scan_lookback<2><<<(unsigned)nt, kScanBlock, 0, s>>>(p, n, status, nt, epoch, totals);
  return 1;
}
int64_t scan_lookback_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }

int launch_scan_u32(const uint32_t* const* in, uint32_t* const* out, int nch, int64_t n, uint32_t* tile_buf,
                    unsigned long long* totals, cudaStream_t s) {
  ScanPtrs p{};
  for (int c = 0; c < nch; c++) {
    p.in[c] = in[c];
    p.out[c] = out[c];
  }
  const int64_t nt = (n + kScanTile - 1) / kScanTile;
  if (nt == 0) {
    cudaMemsetAsync(totals, 0, sizeof(unsigned long long) * nch, s);
    return 0;
  }
  if (n <= kScanSmallMax) {
    if (nch == 1) k_scan_small<1><<<1, kScanSmallBlock, 0, s>>>(p, n, totals);
    else k_scan_small<2><<<1, kScanSmallBlock, 0, s>>>(p, n, totals);
    return 1;
  }
  if (nch == 1) {
    k_reduce_u32<1><<<(unsigned)nt, kScanBlock, 0, s>>>(p, n, tile_buf, nt);
    k_scan_tiles<1><<<1, 1024, 0, s>>>(tile_buf, nt, totals);
    k_apply_u32<1><<<(unsigned)nt, kScanBlock, 0, s>>>(p, n, tile_buf, nt);
  } else {
    k_reduce_u32<2><<<(unsigned)nt, kScanBlock, 0, s>>>(p, n, tile_buf, nt);
    k_scan_tiles<2><<<1, 1024, 0, s>>>(tile_buf, nt, totals);
    k_apply_u32<2><<<(unsigned)nt, kScanBlock, 0, s>>>(p, n, tile_buf, nt);
  }
  return 3;
}

// ===========================================================================
// K7: polygonization (polygonize.py:110-217)
// ===========================================================================
__constant__ int8_t c_le_of[8][3] = {{0, 1, 2}, {-1, 3, 4}, {5, -1, 6}, {-1, -1, 7},
                                     {8, 9, -1}, {-1, 10, -1}, {11, -1, -1}, {-1, -1, -1}};

template <bool B>
__global__ void __launch_bounds__(128) k_poly_classify(GridP g, OptP o, const uint32_t* __restrict__ L,
                                                       RecView rec,
                                                       const int64_t* __restrict__ edge_key, int64_t K,
                                                       const uint64_t* __restrict__ pinfo,
                                                       const double* __restrict__ verts, int4* __restrict__ pid4,
                                                       uint8_t* __restrict__ kase, uint32_t* __restrict__ ntri,
                                                       uint32_t* __restrict__ nfan, DevStats* st) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int64_t key = edge_key[k], vid = key / 3;
  const int a = (int)(key % 3), b = (a + 1) % 3, c = (a + 2) % 3;
  int64_t vc[3];
  vid_coords(g, vid, vc);
  if constexpr (B) st += localize<B>(g, vc[2]);  // batch: this edge's shape (g is the kernel's copy)
  const bool fwd = label_at(L, g, vid) == 1u;  // v_in == edge_vertex
  const int RING[4][2] = {{-1, -1}, {0, -1}, {0, 0}, {-1, 0}};
  int pid[4];
  bool ok = true;
  for (int j = 0; j < 4; j++) {
    const int rj = fwd ? j : 3 - j;
    int64_t cc[3] = {vc[0], vc[1], vc[2]};
    cc[b] += RING[rj][0];
    cc[c] += RING[rj][1];
    for (int t = 0; t < 3; t++)
      if ((t == 2 && B ? cc[t] - g.zoff : cc[t]) < 0 || (t == 2 && B ? cc[t] - g.zoff : cc[t]) >= g.R) ok = false;
    if (!ok) break;
    const int64_t cbase = cc[0] + cc[1] * g.S + cc[2] * g.S2;
    const int64_t crow = cell_rank(rec, g, cbase);
    const uint64_t pi = pinfo[crow];
    const int corner = (int)(vc[0] - cc[0]) | ((int)(vc[1] - cc[1]) << 1) | ((int)(vc[2] - cc[2]) << 2);
    const int le = c_le_of[corner][a];
    const int cyc = (int)((pi >> (2 * le)) & 3u);
    pid[j] = (int)((pi >> 24) + cyc);
  }
  if (!ok) {
    kase[k] = 0;
    ntri[k] = 0;
    nfan[k] = 0;
    atomicAdd(&st->skipped, 1ull);
    return;
  }
  int cs = 1;
  if (o.split == ODC_SPLIT_IC) {
    // _concavity (polygonize.py:47-75)
    double pin[3], pout[3];
    const int64_t other = vid + vstep(g, a);
    vposition(g, fwd ? vid : other, pin);
    vposition(g, fwd ? other : vid, pout);
    double q[4][3];
    for (int j = 0; j < 4; j++)
      for (int t = 0; t < 3; t++) q[j][t] = verts[3 * (int64_t)pid[j] + t];
    bool conc[4];
    for (int kk = 0; kk < 4; kk++) {
      const double* pk = q[kk];
      const double* da = q[(kk + 3) & 3];
      const double* db = q[(kk + 1) & 3];
      double u[3], v[3], w[3], x[3];
      for (int t = 0; t < 3; t++) {
        u[t] = da[t] - pout[t];
        v[t] = db[t] - pout[t];
        w[t] = pk[t] - pout[t];
      }
      cross3(u, v, x);
      const bool plus = einsum3(w, x) < 0.0;
      for (int t = 0; t < 3; t++) {
        u[t] = da[t] - pin[t];
        v[t] = db[t] - pin[t];
        w[t] = pk[t] - pin[t];
      }
      cross3(u, v, x);
      const bool minus = einsum3(w, x) > 0.0;
      conc[kk] = plus || minus;
    }
    if (!(conc[1] || conc[3])) cs = 1;
    else if (!(conc[0] || conc[2])) cs = 2;
    else cs = 3;
  }
  pid4[k] = make_int4(pid[0], pid[1], pid[2], pid[3]);
  kase[k] = (uint8_t)cs;
  ntri[k] = cs == 3 ? 4u : 2u;
  nfan[k] = cs == 3 ? 1u : 0u;
  warp_count4<B>(st->split, cs, true);
}

void launch_poly_classify(const GridP& g, const OptP& o, const uint32_t* L, RecView rec,
                          const int64_t* edge_key, int64_t K, const uint64_t* pinfo, const double* verts, int4* pid4,
                          uint8_t* kase, uint32_t* ntri, uint32_t* nfan, DevStats* st, cudaStream_t s) {
  if (!K) return;
  if (g.nb)
    k_poly_classify<true><<<grid_for(K, 128), 128, 0, s>>>(g, o, L, rec, edge_key, K, pinfo, verts, pid4, kase, ntri,
                                                           nfan, st);
  else
    k_poly_classify<false><<<grid_for(K, 128), 128, 0, s>>>(g, o, L, rec, edge_key, K, pinfo, verts, pid4, kase, ntri,
                                                            nfan, st);
}

__global__ void k_poly_emit(int64_t K, int64_t P, const int64_t* __restrict__ edge_key, const int4* __restrict__ pid4,
                            const uint8_t* __restrict__ kase, const uint32_t* __restrict__ tri_off,
                            const uint32_t* __restrict__ fan_rank, const double* __restrict__ pos1d,
                            double* __restrict__ verts, int32_t* __restrict__ tris, int64_t* __restrict__ fan_edge,
                            uint8_t* __restrict__ used) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int cs = kase[k];
  if (cs == 0) return;
  const int4 p = pid4[k];
  int32_t* t = tris + 3 * (int64_t)tri_off[k];
  if (cs == 1) {
    t[0] = p.x; t[1] = p.y; t[2] = p.z;
    t[3] = p.x; t[4] = p.z; t[5] = p.w;
  } else if (cs == 2) {
    t[0] = p.x; t[1] = p.y; t[2] = p.w;
    t[3] = p.y; t[4] = p.z; t[5] = p.w;
  } else {
    const int64_t fr = fan_rank[k];
    const int32_t fv = (int32_t)(P + fr);
    const int q[4] = {p.x, p.y, p.z, p.w};
    for (int j = 0; j < 4; j++) {
      t[3 * j] = fv;
      t[3 * j + 1] = q[j];
      t[3 * j + 2] = q[(j + 1) & 3];
    }
    for (int c = 0; c < 3; c++) verts[3 * (P + fr) + c] = pos1d[3 * k + c];
    fan_edge[fr] = edge_key[k];
  }
  used[p.x] = 1;
  used[p.y] = 1;
  used[p.z] = 1;
  used[p.w] = 1;
}

void launch_poly_emit(int64_t K, int64_t P, const int64_t* edge_key, const int4* pid4, const uint8_t* kase,
                      const uint32_t* tri_off, const uint32_t* fan_rank, const double* pos1d, double* verts,
                      int32_t* tris, int64_t* fan_edge, uint8_t* used, cudaStream_t s) {
  if (K)
    k_poly_emit<<<grid_for(K, 256), 256, 0, s>>>(K, P, edge_key, pid4, kase, tri_off, fan_rank, pos1d, verts, tris,
                                                 fan_edge, used);
}

// used flags are 0/1 bytes: 16 per thread per step (the arena aligns to
// 256 B), one atomic per block (a same-address atomic per warp serialised
// in L2: 75 us for 3.5 M flags)
__global__ void __launch_bounds__(256) k_count_used(const uint8_t* __restrict__ used, int64_t P, DevStats* st) {
  __shared__ uint32_t part[8];
  uint32_t v = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 16;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; i < P; i += stride) {
    if (i + 16 <= P) {
      const uint4 w = *reinterpret_cast<const uint4*>(used + i);
      v += __popc(w.x & 0x01010101u) + __popc(w.y & 0x01010101u) + __popc(w.z & 0x01010101u) +
           __popc(w.w & 0x01010101u);
    } else {
      for (int64_t j = i; j < P; j++) v += used[j] ? 1u : 0u;
    }
  }
  v = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; w++) t += part[w];
    if (t) atomicAdd(&st->used_partitions, (unsigned long long)t);
  }
}
void launch_count_used(const uint8_t* used, int64_t P, DevStats* st, cudaStream_t s) {
  if (!P) return;
  const int64_t blocks = std::min<int64_t>((P + 256 * 16 - 1) / (256 * 16), 148 * 8);
  k_count_used<<<(unsigned)blocks, 256, 0, s>>>(used, P, st);
}

// drop unreferenced partition vertices (polygonize.py:199-209)
__global__ void k_remap_tris(int64_t T, const uint32_t* __restrict__ new_id, int32_t* __restrict__ tris) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * T) return;
  tris[i] = (int32_t)new_id[tris[i]];
}
__global__ void k_compact_verts(int64_t V, const uint8_t* __restrict__ used, const uint32_t* __restrict__ new_id,
                                const double* __restrict__ vin, double* __restrict__ vout,
                                int64_t* __restrict__ src_of) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V || !used[i]) return;
  const int64_t j = new_id[i];
  for (int c = 0; c < 3; c++) vout[3 * j + c] = vin[3 * i + c];
  src_of[j] = i;
}
void launch_remap_vertices(int64_t V, int64_t T, const uint8_t* used, const uint32_t* new_id, const double* v_in,
                           double* v_out, int32_t* tris, int64_t* src_of, cudaStream_t s) {
  if (V) k_compact_verts<<<grid_for(V, 256), 256, 0, s>>>(V, used, new_id, v_in, v_out, src_of);
  if (T) k_remap_tris<<<grid_for(3 * T, 256), 256, 0, s>>>(T, new_id, tris);
}

__global__ void k_split_cases(int64_t K, const uint8_t* __restrict__ kase, const uint32_t* __restrict__ rank,
                              int64_t* __restrict__ out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K || kase[k] == 0) return;
  out[rank[k]] = kase[k];
}
void launch_split_cases(int64_t K, const uint8_t* kase, int64_t* out, uint32_t* rank, cudaStream_t s) {
  if (K) k_split_cases<<<grid_for(K, 256), 256, 0, s>>>(K, kase, rank, out);
}
__global__ void k_interior_flags(int64_t K, const uint8_t* __restrict__ kase, uint32_t* __restrict__ flag) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < K) flag[k] = kase[k] != 0;
}
void launch_interior_flags(int64_t K, const uint8_t* kase, uint32_t* flag, cudaStream_t s) {
  if (K) k_interior_flags<<<grid_for(K, 256), 256, 0, s>>>(K, kase, flag);
}

// ===========================================================================
// K8: repair_nonmanifold (polygonize.py:220-374).  Per vertex: its incident
// triangles (ascending), the edges (v,u) to its neighbours with their
// triangle lists (every triangle on edge (v,u) contains v, so the local count
// is the global count), sheet pairing of >2-triangle edges by dihedral angle
// (polygonize.py:279-305) and union-find over incident triangles
// (polygonize.py:308-347).  Extra components get new vertex ids in vertex
// order (polygonize.py:348-358).
// ===========================================================================
constexpr int kMaxFan = 64;

// Vertex -> incident-triangle CSR.  dirty (repair passes after the first):
// only the fans of flagged vertices, the only ones the pass examines.
// T_dev: the triangle count on the device (T is then only the launch's
// upper bound: the extraction sized the mesh before reading its totals back)
__global__ void k_vertex_degree(const int32_t* __restrict__ tris, int64_t T, uint32_t* __restrict__ deg,
                                const uint8_t* __restrict__ dirty, const unsigned long long* __restrict__ T_dev) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * (T_dev ? (int64_t)*T_dev : T)) return;
  const int32_t v = tris[i];
  if (!dirty || dirty[v]) atomicAdd(&deg[v], 1u);
}
void launch_vertex_degree(const int32_t* tris, int64_t T, uint32_t* deg, cudaStream_t s, const uint8_t* dirty,
                          const unsigned long long* T_dev) {
  if (T) k_vertex_degree<<<grid_for(3 * T, 256), 256, 0, s>>>(tris, T, deg, dirty, T_dev);
}
__global__ void k_vertex_fill(const int32_t* __restrict__ tris, int64_t T, const uint32_t* __restrict__ off,
                              uint32_t* __restrict__ cursor, int32_t* __restrict__ inc,
                              const uint8_t* __restrict__ dirty, const unsigned long long* __restrict__ T_dev) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * (T_dev ? (int64_t)*T_dev : T)) return;
  const int32_t v = tris[i];
  if (dirty && !dirty[v]) return;
  const uint32_t slot = atomicAdd(&cursor[v], 1u);
  inc[off[v] + slot] = (int32_t)(i / 3);
}
void launch_vertex_fill(const int32_t* tris, int64_t T, const uint32_t* off, uint32_t* cursor, int32_t* inc,
                        cudaStream_t s, const uint8_t* dirty, const unsigned long long* T_dev) {
  if (T) k_vertex_fill<<<grid_for(3 * T, 256), 256, 0, s>>>(tris, T, off, cursor, inc, dirty, T_dev);
}

// Scratch of one fan (nt incident triangles).  Fans of up to kMaxFan
// triangles live in the thread's local arrays; a larger fan (no cap in the
// reference, polygonize.py:308-358) uses a global-memory region sized by its
// degree: the region of vertex v starts at byte kFanSlotBytes * off[v] of
// the CSR incidence offsets, so no separate allocation pass is needed.
constexpr int kFanSlotBytes = 72;  // 4 doubles + 9 ints + 1 bool per incident triangle, rounded to 8
struct FanScratch {
  double* rel;  // [3 nt]
  double* th;   // [nt]
  int32_t* tl;  // [nt]
  int* parent;
  int* mem;
  int* order;
  int* root_comp;
  int* comp;
  int32_t* nb;  // [2 nt]
  int* pa;      // [nt / 2]
  int* pb;      // [nt / 2]
  bool* fwd;    // [nt]
};
struct FanLocal {
  double rel[3 * kMaxFan], th[kMaxFan];
  int32_t tl[kMaxFan];
  int parent[kMaxFan], mem[kMaxFan], order[kMaxFan], root_comp[kMaxFan], comp[kMaxFan];
  int32_t nb[2 * kMaxFan];
  int pa[kMaxFan / 2], pb[kMaxFan / 2];
  bool fwd[kMaxFan];
  __device__ FanScratch view() { return {rel, th, tl, parent, mem, order, root_comp, comp, nb, pa, pb, fwd}; }
};
__device__ __forceinline__ FanScratch fan_global(char* base, uint32_t start, int nt) {
  char* p = base + (size_t)kFanSlotBytes * start;
  FanScratch f;
  f.rel = (double*)p;
  f.th = f.rel + 3 * nt;
  int* ip = (int*)(f.th + nt);
  f.tl = ip;
  f.parent = ip + nt;
  f.mem = ip + 2 * nt;
  f.order = ip + 3 * nt;
  f.root_comp = ip + 4 * nt;
  f.comp = ip + 5 * nt;
  f.nb = ip + 6 * nt;
  f.pa = ip + 8 * nt;
  f.pb = f.pa + nt / 2;
  f.fwd = (bool*)(ip + 9 * nt);
  return f;
}

// components of vertex v's fan; comp[i] in first-appearance order (= order
// of the minimum triangle id, since tl is ascending)
static __device__ int fan_components(const double* __restrict__ verts, const int32_t* __restrict__ tris, int32_t v,
                                     int nt, FanScratch& f) {
  const int32_t* tl = f.tl;
  int* parent = f.parent;
  for (int i = 0; i < nt; i++) parent[i] = i;
  auto find = [&](int x) {
    while (parent[x] != x) {
      parent[x] = parent[parent[x]];
      x = parent[x];
    }
    return x;
  };
  auto unite = [&](int x, int y) {
    int rx = find(x), ry = find(y);
    if (rx != ry) parent[rx] = ry;
  };
  // neighbours u: for each, the local triangle indices containing edge (v,u)
  int32_t* nb = f.nb;
  int nnb = 0;
  for (int i = 0; i < nt; i++) {
    const int32_t* t = tris + 3 * (int64_t)tl[i];
    for (int c = 0; c < 3; c++) {
      const int32_t u = t[c];
      if (u == v) continue;
      bool seen = false;
      for (int j = 0; j < nnb; j++)
        if (nb[j] == u) seen = true;
      if (!seen) nb[nnb++] = u;  // at most 2 per triangle
    }
  }
  int* mem = f.mem;
  for (int j = 0; j < nnb; j++) {
    const int32_t u = nb[j];
    int nm = 0;
    for (int i = 0; i < nt; i++) {
      const int32_t* t = tris + 3 * (int64_t)tl[i];
      if (t[0] == u || t[1] == u || t[2] == u) mem[nm++] = i;
    }
    if (nm == 2) {
      unite(mem[0], mem[1]);
    } else if (nm > 2) {
      // sheet pairing by dihedral angle around edge (a,b), a < b
      const int32_t a = v < u ? v : u, b = v < u ? u : v;
      double axis[3];
      for (int c = 0; c < 3; c++) axis[c] = verts[3 * (int64_t)b + c] - verts[3 * (int64_t)a + c];
      double an = sqrt(dot3_fma(axis, axis));
      if (an == 0.0) an = 1.0;
      for (int c = 0; c < 3; c++) axis[c] /= an;
      double* rel = f.rel;
      bool* fwd = f.fwd;
      for (int m = 0; m < nm; m++) {
        const int32_t* t = tris + 3 * (int64_t)tl[mem[m]];
        int32_t other = -1;
        for (int c = 0; c < 3 && other < 0; c++)
          if (t[c] != a && t[c] != b) other = t[c];
        double rr[3];
        for (int c = 0; c < 3; c++) rr[c] = verts[3 * (int64_t)other + c] - verts[3 * (int64_t)a + c];
        const double pr = dot3_fma(rr, axis);
        for (int c = 0; c < 3; c++) rel[3 * m + c] = rr[c] - axis[c] * pr;
        // direction of the slot holding edge (a,b): e0 < e1 (polygonize.py:229)
        bool d = false;
        for (int c = 0; c < 3; c++) {
          const int32_t e0 = t[c], e1 = t[(c + 1) % 3];
          if ((e0 == a && e1 == b) || (e0 == b && e1 == a)) d = e0 < e1;
        }
        fwd[m] = d;
      }
      double ref[3] = {rel[0], rel[1], rel[2]};
      double rn = sqrt(dot3_fma(ref, ref));
      if (rn == 0.0) rn = 1.0;
      for (int c = 0; c < 3; c++) ref[c] /= rn;
      double perp[3];
      cross3(axis, ref, perp);
      double* th = f.th;
      int* order = f.order;
      for (int m = 0; m < nm; m++) {
        th[m] = atan2(dot3_fma(rel + 3 * m, perp), dot3_fma(rel + 3 * m, ref));
        order[m] = m;
      }
      for (int x = 1; x < nm; x++) {  // stable insertion sort
        int y = x;
        while (y > 0 && th[order[y - 1]] > th[order[y]]) {
          int tmp = order[y];
          order[y] = order[y - 1];
          order[y - 1] = tmp;
          y--;
        }
      }
      // _pair_fan_triangles (polygonize.py:233-250)
      const int np = nm / 2;
      int *pa = f.pa, *pb = f.pb;
      bool done = false;
      const int nstarts = (nm % 2 == 0) ? 2 : 1;
      for (int st = 0; st < nstarts && !done; st++) {
        bool okp = true;
        for (int i = 0; i < np; i++) {
          pa[i] = order[(st + 2 * i) % nm];
          pb[i] = order[(st + 2 * i + 1) % nm];
          if (fwd[pa[i]] == fwd[pb[i]]) okp = false;
        }
        done = okp;
      }
      if (!done)
        for (int i = 0; i < np; i++) {
          pa[i] = order[2 * i];
          pb[i] = order[2 * i + 1];
        }
      for (int i = 0; i < np; i++) unite(mem[pa[i]], mem[pb[i]]);
    }
  }
  int* root_comp = f.root_comp;
  for (int i = 0; i < nt; i++) root_comp[i] = -1;
  int ncomp = 0;
  for (int i = 0; i < nt; i++) {
    const int r = find(i);
    if (root_comp[r] < 0) root_comp[r] = ncomp++;
    f.comp[i] = root_comp[r];
  }
  return ncomp;
}

// vertex v's incident triangles, ascending, into f.tl; returns the count
__device__ __forceinline__ int load_fan(const uint32_t* off, const int32_t* inc, int64_t v, int32_t* tl) {
  const uint32_t b = off[v], e = off[v + 1];
  const int nt = (int)(e - b);
  for (int i = 0; i < nt; i++) tl[i] = inc[b + i];
  for (int x = 1; x < nt; x++) {  // ascending triangle ids
    int32_t key = tl[x];
    int y = x - 1;
    while (y >= 0 && tl[y] > key) {
      tl[y + 1] = tl[y];
      y--;
    }
    tl[y + 1] = key;
  }
  return nt;
}

// The fan of vertex v in local arrays, or (more than kMaxFan triangles) in
// its global scratch region; returns false when the fan is large and no
// scratch was provided (the host then re-runs with scratch).
__device__ __forceinline__ bool fan_scratch(const uint32_t* off, int64_t v, char* big, FanLocal& loc, FanScratch& f) {
  const int nt = (int)(off[v + 1] - off[v]);
  if (nt <= kMaxFan) {
    f = loc.view();
    return true;
  }
  if (!big) return false;
  f = fan_global(big, off[v], nt);
  return true;
}

__global__ void __launch_bounds__(128) k_repair_count(const double* __restrict__ verts,
                                                      const int32_t* __restrict__ tris, int64_t V,
                                                      const uint32_t* __restrict__ off,
                                                      const int32_t* __restrict__ inc, uint32_t* __restrict__ extra,
                                                      char* big, DevStats* st, const uint8_t* __restrict__ dirty) {
  int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  if ((dirty && !dirty[v]) || fan_is_disc(tris, off, inc, v)) {
    extra[v] = 0u;
    return;
  }
  FanLocal loc;
  FanScratch f;
  if (!fan_scratch(off, v, big, loc, f)) {
    atomicAdd(&st->repair_overflow, 1ull);
    return;
  }
  const int nt = load_fan(off, inc, v, f.tl);
  uint32_t ex = 0;
  if (nt > 1) ex = (uint32_t)(fan_components(verts, tris, (int32_t)v, nt, f) - 1);
  extra[v] = ex;
}
void launch_repair_count(const double* verts, const int32_t* tris, int64_t V, const uint32_t* off, const int32_t* inc,
                         uint32_t* extra, char* big, DevStats* st, cudaStream_t s, const uint8_t* dirty) {
  if (V) k_repair_count<<<grid_for(V, 128), 128, 0, s>>>(verts, tris, V, off, inc, extra, big, st, dirty);
}

// Vertices whose fan a repair pass changed: every corner (before and after)
// of a renamed triangle.  Any other vertex keeps its fan, so the next pass
// finds it as the last one did -- one component, nothing to add
// (polygonize.py:348-373 re-runs until nothing changes).
__global__ void k_mark_dirty(const int32_t* __restrict__ cur, const int32_t* __restrict__ next, int64_t T,
                             uint8_t* __restrict__ dirty) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int32_t a0 = cur[3 * t], a1 = cur[3 * t + 1], a2 = cur[3 * t + 2];
  const int32_t b0 = next[3 * t], b1 = next[3 * t + 1], b2 = next[3 * t + 2];
  if (a0 == b0 && a1 == b1 && a2 == b2) return;
  dirty[a0] = dirty[a1] = dirty[a2] = 1;
  dirty[b0] = dirty[b1] = dirty[b2] = 1;
}
void launch_mark_dirty(const int32_t* cur, const int32_t* next, int64_t T, uint8_t* dirty, cudaStream_t s) {
  if (T) k_mark_dirty<<<grid_for(T, 256), 256, 0, s>>>(cur, next, T, dirty);
}
size_t repair_scratch_bytes(int64_t T) { return (size_t)kFanSlotBytes * 3 * (size_t)T; }

__global__ void __launch_bounds__(128) k_repair_apply(const double* __restrict__ verts,
                                                      const int32_t* __restrict__ tris, int64_t V,
                                                      const uint32_t* __restrict__ off,
                                                      const int32_t* __restrict__ inc,
                                                      const uint32_t* __restrict__ extra_off, char* big,
                                                      int32_t* __restrict__ tris_next,
                                                      int64_t* __restrict__ src_of_new) {
  int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const uint32_t e0 = extra_off[v], e1 = extra_off[v + 1];
  if (e1 == e0) return;
  FanLocal loc;
  FanScratch f;
  if (!fan_scratch(off, v, big, loc, f)) return;  // (unreachable: count ran with the same scratch)
  const int nt = load_fan(off, inc, v, f.tl);
  fan_components(verts, tris, (int32_t)v, nt, f);
  for (uint32_t x = e0; x < e1; x++) src_of_new[x] = v;
  for (int i = 0; i < nt; i++) {
    if (f.comp[i] == 0) continue;
    const int32_t nv = (int32_t)(V + e0 + f.comp[i] - 1);
    const int64_t t = f.tl[i];
    for (int c = 0; c < 3; c++)
      if (tris[3 * t + c] == (int32_t)v) tris_next[3 * t + c] = nv;
  }
}
void launch_repair_apply(const double* verts, const int32_t* tris, int64_t V, const uint32_t* off, const int32_t* inc,
                         const uint32_t* extra_off, char* big, int32_t* tris_next, int64_t* src_of_new,
                         cudaStream_t s) {
  if (V) k_repair_apply<<<grid_for(V, 128), 128, 0, s>>>(verts, tris, V, off, inc, extra_off, big, tris_next,
                                                         src_of_new);
}

__global__ void k_copy_vertices(const double* __restrict__ src, const int64_t* __restrict__ src_of, int64_t base,
                                int64_t n, double* __restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = src_of[i];
  for (int c = 0; c < 3; c++) dst[3 * (base + i) + c] = src[3 * s + c];
}
void launch_copy_vertices(const double* src, const int64_t* src_of, int64_t base, int64_t n, double* dst,
                          cudaStream_t s) {
  if (n) k_copy_vertices<<<grid_for(n, 256), 256, 0, s>>>(src, src_of, base, n, dst);
}

// ===========================================================================
// slab mode helpers
// ===========================================================================
__global__ void k_count_owned_faces(GridP g, RecView rec, DevStats* st) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t nf = 0, n4 = 0;
  if (idx < g.NW) {
    const int64_t z = g.z0 + idiv(idiv(idx, g.W), g.S);
    if (z >= g.own0 && z < g.own1) {
      const WordRec* r = rec_find(rec, idx);
      if (r)
        for (int a = 0; a < 3; a++) {
          nf += __popc(r->f[a]);
          n4 += __popc(r->f4[a]);
        }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    nf += __shfl_xor_sync(0xffffffffu, nf, o);
    n4 += __shfl_xor_sync(0xffffffffu, n4, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (nf) atomicAdd(&st->faces_own, (unsigned long long)nf);
    if (n4) atomicAdd(&st->faces4_own, (unsigned long long)n4);
  }
}
void launch_count_owned_faces(const GridP& g, RecView rec, DevStats* st, cudaStream_t s) {
  k_count_owned_faces<<<grid_for(g.NW, 256), 256, 0, s>>>(g, rec, st);
}

// local ids: [0, P_halo) halo partitions (owned by the rank below, which
// numbers them last), [P_halo, P_window) owned partitions, then fans
__global__ void k_globalize_tris(const int32_t* __restrict__ tris, int64_t n, int64_t P_halo, int64_t P_window,
                                 int64_t part_base, int64_t P_total, int64_t fan_base, int32_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = tris[i];
  int64_t gv;
  if (v < P_halo) gv = part_base - P_halo + v;
  else if (v < P_window) gv = part_base + (v - P_halo);
  else gv = P_total + fan_base + (v - P_window);
  out[i] = (int32_t)gv;
}
void launch_globalize_tris(const int32_t* tris, int64_t T, int64_t P_halo, int64_t P_window, int64_t part_base,
                           int64_t P_total, int64_t fan_base, int32_t* out, cudaStream_t s) {
  if (T) k_globalize_tris<<<grid_for(3 * T, 256), 256, 0, s>>>(tris, 3 * T, P_halo, P_window, part_base, P_total,
                                                                fan_base, out);
}
__global__ void k_mark_used(const int32_t* __restrict__ tris, int64_t n, uint8_t* __restrict__ used) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) used[tris[i]] = 1;
}
void launch_mark_used(const int32_t* tris, int64_t T, uint8_t* used, cudaStream_t s) {
  if (T) k_mark_used<<<grid_for(3 * T, 256), 256, 0, s>>>(tris, 3 * T, used);
}
__global__ void k_widen_flags(const uint8_t* __restrict__ f, int64_t n, uint32_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = f[i] ? 1u : 0u;
}
void launch_widen_flags(const uint8_t* f, int64_t n, uint32_t* out, cudaStream_t s) {
  if (n) k_widen_flags<<<grid_for(n, 256), 256, 0, s>>>(f, n, out);
}
__global__ void k_gather_provenance(int64_t V, const int64_t* __restrict__ src_of, const int64_t* __restrict__ kin,
                                    const int64_t* __restrict__ rin, int64_t* __restrict__ kind,
                                    int64_t* __restrict__ ref) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int64_t s = src_of ? src_of[i] : i;
  kind[i] = kin[s];
  ref[2 * i] = rin[2 * s];
  ref[2 * i + 1] = rin[2 * s + 1];
}
void launch_gather_provenance(int64_t V, const int64_t* src_of, const int64_t* kind_in, const int64_t* ref_in,
                              int64_t* kind, int64_t* ref, cudaStream_t s) {
  if (V) k_gather_provenance<<<grid_for(V, 256), 256, 0, s>>>(V, src_of, kind_in, ref_in, kind, ref);
}

__global__ void k_provenance(int64_t V, int64_t P, const int64_t* __restrict__ src_of,
                             const int64_t* __restrict__ part_cell, const int64_t* __restrict__ part_index,
                             const int64_t* __restrict__ fan_edge, int64_t* __restrict__ kind,
                             int64_t* __restrict__ ref) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int64_t s = src_of ? src_of[i] : i;
  if (s < P) {
    kind[i] = 0;
    ref[2 * i] = part_cell[s];
    ref[2 * i + 1] = part_index[s];
  } else {
    kind[i] = 1;
    ref[2 * i] = fan_edge[s - P];
    ref[2 * i + 1] = -1;
  }
}
void launch_provenance(int64_t V, int64_t P, const int64_t* src_of, const int64_t* part_cell,
                       const int64_t* part_index, const int64_t* fan_edge, int64_t* kind, int64_t* ref,
                       cudaStream_t s) {
  if (V) k_provenance<<<grid_for(V, 256), 256, 0, s>>>(V, P, src_of, part_cell, part_index, fan_edge, kind, ref);
}

__global__ void k_widen_i32(const int32_t* __restrict__ src, int64_t* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
void launch_widen_i32(const int32_t* src, int64_t* dst, int64_t n, cudaStream_t s) {
  if (n) k_widen_i32<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n);
}

__global__ void k_dup_provenance(int64_t V0, int64_t V, int64_t* __restrict__ kind, int64_t* __restrict__ ref) {
  const int64_t i = V0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  if (kind) kind[i] = 2;
  if (ref) {
    ref[2 * i] = -1;
    ref[2 * i + 1] = -1;
  }
}
void launch_dup_provenance(int64_t V0, int64_t V, int64_t* kind, int64_t* ref, cudaStream_t s) {
  if (V > V0) k_dup_provenance<<<grid_for(V - V0, 256), 256, 0, s>>>(V0, V, kind, ref);
}


// ===========================================================================
// Marching-cubes baseline (baseline.py:48-127): one vertex per crossing edge,
// each partition cycle fanned from its first edge and oriented outward.
// ===========================================================================
// vertex of crossing edge k: binary = midpoint, continuous = inverse lerp of
// the raw grid values (baseline.py:78-89)
__global__ void k_mc_points(GridP g, const uint32_t* __restrict__ L, const int64_t* __restrict__ edge_key, int64_t K,
                            const double* __restrict__ raw_in, const double* __restrict__ raw_out, double iso,
                            double* __restrict__ pos) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const EdgeGeom e = edge_geom(g, L, edge_key[k]);
  double t = 0.5;
  if (raw_in) {
    const double pin = raw_in[k] - iso, pout = raw_out[k] - iso;
    const double den = pin - pout;
    t = pin / (fabs(den) < 1e-300 ? 1.0 : den);
    if (!isnan(t)) t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  }
  for (int c = 0; c < 3; c++) pos[3 * k + c] = e.pin[c] + t * e.span[c];
}
void launch_mc_points(const GridP& g, const uint32_t* L, const int64_t* edge_key, int64_t K, const double* raw_in,
                      const double* raw_out, double iso, double* pos, cudaStream_t s) {
  if (K) k_mc_points<<<grid_for(K, 256), 256, 0, s>>>(g, L, edge_key, K, raw_in, raw_out, iso, pos);
}

// triangles per cell: sum over its cycles of (len - 2) = edges - 2 * cycles
__global__ void k_mc_count(int64_t C, const uint32_t* __restrict__ ncyc, const uint32_t* __restrict__ nedge,
                           uint32_t* __restrict__ ntri) {
  const int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ci < C) ntri[ci] = nedge[ci] - 2 * ncyc[ci];
}
void launch_mc_count(int64_t C, const uint32_t* ncyc, const uint32_t* nedge, uint32_t* ntri, cudaStream_t s) {
  if (C) k_mc_count<<<grid_for(C, 256), 256, 0, s>>>(C, ncyc, nedge, ntri);
}

__global__ void k_mc_fans(GridP g, const uint32_t* __restrict__ L, RecView rec,
                          const int64_t* __restrict__ cell_id, int64_t C, const CellTabEntry* __restrict__ table,
                          const uint16_t* __restrict__ cfg, const uint32_t* __restrict__ tri_off,
                          const double* __restrict__ pos, int32_t* __restrict__ tris, uint8_t* __restrict__ used) {
  const int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ci >= C) return;
  const int64_t base = cell_base_vid(g, cell_id[ci]);
  const CellTabEntry T = table[cfg[ci]];
  int64_t out = tri_off[ci];
  int slot = 0;
  for (int k = 0; k < T.ncyc; k++) {
    const int len = (T.lens >> (4 * k)) & 15;
    int64_t rows[12];
    double outward[3] = {0.0, 0.0, 0.0};
    for (int j = 0; j < len; j++) {
      const int le = (int)((T.edges >> (4 * (slot + j))) & 15);
      const int64_t ev = base + corner_off(g, c_LE_CORNER[le]);
      const int ax = c_LE_AXIS[le];
      rows[j] = edge_rank(rec, g, ev, ax);
      const EdgeGeom e = edge_geom(g, L, ev * 3 + ax);
      for (int c = 0; c < 3; c++) outward[c] = j == 0 ? e.span[c] : outward[c] + e.span[c];
    }
    slot += len;
    if (len < 3) continue;
    // normal = sum of the fan triangles' cross products, in fan order
    double nrm[3] = {0.0, 0.0, 0.0};
    const double* a = pos + 3 * rows[0];
    for (int j = 1; j + 1 < len; j++) {
      const double* b = pos + 3 * rows[j];
      const double* c = pos + 3 * rows[j + 1];
      const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
      const double w[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
      double x[3];
      cross3(u, w, x);
      for (int q = 0; q < 3; q++) nrm[q] = nrm[q] + x[q];
    }
    // normal @ outward: numpy's 1-D matmul is an fma chain (BLAS ddot)
    const double dot = __fma_rn(nrm[2], outward[2], __fma_rn(nrm[1], outward[1], nrm[0] * outward[0]));
    const bool flip = dot < 0.0;
    for (int j = 1; j + 1 < len; j++, out++) {
      tris[3 * out] = (int32_t)rows[0];
      tris[3 * out + 1] = (int32_t)(flip ? rows[j + 1] : rows[j]);
      tris[3 * out + 2] = (int32_t)(flip ? rows[j] : rows[j + 1]);
    }
    for (int j = 0; j < len; j++) used[rows[j]] = 1;
  }
}
void launch_mc_fans(const GridP& g, const uint32_t* L, RecView rec, const int64_t* cell_id, int64_t C,
                    const CellTabEntry* table, const uint16_t* cfg, const uint32_t* tri_off, const double* pos,
                    int32_t* tris, uint8_t* used, cudaStream_t s) {
  if (C) k_mc_fans<<<grid_for(C, 128), 128, 0, s>>>(g, L, rec, cell_id, C, table, cfg, tri_off, pos, tris, used);
}

}  // namespace odc
