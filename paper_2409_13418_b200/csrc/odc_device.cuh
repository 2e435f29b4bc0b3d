// odc_device.cuh -- shared device definitions for the ODC extraction kernels.
//
// Numerics: every fp64 expression that mirrors a numpy expression of the
// reference is written in numpy's evaluation order and this translation unit
// is compiled with --fmad=false, so no multiply/add pair is contracted.  Explicit
// fma() appears only where the reference's BLAS uses one (OpenBLAS dgemm for
// (N,3)@(3,3), ddot) -- see SURVEY.md Appendix A.
#pragma once
#include <cstdint>

#include "../../include/odc.h"

namespace odc {

constexpr int kMaxValueStack = 32;
constexpr int kMaxPointStack = 8;

// ---------------------------------------------------------------------------
// grid (grid.py:17-91): vertex id = x + y*S + z*S^2, h = (hi - lo) / R,
// position = lo + coord * h.  Bit-packed rows: a row is (y, z), W 32-bit words
// cover x in [0, 32W); word index = (z*S + y)*W + x/32.
// ---------------------------------------------------------------------------
// z-window (slab mode): the device holds vertex layers
// [z0, z0 + nz) of the global grid; ids, keys and positions stay global.
// Edges/faces/vertices with base layer in [own0, own1) are owned by this
// extraction (the full grid: z0 = 0, nz = S, own = [0, S)).
//
// Batch (BASELINE config 5, odc_extract_batch): nb grids of the same R
// stacked along z -- shape b holds global vertex layers [b S, b S + S) --
// so every kernel runs once over all shapes and the flat index space
// carries the shape in its high part.  Keys and ids stay global (ordered
// shape by shape); a kernel that needs a shape's geometry calls localize()
// with the element's z, which loads that shape's lo/h and z offset.
struct GridP {
  int64_t R, S, S2, S3;
  int64_t W;   // words per row
  int64_t NW;  // nz*S*W words held
  int64_t z0, nz, own0, own1;
  double lo[3], h[3];
  int64_t zoff = 0;            // z of the localized shape's layer 0 (positions use z - zoff)
  // word index -> (row, x word) and row -> (z, y) by multiply-shift
  // (set_word_divisors; exact for dividends below 2^31)
  uint32_t w_m = 0, w_s = 0, s_m = 0, s_s = 0;
  int32_t nb = 0;              // batch: shapes stacked along z (0: one grid)
  const double* geo = nullptr;  // batch: device (nb, 6) = lo[3], h[3] per shape
};

// Per-word record of every derived bitmap plus the exclusive ranks of the
// word's first element (edges, 2D-point instances, cells).  Records exist
// only for ACTIVE words (any crossing edge, face or cell bit): the surface
// touches a few percent of the grid's words, so a dense per-word array
// (64 B for every 4 B label word) was 16x the label traffic at 1025^3.
struct __align__(16) WordRec {
  uint32_t e[3];   // crossing edges by axis, bit at the lower vertex
  uint32_t f[3];   // crossing faces (2 or 4 crossing edges) by normal axis
  uint32_t f4[3];  // faces with 4 crossing edges
  uint32_t cf[3];  // face-centre labels of 4-crossing faces
  uint32_t cell;   // crossing cells (bit at the cell's base vertex)
  uint32_t pe, pq, pc;  // exclusive prefix: edges, instances, cells
};
static_assert(sizeof(WordRec) == 64, "WordRec must be one 64-byte record");

// Sparse word records: occ[w / 32] = {bitmap of active words w' in the
// group of 32, number of active words before the group}; the record of an
// active word w is rec[occ.y + popc(occ.x & lowmask(w % 32))].
struct RecView {
  const uint2* occ;
  WordRec* rec;
};

__device__ __forceinline__ int64_t word_of(const GridP& g, int64_t x, int64_t y, int64_t z) {
  return ((z - g.z0) * g.S + y) * g.W + (x >> 5);
}
// non-negative a / b and a % b with the 32-bit divider when both fit (the
// 64-bit one is a long software routine)
__device__ __forceinline__ int64_t idiv(int64_t a, int64_t b) {
  return ((uint64_t)a <= 0xffffffffull && (uint64_t)b <= 0xffffffffull) ? (int64_t)((uint32_t)a / (uint32_t)b) : a / b;
}
__device__ __forceinline__ int64_t imod(int64_t a, int64_t b) {
  return ((uint64_t)a <= 0xffffffffull && (uint64_t)b <= 0xffffffffull) ? (int64_t)((uint32_t)a % (uint32_t)b) : a % b;
}

// host: multiply-shift constants for n / d, n < 2^31 (round-up multiplier)
inline void magic_u31(uint32_t d, uint32_t& m, uint32_t& sh) {
  uint32_t l = 0;
  while ((1u << l) < d) l++;
  const uint32_t pw = 31 + l;
  m = (uint32_t)(((1ull << pw) + d - 1) / d);
  sh = pw - 32;
}
inline void set_word_divisors(GridP& g) {
  g.w_m = g.s_m = 0;  // 0: word_coords divides (a divisor of 1 has no 32-bit multiplier)
  if (g.W < 2 || g.S < 2 || g.W > 0xffff || g.S > 0xffff) return;
  magic_u31((uint32_t)g.W, g.w_m, g.w_s);
  magic_u31((uint32_t)g.S, g.s_m, g.s_s);
}
// label word w -> (y, z, x word) of the window (w < 2^31 words)
__device__ __forceinline__ void word_coords(const GridP& g, int64_t w, int64_t& y, int64_t& z, int64_t& wx) {
  if (g.w_m && w < (1ll << 31)) {
    const uint32_t row = __umulhi((uint32_t)w, g.w_m) >> g.w_s;
    const uint32_t zr = __umulhi(row, g.s_m) >> g.s_s;
    wx = (int64_t)((uint32_t)w - row * (uint32_t)g.W);
    y = (int64_t)(row - zr * (uint32_t)g.S);
    z = g.z0 + (int64_t)zr;
    return;
  }
  const int64_t row = idiv(w, g.W);
  wx = w - row * g.W;
  y = imod(row, g.S);
  z = g.z0 + idiv(row, g.S);
}
__device__ __forceinline__ void vid_coords(const GridP& g, int64_t vid, int64_t c[3]) {
  if ((uint64_t)vid <= 0xffffffffull && g.S <= 0xffff) {  // 32-bit divisions (every grid up to 2^32 vertices)
    const uint32_t v = (uint32_t)vid, S = (uint32_t)g.S;
    const uint32_t q = v / S;
    c[0] = v - q * S;
    c[1] = q % S;
    c[2] = q / S;
    return;
  }
  c[0] = vid % g.S;
  c[1] = (vid / g.S) % g.S;
  c[2] = vid / g.S2;
}
__device__ __forceinline__ int64_t vstep(const GridP& g, int a) { return a == 0 ? 1 : (a == 1 ? g.S : g.S2); }
__device__ __forceinline__ double gpos(const GridP& g, int a, int64_t c) {
  return __dadd_rn(g.lo[a], __dmul_rn((double)(a == 2 ? c - g.zoff : c), g.h[a]));
}
// batch: shape of global vertex layer z (0 for one grid)
__device__ __forceinline__ int shape_of_z(const GridP& g, int64_t z) { return g.nb ? (int)idiv(z, g.S) : 0; }
// batch: switch g to the geometry of the shape holding layer z; returns it
template <bool B = true>
__device__ __forceinline__ int localize(GridP& g, int64_t z) {
  if (!B || !g.nb) return 0;
  const int b = (int)idiv(z, g.S);
  g.zoff = (int64_t)b * g.S;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    g.lo[a] = g.geo[6 * b + a];
    g.h[a] = g.geo[6 * b + 3 + a];
  }
  return b;
}
__device__ __forceinline__ void vposition(const GridP& g, int64_t vid, double p[3]) {
  int64_t c[3];
  vid_coords(g, vid, c);
#pragma unroll
  for (int a = 0; a < 3; a++) p[a] = gpos(g, a, c[a]);
}
__device__ __forceinline__ uint32_t label_at(const uint32_t* L, const GridP& g, int64_t vid) {
  int64_t c[3];
  vid_coords(g, vid, c);
  return (L[word_of(g, c[0], c[1], c[2])] >> (c[0] & 31)) & 1u;
}
__device__ __forceinline__ uint32_t lowmask(int bit) { return bit == 0 ? 0u : (0xffffffffu >> (32 - bit)); }
// record of word w, or nullptr when the word has no crossing element
__device__ __forceinline__ WordRec* rec_find(const RecView& rv, int64_t w) {
  const uint2 o = rv.occ[w >> 5];
  const int b = (int)(w & 31);
  if (!((o.x >> b) & 1u)) return nullptr;
  return rv.rec + o.y + __popc(o.x & lowmask(b));
}

// Ranks from vertex coordinates (callers that already hold them skip the
// vid -> (x, y, z) divisions).
// rank of crossing edge (x, y, z, axis) in ascending edge-key order
__device__ __forceinline__ int64_t edge_rank_c(const RecView& rec, const GridP& g, int64_t x, int64_t y, int64_t z,
                                               int axis) {
  const WordRec& r = *rec_find(rec, word_of(g, x, y, z));  // the element's word is active
  int bit = (int)(x & 31);
  uint32_t m = lowmask(bit);
  int64_t k = (int64_t)r.pe + __popc(r.e[0] & m) + __popc(r.e[1] & m) + __popc(r.e[2] & m);
  for (int a = 0; a < axis; a++) k += (r.e[a] >> bit) & 1u;
  return k;
}
// id of the first 2D-point instance of face (x, y, z, normal): instances
// are numbered in face-key order, two per 4-crossing face (dualize.py:72-88)
__device__ __forceinline__ int64_t inst_rank_c(const RecView& rec, const GridP& g, int64_t x, int64_t y, int64_t z,
                                               int n) {
  const WordRec& r = *rec_find(rec, word_of(g, x, y, z));  // the element's word is active
  int bit = (int)(x & 31);
  uint32_t m = lowmask(bit);
  int64_t k = (int64_t)r.pq;
#pragma unroll
  for (int a = 0; a < 3; a++) k += __popc(r.f[a] & m) + __popc(r.f4[a] & m);
  for (int a = 0; a < n; a++) k += ((r.f[a] >> bit) & 1u) + ((r.f4[a] >> bit) & 1u);
  return k;
}
__device__ __forceinline__ int64_t edge_rank(const RecView& rec, const GridP& g, int64_t vid, int axis) {
  int64_t c[3];
  vid_coords(g, vid, c);
  return edge_rank_c(rec, g, c[0], c[1], c[2], axis);
}
__device__ __forceinline__ int64_t inst_rank(const RecView& rec, const GridP& g, int64_t vid, int n) {
  int64_t c[3];
  vid_coords(g, vid, c);
  return inst_rank_c(rec, g, c[0], c[1], c[2], n);
}
__device__ __forceinline__ int64_t cell_rank(const RecView& rec, const GridP& g, int64_t base_vid) {
  int64_t c[3];
  vid_coords(g, base_vid, c);
  const WordRec& r = *rec_find(rec, word_of(g, c[0], c[1], c[2]));  // the element's word is active
  int bit = (int)(c[0] & 31);
  return (int64_t)r.pc + __popc(r.cell & lowmask(bit));
}
__device__ __forceinline__ uint32_t label_c(const uint32_t* L, const GridP& g, int64_t x, int64_t y, int64_t z) {
  return (L[word_of(g, x, y, z)] >> (x & 31)) & 1u;
}
__device__ __forceinline__ void vposition_c(const GridP& g, int64_t x, int64_t y, int64_t z, double p[3]) {
  p[0] = gpos(g, 0, x);
  p[1] = gpos(g, 1, y);
  p[2] = gpos(g, 2, z);
}

// ---------------------------------------------------------------------------
// field programs (fields.py:64-242)
// ---------------------------------------------------------------------------
struct FieldP {
  const odc_node* nodes;  // device
  int32_t n_nodes;
  int32_t kind;  // 0 analytic program, 1 MLP
  double iso;
  // Fast paths, by value (kernel-parameter space: uniform constant-bank
  // reads instead of per-thread global loads, which bound the label kernel
  // on L1 throughput).  fast: 0 none (interpreter), 1 prim -> sd2raw,
  // 2 prim -> smooth(k), 3 prim, sd2raw, prim, sd2raw, raw op fop[2].
  int32_t fast = 0;
  int32_t fop[3] = {0, 0, 0};
  double fq[2][16] = {};
  double fk = 0.0;
  const FieldP* batch = nullptr;  // batch: device (nb) fields, one per shape
  int32_t ev = 0;                 // evaluation mode (ev_mode_of), set by the host
};
__device__ __forceinline__ const FieldP& field_of(const FieldP& f, int b) { return f.batch ? f.batch[b] : f; }
// host: classify a program for FieldP's fast paths (same patterns as field_raw)
inline void fieldp_set_fast(FieldP& f, const odc_node* h, int32_t n) {
  auto prim = [](int op) {
    return op == ODC_OP_SPHERE_SD || op == ODC_OP_BOX_SD || op == ODC_OP_TORUS_SD || op == ODC_OP_PLANE_SD;
  };
  f.fast = 0;
  if (n == 2 && prim(h[0].op) && (h[1].op == ODC_OP_SD2RAW || h[1].op == ODC_OP_SMOOTH)) {
    f.fast = h[1].op == ODC_OP_SD2RAW ? 1 : 2;
    f.fop[0] = h[0].op;
    for (int i = 0; i < 16; i++) f.fq[0][i] = h[0].p[i];
    f.fk = h[1].p[0];
  } else if (n == 5 && prim(h[0].op) && h[1].op == ODC_OP_SD2RAW && prim(h[2].op) && h[3].op == ODC_OP_SD2RAW &&
             (h[4].op == ODC_OP_RAW_MAX || h[4].op == ODC_OP_RAW_MIN || h[4].op == ODC_OP_RAW_DIFF)) {
    f.fast = 3;
    f.fop[0] = h[0].op;
    f.fop[1] = h[2].op;
    f.fop[2] = h[4].op;
    for (int i = 0; i < 16; i++) {
      f.fq[0][i] = h[0].p[i];
      f.fq[1][i] = h[2].p[i];
    }
  }
}

// glibc 2.39 hypot (x86-64 baseline build): Borges' corrected sqrt kernel,
// reproduced bit-for-bit (checked on 2e7 random pairs against libm).
static __device__ __forceinline__ double hypot_glibc(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ay <= __dmul_rn(ax, 0x1p-54)) return __dadd_rn(ax, ay);
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    double delta = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
    t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
  } else {
    double delta = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

// sqrt((x0*x0 + x1*x1) + x2*x2): numpy linalg.norm over the last axis of (N,3)
__device__ __forceinline__ double norm3(const double x[3]) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x[0], x[0]), __dmul_rn(x[1], x[1])), __dmul_rn(x[2], x[2])));
}
// einsum('ij,ij->i') with three terms: (p0 + p2) + p1
__device__ __forceinline__ double einsum3(const double a[3], const double b[3]) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[2], b[2])), __dmul_rn(a[1], b[1]));
}
__device__ __forceinline__ double dot3_fma(const double a[3], const double b[3]) {
  return fma(a[2], b[2], fma(a[1], b[1], __dmul_rn(a[0], b[0])));
}
__device__ __forceinline__ void cross3(const double a[3], const double b[3], double o[3]) {
  o[0] = __dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1]));
  o[1] = __dsub_rn(__dmul_rn(a[2], b[0]), __dmul_rn(a[0], b[2]));
  o[2] = __dsub_rn(__dmul_rn(a[0], b[1]), __dmul_rn(a[1], b[0]));
}
// (p - c) @ R with OpenBLAS dgemm's fma chain (fields.py:107, :179)
__device__ __forceinline__ void rot_rows(const double l[3], const double* R, double o[3]) {
#pragma unroll
  for (int j = 0; j < 3; j++) o[j] = fma(l[2], R[6 + j], fma(l[1], R[3 + j], __dmul_rn(l[0], R[j])));
}

// signed distance of one primitive node at p (fields.py:75-139); shared by
// the interpreter and the fast paths so both give identical bits
__device__ __forceinline__ double prim_sd(int op, const double* q, const double p[3]) {
  if (op == ODC_OP_SPHERE_SD) {  // fields.py:80-82
    double d[3] = {__dsub_rn(p[0], q[0]), __dsub_rn(p[1], q[1]), __dsub_rn(p[2], q[2])};
    return __dsub_rn(norm3(d), q[3]);
  }
  if (op == ODC_OP_BOX_SD) {  // fields.py:103-111
    double l[3] = {__dsub_rn(p[0], q[0]), __dsub_rn(p[1], q[1]), __dsub_rn(p[2], q[2])};
    if (q[6] != 0.0) {
      double R[9], o[3];
      for (int j = 0; j < 9; j++) R[j] = q[7 + j];
      rot_rows(l, R, o);
      l[0] = o[0]; l[1] = o[1]; l[2] = o[2];
    }
    double qq[3], mq[3];
    for (int a = 0; a < 3; a++) {
      qq[a] = __dsub_rn(fabs(l[a]), q[3 + a]);
      mq[a] = qq[a] > 0.0 ? qq[a] : 0.0;
    }
    const double outside = norm3(mq);
    double mx = qq[0];
    if (qq[1] > mx) mx = qq[1];
    if (qq[2] > mx) mx = qq[2];
    const double inside = mx < 0.0 ? mx : 0.0;
    return __dadd_rn(outside, inside);
  }
  if (op == ODC_OP_TORUS_SD) {  // fields.py:122-126
    double l[3] = {__dsub_rn(p[0], q[0]), __dsub_rn(p[1], q[1]), __dsub_rn(p[2], q[2])};
    const double ring = __dsub_rn(hypot_glibc(l[0], l[1]), q[3]);
    return __dsub_rn(hypot_glibc(ring, l[2]), q[4]);
  }
  // ODC_OP_PLANE_SD, fields.py:138-139 (dgemv)
  double l[3] = {__dsub_rn(p[0], q[0]), __dsub_rn(p[1], q[1]), __dsub_rn(p[2], q[2])};
  double nn[3] = {q[3], q[4], q[5]};
  return dot3_fma(l, nn);
}
// sd < 0 for one primitive.  For a box, sd = |max(q, 0)| + min(max_i q_i, 0)
// is negative exactly when every q_i < 0 (otherwise the min term is 0 and
// the norm is >= 0), so the label needs neither the norm nor its sqrt.
//
// Sphere: sd = sqrt_rn(s) - r with s = (x^2 + y^2) + z^2 rounded as numpy
// does, and sd < 0 <=> sqrt_rn(s) < r.  fma(r, r, -s) has the exact sign of
// r^2 - s: if it is <= 0, sqrt(s) >= r and so is its rounding; if it exceeds
// 2^-50 r^2, sqrt(s) < r by more than an ulp of r and its rounding stays
// below r.  Only the sliver in between takes the sqrt.
__device__ __forceinline__ bool sphere_inside(const double* q, const double p[3]) {
  const double d[3] = {__dsub_rn(p[0], q[0]), __dsub_rn(p[1], q[1]), __dsub_rn(p[2], q[2])};
  const double s = __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2]));
  const double r = q[3];
  if (r > 1e-150 && r < 1e150) {
    const double e = fma(r, r, -s);
    if (e <= 0.0) return false;
    if (e > 0x1p-50 * __dmul_rn(r, r)) return true;
  }
  return __dsub_rn(__dsqrt_rn(s), r) < 0.0;
}
__device__ __forceinline__ bool prim_inside(int op, const double* q, const double p[3]) {
  if (op == ODC_OP_SPHERE_SD) return sphere_inside(q, p);
  if (op != ODC_OP_BOX_SD) return prim_sd(op, q, p) < 0.0;
  double l[3] = {__dsub_rn(p[0], q[0]), __dsub_rn(p[1], q[1]), __dsub_rn(p[2], q[2])};
  if (q[6] != 0.0) {
    double R[9], o[3];
    for (int j = 0; j < 9; j++) R[j] = q[7 + j];
    rot_rows(l, R, o);
    l[0] = o[0]; l[1] = o[1]; l[2] = o[2];
  }
  bool in = true;
  for (int a = 0; a < 3; a++) in &= __dsub_rn(fabs(l[a]), q[3 + a]) < 0.0;
  return in;
}
__device__ __forceinline__ bool is_prim(int op) {
  return op == ODC_OP_SPHERE_SD || op == ODC_OP_BOX_SD || op == ODC_OP_TORUS_SD || op == ODC_OP_PLANE_SD;
}
// fields.py:239-242
__device__ __forceinline__ double smooth_raw(double k, double sd) {
  double kd = __dmul_rn(k, sd);
  kd = kd < -500.0 ? -500.0 : kd;
  kd = kd > 500.0 ? 500.0 : kd;
  return __ddiv_rn(1.0, __dadd_rn(1.0, exp(kd)));
}

static __device__ __noinline__ double field_raw_prog(const odc_node* __restrict__ nodes, int n_nodes, const double pt[3]) {
  double st[kMaxValueStack];
  double pst[kMaxPointStack][3];
  int sp = 0, pp = 0;
  double p[3] = {pt[0], pt[1], pt[2]};
  for (int i = 0; i < n_nodes; i++) {
    const int op = __ldg(&nodes[i].op);
    const double* q = nodes[i].p;
    switch (op) {
      case ODC_OP_SPHERE_SD:
      case ODC_OP_BOX_SD:
      case ODC_OP_TORUS_SD:
      case ODC_OP_PLANE_SD: st[sp++] = prim_sd(op, q, p); break;
      case ODC_OP_SD2RAW: st[sp - 1] = st[sp - 1] < 0.0 ? 1.0 : 0.0; break;  // fields.py:70-72
      case ODC_OP_RAW_MAX:
      case ODC_OP_SD_MAX: {
        double b = st[--sp], a = st[sp - 1];
        st[sp - 1] = (a >= b) ? a : b;
        break;
      }
      case ODC_OP_RAW_MIN:
      case ODC_OP_SD_MIN: {
        double b = st[--sp], a = st[sp - 1];
        st[sp - 1] = (a <= b) ? a : b;
        break;
      }
      case ODC_OP_RAW_DIFF: {  // min(a, 1 - b), fields.py:197
        double b = __dsub_rn(1.0, st[--sp]), a = st[sp - 1];
        st[sp - 1] = (a <= b) ? a : b;
        break;
      }
      case ODC_OP_RAW_COMPL: st[sp - 1] = __dsub_rn(1.0, st[sp - 1]); break;
      case ODC_OP_SD_DIFF: {  // max(a, -b), fields.py:216
        double b = -st[--sp], a = st[sp - 1];
        st[sp - 1] = (a >= b) ? a : b;
        break;
      }
      case ODC_OP_SD_NEG: st[sp - 1] = -st[sp - 1]; break;
      case ODC_OP_XFORM_BEGIN: {  // (p - t) @ R, fields.py:176-180
        pst[pp][0] = p[0]; pst[pp][1] = p[1]; pst[pp][2] = p[2];
        pp++;
        double l[3] = {__dsub_rn(p[0], __ldg(q)), __dsub_rn(p[1], __ldg(q + 1)), __dsub_rn(p[2], __ldg(q + 2))};
        if (__ldg(q + 6) != 0.0) {
          double R[9], o[3];
          for (int j = 0; j < 9; j++) R[j] = __ldg(q + 7 + j);
          rot_rows(l, R, o);
          l[0] = o[0]; l[1] = o[1]; l[2] = o[2];
        }
        p[0] = l[0]; p[1] = l[1]; p[2] = l[2];
        break;
      }
      case ODC_OP_XFORM_END:
        pp--;
        p[0] = pst[pp][0]; p[1] = pst[pp][1]; p[2] = pst[pp][2];
        break;
      case ODC_OP_SMOOTH: st[sp - 1] = smooth_raw(__ldg(q), st[sp - 1]); break;
      default: break;
    }
  }
  return sp > 0 ? st[sp - 1] : 0.0;
}

// Fast paths (registers only, no stack) for the program shapes of the
// scenes: one primitive -> raw or smoothed, and a CSG pair of primitives
// (union / intersection / difference of their binary raws).  Same node
// arithmetic as the interpreter, so identical bits; anything else runs the
// interpreter.
// One primitive's label / sd from kernel-parameter space: each primitive
// loads only its own parameters (a sphere 4 doubles, not the 16 of a
// rotated box) -- the loads are a large share of a search kernel's
// instructions, one field evaluation per step.
template <int N>
__device__ __forceinline__ void load_params(const double (&q)[16], double (&o)[16]) {
#pragma unroll
  for (int i = 0; i < N; i++) o[i] = q[i];
}
__device__ __forceinline__ bool prim_inside_p(int op, const double (&q)[16], const double p[3]) {
  double c[16];
  if (op == ODC_OP_SPHERE_SD) {
    load_params<4>(q, c);
    return sphere_inside(c, p);
  }
  if (op == ODC_OP_BOX_SD) {
    load_params<16>(q, c);
    return prim_inside(ODC_OP_BOX_SD, c, p);
  }
  if (op == ODC_OP_TORUS_SD) {
    load_params<5>(q, c);
    return prim_sd(ODC_OP_TORUS_SD, c, p) < 0.0;
  }
  load_params<6>(q, c);
  return prim_sd(ODC_OP_PLANE_SD, c, p) < 0.0;
}
__device__ __forceinline__ double prim_sd_p(int op, const double (&q)[16], const double p[3]) {
  double c[16];
  if (op == ODC_OP_SPHERE_SD) {
    load_params<4>(q, c);
    return prim_sd(ODC_OP_SPHERE_SD, c, p);
  }
  if (op == ODC_OP_BOX_SD) {
    load_params<16>(q, c);
    return prim_sd(ODC_OP_BOX_SD, c, p);
  }
  if (op == ODC_OP_TORUS_SD) {
    load_params<5>(q, c);
    return prim_sd(ODC_OP_TORUS_SD, c, p);
  }
  load_params<6>(q, c);
  return prim_sd(ODC_OP_PLANE_SD, c, p);
}

// SEL: per-primitive parameter loads (prim_inside_p) -- faster when the
// FieldP sits in global memory (batches); a kernel-parameter FieldP keeps
// the copy-all form, which its uniform constant loads serve better.
// Evaluation modes: 0 kernel-parameter FieldP (copy its parameters), 1
// per-primitive loads (FieldP in global memory: batches), and kernels
// specialised for the commonest fast paths (the host picks them from the
// FieldP): one sphere / box / torus, a CSG pair of spheres.
// EV_BOX2F: a CSG pair of boxes in the same frame (bitwise-equal centre and
// rotation, e.g. a hollow box): the rotated local point is computed once.
enum { EV_PARAM = 0, EV_SEL = 1, EV_SPHERE = 2, EV_BOX = 3, EV_TORUS = 4, EV_SPHERE2 = 5, EV_BOX2F = 6 };
__host__ __device__ inline int ev_mode_of(const FieldP& f) {
  if (f.fast == 1 && f.fop[0] == ODC_OP_SPHERE_SD) return EV_SPHERE;
  if (f.fast == 1 && f.fop[0] == ODC_OP_BOX_SD) return EV_BOX;
  if (f.fast == 1 && f.fop[0] == ODC_OP_TORUS_SD) return EV_TORUS;
  if (f.fast == 3 && f.fop[0] == ODC_OP_SPHERE_SD && f.fop[1] == ODC_OP_SPHERE_SD) return EV_SPHERE2;
  if (f.fast == 3 && f.fop[0] == ODC_OP_BOX_SD && f.fop[1] == ODC_OP_BOX_SD) {
    bool same = true;
    for (int i = 0; i < 16; i++)
      if (i < 3 || i > 5) same = same && f.fq[0][i] == f.fq[1][i] && ((f.fq[0][i] == 0.0) == (f.fq[1][i] == 0.0));
    if (same) return EV_BOX2F;
  }
  return EV_PARAM;
}
template <int SEL = EV_PARAM>
__device__ __forceinline__ double field_raw_t(const FieldP& f, const double p[3]) {
  if constexpr (SEL == EV_SPHERE) {
    double c[16];
    load_params<4>(f.fq[0], c);
    return sphere_inside(c, p) ? 1.0 : 0.0;
  } else if constexpr (SEL == EV_BOX) {
    double c[16];
    load_params<16>(f.fq[0], c);
    return prim_inside(ODC_OP_BOX_SD, c, p) ? 1.0 : 0.0;
  } else if constexpr (SEL == EV_TORUS) {
    double c[16];
    load_params<5>(f.fq[0], c);
    return prim_sd(ODC_OP_TORUS_SD, c, p) < 0.0 ? 1.0 : 0.0;
  } else if constexpr (SEL == EV_BOX2F) {
    // box inside test of prim_inside, the shared rotation applied once
    double l[3] = {__dsub_rn(p[0], f.fq[0][0]), __dsub_rn(p[1], f.fq[0][1]), __dsub_rn(p[2], f.fq[0][2])};
    if (f.fq[0][6] != 0.0) {
      double R[9], o[3];
      for (int j = 0; j < 9; j++) R[j] = f.fq[0][7 + j];
      rot_rows(l, R, o);
      l[0] = o[0]; l[1] = o[1]; l[2] = o[2];
    }
    bool ia = true, ib = true;
    for (int a = 0; a < 3; a++) {
      const double al = fabs(l[a]);
      ia &= __dsub_rn(al, f.fq[0][3 + a]) < 0.0;
      ib &= __dsub_rn(al, f.fq[1][3 + a]) < 0.0;
    }
    const double A = ia ? 1.0 : 0.0;
    double B = ib ? 1.0 : 0.0;
    if (f.fop[2] == ODC_OP_RAW_MAX) return (A >= B) ? A : B;
    if (f.fop[2] == ODC_OP_RAW_MIN) return (A <= B) ? A : B;
    B = __dsub_rn(1.0, B);
    return (A <= B) ? A : B;
  } else if constexpr (SEL == EV_SPHERE2) {
    double c0[16], c1[16];
    load_params<4>(f.fq[0], c0);
    load_params<4>(f.fq[1], c1);
    const double a = sphere_inside(c0, p) ? 1.0 : 0.0;
    double b = sphere_inside(c1, p) ? 1.0 : 0.0;
    if (f.fop[2] == ODC_OP_RAW_MAX) return (a >= b) ? a : b;
    if (f.fop[2] == ODC_OP_RAW_MIN) return (a <= b) ? a : b;
    b = __dsub_rn(1.0, b);
    return (a <= b) ? a : b;
  }
  if (f.fast) {
    if constexpr (SEL == EV_SEL) {
      if (f.fast == 1) return prim_inside_p(f.fop[0], f.fq[0], p) ? 1.0 : 0.0;
      if (f.fast == 2) return smooth_raw(f.fk, prim_sd_p(f.fop[0], f.fq[0], p));
      const double a = prim_inside_p(f.fop[0], f.fq[0], p) ? 1.0 : 0.0;
      double b = prim_inside_p(f.fop[1], f.fq[1], p) ? 1.0 : 0.0;
      if (f.fop[2] == ODC_OP_RAW_MAX) return (a >= b) ? a : b;
      if (f.fop[2] == ODC_OP_RAW_MIN) return (a <= b) ? a : b;
      b = __dsub_rn(1.0, b);
      return (a <= b) ? a : b;
    } else {  // parameters by value: copied to registers (constant indices)
      double q0[16];
#pragma unroll
      for (int i = 0; i < 16; i++) q0[i] = f.fq[0][i];
      if (f.fast == 1) return prim_inside(f.fop[0], q0, p) ? 1.0 : 0.0;
      if (f.fast == 2) return smooth_raw(f.fk, prim_sd(f.fop[0], q0, p));
      double q1[16];
#pragma unroll
      for (int i = 0; i < 16; i++) q1[i] = f.fq[1][i];
      const double a = prim_inside(f.fop[0], q0, p) ? 1.0 : 0.0;
      double b = prim_inside(f.fop[1], q1, p) ? 1.0 : 0.0;
      if (f.fop[2] == ODC_OP_RAW_MAX) return (a >= b) ? a : b;
      if (f.fop[2] == ODC_OP_RAW_MIN) return (a <= b) ? a : b;
      b = __dsub_rn(1.0, b);
      return (a <= b) ? a : b;
    }
  }
  const odc_node* nd = f.nodes;
  if (f.n_nodes == 2) {
    const int op0 = __ldg(&nd[0].op), op1 = __ldg(&nd[1].op);
    if (is_prim(op0) && op1 == ODC_OP_SD2RAW) return prim_inside(op0, nd[0].p, p) ? 1.0 : 0.0;
    if (is_prim(op0) && op1 == ODC_OP_SMOOTH) return smooth_raw(__ldg(nd[1].p), prim_sd(op0, nd[0].p, p));
  } else if (f.n_nodes == 5) {
    const int op0 = __ldg(&nd[0].op), op1 = __ldg(&nd[1].op), op2 = __ldg(&nd[2].op), op3 = __ldg(&nd[3].op),
              op4 = __ldg(&nd[4].op);
    if (is_prim(op0) && op1 == ODC_OP_SD2RAW && is_prim(op2) && op3 == ODC_OP_SD2RAW &&
        (op4 == ODC_OP_RAW_MAX || op4 == ODC_OP_RAW_MIN || op4 == ODC_OP_RAW_DIFF)) {
      const double a = prim_inside(op0, nd[0].p, p) ? 1.0 : 0.0;
      double b = prim_inside(op2, nd[2].p, p) ? 1.0 : 0.0;
      if (op4 == ODC_OP_RAW_MAX) return (a >= b) ? a : b;
      if (op4 == ODC_OP_RAW_MIN) return (a <= b) ? a : b;
      b = __dsub_rn(1.0, b);
      return (a <= b) ? a : b;
    }
  }
  return field_raw_prog(f.nodes, f.n_nodes, p);
}
__device__ __forceinline__ double field_raw(const FieldP& f, const double p[3]) { return field_raw_t<EV_PARAM>(f, p); }
template <int SEL = EV_PARAM>
__device__ __forceinline__ uint32_t field_label_t(const FieldP& f, const double p[3]) {
  return field_raw_t<SEL>(f, p) > f.iso ? 1u : 0u;
}
__device__ __forceinline__ uint32_t field_label(const FieldP& f, const double p[3]) {
  return field_raw(f, p) > f.iso ? 1u : 0u;
}

// ---------------------------------------------------------------------------
// Label culling: a conservative bound of the field over a ball, used by the
// grid-label pass to decide 32 vertices of a label word with one evaluation.
//
// Every primitive is an exact signed distance (fields.py:75-139), so it is
// Lipschitz in the point with constant |R|_F per rotation applied (1 without)
// and |n| for a plane; the sd-level CSG ops (min, max, negation) and the raw
// ops (max, min, 1 - x) are monotone, so intervals propagate exactly through
// them, and the logistic of smoothed fields (fields.py:239-242) is monotone
// in sd.  A primitive's interval is its fp64 value at the centre widened by
// L * radius plus an absolute margin of 1e-9 x (1 + the magnitudes involved):
// the rounding of either evaluation is below 1e-13 of those magnitudes, so
// the interval holds the value the per-vertex evaluation computes at every
// grid vertex of the ball.  A word is decided only when the whole interval
// lies on one side of iso -- the labels are then the same bits the
// per-vertex path produces.  Returns 1 (all inside), 0 (all outside) or -1.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double frob9(const double* R) {
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 9; j++) s = fma(R[j], R[j], s);
  return sqrt(s) * (1.0 + 1e-12);
}
// interval [lo, hi] of one primitive's computed sd over the ball (see above)
__device__ __forceinline__ void prim_ball(int op, const double* qq, const double p[3], double lip, double rad,
                                          double& lo, double& hi) {
  double L = lip;
  if (op == ODC_OP_BOX_SD && qq[6] != 0.0) L *= frob9(qq + 7);
  if (op == ODC_OP_PLANE_SD) L *= sqrt(qq[3] * qq[3] + qq[4] * qq[4] + qq[5] * qq[5]) * (1.0 + 1e-12);
  const double sd = prim_sd(op, qq, p);
  const double mag = 1.0 + fabs(p[0]) + fabs(p[1]) + fabs(p[2]) + fabs(qq[0]) + fabs(qq[1]) + fabs(qq[2]) +
                     fabs(qq[3]) + fabs(qq[4]) + fabs(qq[5]);
  const double m = L * rad * (1.0 + 1e-9) + 1e-9 * mag;
  if (!(fabs(sd) < 1e300) || !(m < 1e300)) {  // undecidable: the whole real line
    lo = -1e308;
    hi = 1e308;
    return;
  }
  lo = sd - m;
  hi = sd + m;
}
// binary raw of an sd interval (SD2RAW: sd < 0 -> 1)
__device__ __forceinline__ void sd2raw_ball(double& lo, double& hi) {
  const double l = lo, h = hi;
  lo = h < 0.0 ? 1.0 : 0.0;
  hi = l >= 0.0 ? 0.0 : 1.0;
}
__device__ __forceinline__ int ball_decide(double lo, double hi, double iso) {
  if (lo > iso) return 1;
  if (hi <= iso) return 0;
  return -1;
}
// Fast paths of FieldP (parameters by value, registers only): one primitive
// -> raw or smoothed, a CSG pair of binary raws; anything else runs the
// interval interpreter below.
static __device__ __noinline__ int field_label_ball_prog(const odc_node* __restrict__ nodes, int n_nodes, double iso,
                                                       double pc0, double pc1, double pc2, double rad);
// SEL: load only the primitive's own parameters (the rest are zero in the
// node; batches read the FieldP from global memory, see field_raw_t)
template <bool SEL>
__device__ __forceinline__ void prim_ball_fp(int op, const double (&q)[16], const double pc[3], double rad,
                                             double& lo, double& hi) {
  double c[16];
  if constexpr (SEL) {
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = 0.0;
    if (op == ODC_OP_SPHERE_SD) load_params<4>(q, c);
    else if (op == ODC_OP_TORUS_SD) load_params<5>(q, c);
    else if (op == ODC_OP_PLANE_SD) load_params<6>(q, c);
    else load_params<16>(q, c);
  } else {
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = q[i];
  }
  prim_ball(op, c, pc, 1.0, rad, lo, hi);
}
// box sd (fields.py:103-111) from the box-local point: |max(q,0)| + min(max q, 0)
__device__ __forceinline__ double box_sd_local(const double l[3], const double* h) {
  double qq[3], mq[3];
  for (int a = 0; a < 3; a++) {
    qq[a] = __dsub_rn(fabs(l[a]), h[a]);
    mq[a] = qq[a] > 0.0 ? qq[a] : 0.0;
  }
  const double outside = norm3(mq);
  double mx = qq[0];
  if (qq[1] > mx) mx = qq[1];
  if (qq[2] > mx) mx = qq[2];
  const double inside = mx < 0.0 ? mx : 0.0;
  return __dadd_rn(outside, inside);
}
// EV_BOX2F ball (two boxes in one frame): the rotation and its norm once
__device__ __forceinline__ int field_label_ball_box2f(const FieldP& f, const double pc[3], double rad) {
  double l[3] = {__dsub_rn(pc[0], f.fq[0][0]), __dsub_rn(pc[1], f.fq[0][1]), __dsub_rn(pc[2], f.fq[0][2])};
  double L = 1.0;
  if (f.fq[0][6] != 0.0) {
    double R[9], o[3];
    for (int j = 0; j < 9; j++) R[j] = f.fq[0][7 + j];
    rot_rows(l, R, o);
    l[0] = o[0]; l[1] = o[1]; l[2] = o[2];
    L = frob9(R);
  }
  const double base = 1.0 + fabs(pc[0]) + fabs(pc[1]) + fabs(pc[2]) + fabs(f.fq[0][0]) + fabs(f.fq[0][1]) +
                      fabs(f.fq[0][2]);
  double lo[2], hi[2];
  for (int k = 0; k < 2; k++) {
    const double* h = &f.fq[k][3];
    const double sd = box_sd_local(l, h);
    const double m = L * rad * (1.0 + 1e-9) + 1e-9 * (base + fabs(h[0]) + fabs(h[1]) + fabs(h[2]));
    if (!(fabs(sd) < 1e300) || !(m < 1e300)) return -1;
    lo[k] = sd - m;
    hi[k] = sd + m;
    sd2raw_ball(lo[k], hi[k]);
  }
  double a0 = lo[0], a1 = hi[0], b0 = lo[1], b1 = hi[1];
  if (f.fop[2] == ODC_OP_RAW_MAX) {
    a0 = fmax(a0, b0);
    a1 = fmax(a1, b1);
  } else if (f.fop[2] == ODC_OP_RAW_MIN) {
    a0 = fmin(a0, b0);
    a1 = fmin(a1, b1);
  } else {  // min(a, 1 - b)
    const double t = __dsub_rn(1.0, b1);
    b1 = __dsub_rn(1.0, b0);
    b0 = t;
    a0 = fmin(a0, b0);
    a1 = fmin(a1, b1);
  }
  return ball_decide(a0, a1, f.iso);
}
template <bool SEL = false>
__device__ __forceinline__ int field_label_ball(const FieldP& f, const double pc[3], double rad) {
  if (f.fast) {
    double lo, hi;
    prim_ball_fp<SEL>(f.fop[0], f.fq[0], pc, rad, lo, hi);
    if (f.fast == 1) {
      sd2raw_ball(lo, hi);
    } else if (f.fast == 2) {
      const double ra = smooth_raw(f.fk, lo), rb = smooth_raw(f.fk, hi);
      lo = fmin(ra, rb) - 1e-12;
      hi = fmax(ra, rb) + 1e-12;
    } else {
      double blo, bhi;
      prim_ball_fp<SEL>(f.fop[1], f.fq[1], pc, rad, blo, bhi);
      sd2raw_ball(lo, hi);
      sd2raw_ball(blo, bhi);
      if (f.fop[2] == ODC_OP_RAW_MAX) {
        lo = fmax(lo, blo);
        hi = fmax(hi, bhi);
      } else if (f.fop[2] == ODC_OP_RAW_MIN) {
        lo = fmin(lo, blo);
        hi = fmin(hi, bhi);
      } else {  // min(a, 1 - b)
        const double t = __dsub_rn(1.0, bhi);
        bhi = __dsub_rn(1.0, blo);
        blo = t;
        lo = fmin(lo, blo);
        hi = fmin(hi, bhi);
      }
    }
    return ball_decide(lo, hi, f.iso);
  }
  return field_label_ball_prog(f.nodes, f.n_nodes, f.iso, pc[0], pc[1], pc[2], rad);
}
static __device__ __noinline__ int field_label_ball_prog(const odc_node* __restrict__ nodes, int n_nodes, double iso,
                                                       double pc0, double pc1, double pc2, double rad) {
  constexpr int kStack = 8, kPts = 4;
  double slo[kStack], shi[kStack];
  double pst[kPts][4];
  int sp = 0, pp = 0;
  double p[3] = {pc0, pc1, pc2};
  double lip = 1.0;
  for (int i = 0; i < n_nodes; i++) {
    const int op = __ldg(&nodes[i].op);
    const double* q = nodes[i].p;
    switch (op) {
      case ODC_OP_SPHERE_SD:
      case ODC_OP_BOX_SD:
      case ODC_OP_TORUS_SD:
      case ODC_OP_PLANE_SD: {
        if (sp >= kStack) return -1;
        double qq[16];
#pragma unroll
        for (int j = 0; j < 16; j++) qq[j] = __ldg(q + j);
        prim_ball(op, qq, p, lip, rad, slo[sp], shi[sp]);
        sp++;
        break;
      }
      case ODC_OP_SD2RAW: {  // fields.py:70-72: sd < 0 -> 1
        if (sp < 1) return -1;
        sd2raw_ball(slo[sp - 1], shi[sp - 1]);
        break;
      }
      case ODC_OP_RAW_MAX:
      case ODC_OP_SD_MAX:
      case ODC_OP_RAW_MIN:
      case ODC_OP_SD_MIN:
      case ODC_OP_RAW_DIFF:
      case ODC_OP_SD_DIFF: {
        if (sp < 2) return -1;
        double blo = slo[--sp], bhi = shi[sp];
        const double alo = slo[sp - 1], ahi = shi[sp - 1];
        if (op == ODC_OP_RAW_DIFF) {  // min(a, 1 - b): 1 - x is monotone under rounding
          const double t = __dsub_rn(1.0, bhi);
          bhi = __dsub_rn(1.0, blo);
          blo = t;
        } else if (op == ODC_OP_SD_DIFF) {  // max(a, -b)
          const double t = -bhi;
          bhi = -blo;
          blo = t;
        }
        const bool mx = op == ODC_OP_RAW_MAX || op == ODC_OP_SD_MAX || op == ODC_OP_SD_DIFF;
        slo[sp - 1] = mx ? fmax(alo, blo) : fmin(alo, blo);
        shi[sp - 1] = mx ? fmax(ahi, bhi) : fmin(ahi, bhi);
        break;
      }
      case ODC_OP_RAW_COMPL: {
        if (sp < 1) return -1;
        const double t = __dsub_rn(1.0, shi[sp - 1]);
        shi[sp - 1] = __dsub_rn(1.0, slo[sp - 1]);
        slo[sp - 1] = t;
        break;
      }
      case ODC_OP_SD_NEG: {
        if (sp < 1) return -1;
        const double t = -shi[sp - 1];
        shi[sp - 1] = -slo[sp - 1];
        slo[sp - 1] = t;
        break;
      }
      case ODC_OP_XFORM_BEGIN: {  // (p - t) @ R, fields.py:176-180
        if (pp >= kPts) return -1;
        pst[pp][0] = p[0];
        pst[pp][1] = p[1];
        pst[pp][2] = p[2];
        pst[pp][3] = lip;
        pp++;
        double l[3] = {__dsub_rn(p[0], __ldg(q)), __dsub_rn(p[1], __ldg(q + 1)), __dsub_rn(p[2], __ldg(q + 2))};
        if (__ldg(q + 6) != 0.0) {
          double R[9], o[3];
          for (int j = 0; j < 9; j++) R[j] = __ldg(q + 7 + j);
          rot_rows(l, R, o);
          l[0] = o[0]; l[1] = o[1]; l[2] = o[2];
          lip *= frob9(R);
        }
        p[0] = l[0]; p[1] = l[1]; p[2] = l[2];
        break;
      }
      case ODC_OP_XFORM_END:
        if (pp < 1) return -1;
        pp--;
        p[0] = pst[pp][0]; p[1] = pst[pp][1]; p[2] = pst[pp][2];
        lip = pst[pp][3];
        break;
      case ODC_OP_SMOOTH: {  // 1 / (1 + exp(clip(k sd))): monotone in sd
        if (sp < 1) return -1;
        const double k = __ldg(q);
        const double ra = smooth_raw(k, slo[sp - 1]), rb = smooth_raw(k, shi[sp - 1]);
        slo[sp - 1] = fmin(ra, rb) - 1e-12;
        shi[sp - 1] = fmax(ra, rb) + 1e-12;
        break;
      }
      default: return -1;
    }
  }
  if (sp < 1) return -1;
  return ball_decide(slo[sp - 1], shi[sp - 1], iso);
}

// Registers-only test for the common vertex: its fan is one disc.  With
// the two other vertices (a_i, b_i) of each of its nt <= kDiscMax incident
// triangles, walk from triangle 0 across b_0, each step to the other
// triangle holding the shared neighbour; the fan is one closed disc exactly
// when every neighbour met on the walk sits in exactly two triangles and the
// walk returns to triangle 0 after nt steps (then every edge (v,u) has two
// triangles -- no sheet pairing, polygonize.py:279-305 -- and the union-find
// of polygonize.py:308-347 finds one component: no new vertex).  Anything
// else (boundary, >2-triangle edges, several components, degenerate
// triangles) takes the general path.
constexpr int kDiscMax = 12;
__device__ __forceinline__ bool fan_is_disc(const int32_t* __restrict__ tris, const uint32_t* __restrict__ off,
                                            const int32_t* __restrict__ inc, int64_t v) {
  const uint32_t b0 = off[v];
  const int nt = (int)(off[v + 1] - b0);
  if (nt < 3 || nt > kDiscMax) return false;
  const int32_t vv = (int32_t)v;
  int32_t A[kDiscMax], B[kDiscMax];
  bool ok = true;
#pragma unroll
  for (int i = 0; i < kDiscMax; i++) {
    A[i] = -1 - 2 * i;  // sentinels: negative, pairwise distinct
    B[i] = -2 - 2 * i;
    if (i < nt) {
      const int64_t t = inc[b0 + i];
      const int32_t t0 = tris[3 * t], t1 = tris[3 * t + 1], t2 = tris[3 * t + 2];
      const int hits = (t0 == vv) + (t1 == vv) + (t2 == vv);
      ok &= hits == 1;
      A[i] = t0 == vv ? t1 : (t1 == vv ? t2 : t0);
      B[i] = t0 == vv ? t2 : (t1 == vv ? t0 : t1);
      ok &= A[i] != B[i];
    }
  }
  if (!ok) return false;
  int cur = 0;
  int32_t via = B[0];
#pragma unroll
  for (int step = 0; step < kDiscMax; step++) {
    if (step < nt) {
      int cnt = 0, nxt = -1;
      int32_t nvia = 0;
#pragma unroll
      for (int j = 0; j < kDiscMax; j++) {
        const bool ia = A[j] == via, ib = B[j] == via;
        cnt += (int)ia + (int)ib;
        if (j != cur && (ia || ib)) {
          nxt = j;
          nvia = ia ? B[j] : A[j];
        }
      }
      if (cnt != 2 || nxt < 0) return false;
      if (nxt == 0 && step != nt - 1) return false;  // a shorter cycle: several components
      cur = nxt;
      via = nvia;
    }
  }
  return cur == 0;
}

// device-side status word (errors raised inside kernels)
struct DevStatus {
  int32_t code;     // ODC_E_*
  int32_t pad;
  int64_t detail;   // offending element
};
// The reference raises at the first offending element in index order
// (numpy finds the first), so the detail is the smallest index reported
// (detail starts at INT64_MAX, see extract()).
__device__ __forceinline__ void raise_status(DevStatus* st, int code, int64_t detail) {
  atomicCAS(&st->code, 0, code);
  atomicMin(reinterpret_cast<unsigned long long*>(&st->detail), (unsigned long long)detail);
}

}  // namespace odc
