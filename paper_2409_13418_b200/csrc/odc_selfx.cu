// odc_selfx.cu -- triangle-pair self-intersection count on the device
// (occmesh.mesh.count_self_intersections, /root/reference/pkg/src/occmesh/
// mesh.py:395-487, with _tri_tri_cross :300-349 and _coplanar_overlap_area
// :368-392).  SURVEY 8(f) item 2.
//
// Same steps, same fp64 arithmetic order (numpy: no FMA, textbook cross,
// norm = sqrt((x0^2 + x1^2) + x2^2), 3-term einsum = (p0 + p2) + p1), so
// every tolerance decision is taken on the same double values:
//   1. normalise into the unit box (lo = per-axis min, extent = max span);
//   2. per triangle: corners, area (degenerate below 1e-20), bounding box;
//   3. uniform hash: cell = max(1.0001 * largest box side, 1e-9); each
//      triangle lands in the <= 8 cells of its box corners;
//   4. radix sort (cell key, triangle); every pair inside a cell is a
//      candidate, emitted once -- in the smallest cell the two share;
//   5. drop pairs sharing a vertex, with a degenerate triangle, or whose
//      boxes are apart by more than the tolerance; exact interval test;
//      coplanar pairs count when their overlap area exceeds the tolerance;
//   6. hits sorted by (a, b).
// CUB's radix sort is the only library call (step 4 and 6).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "odc_kernels.h"

namespace odc {

namespace {
inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

struct V3 {
  double x, y, z;
};
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 crs(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double dot_e(V3 a, V3 b) { return (a.x * b.x + a.z * b.z) + a.y * b.y; }
__device__ __forceinline__ double nrm(V3 a) { return sqrt((a.x * a.x + a.y * a.y) + a.z * a.z); }
__device__ __forceinline__ double comp(V3 a, int k) { return k == 0 ? a.x : (k == 1 ? a.y : a.z); }
// numpy minimum / maximum: NaN propagates
__device__ __forceinline__ double np_min(double a, double b) { return (isnan(a) || isnan(b)) ? NAN : (a < b ? a : b); }
__device__ __forceinline__ double np_max(double a, double b) { return (isnan(a) || isnan(b)) ? NAN : (a > b ? a : b); }

// order-preserving map of doubles onto uint64 (for atomic min/max)
__device__ __forceinline__ unsigned long long ord_of(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double of_ord(unsigned long long o) {
  const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  return __longlong_as_double((long long)b);
}
}  // namespace

// stats: [0..2] min ord, [3..5] max ord of vertex coordinates; [6] max box side ord
__global__ void k_sx_bounds(const double* __restrict__ v, int64_t nv, unsigned long long* __restrict__ st) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const double x = v[3 * i + a];
      lo[a] = x < lo[a] ? x : lo[a];
      hi[a] = x > hi[a] ? x : hi[a];
    }
#pragma unroll
  for (int a = 0; a < 3; a++) {
    atomicMin(&st[a], ord_of(lo[a]));
    atomicMax(&st[3 + a], ord_of(hi[a]));
  }
}

// per triangle: normalised corners (9), box (6), degenerate flag; max box side
__global__ void k_sx_tris(const double* __restrict__ v, const int32_t* __restrict__ t, int64_t nt,
                          unsigned long long* __restrict__ st, double* __restrict__ corners,
                          double* __restrict__ box, uint8_t* __restrict__ degen) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double side = -INFINITY;
  if (i < nt) {
    const double lo[3] = {of_ord(st[0]), of_ord(st[1]), of_ord(st[2])};
    double ext = 0.0;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const double e = of_ord(st[3 + a]) - lo[a];
      ext = (a == 0 || e > ext) ? e : ext;  // (max - lo).max()
    }
    if (ext == 0.0) ext = 1.0;  // "or 1.0"
    V3 c[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const int64_t vi = t[3 * i + k];
      c[k] = {(v[3 * vi] - lo[0]) / ext, (v[3 * vi + 1] - lo[1]) / ext, (v[3 * vi + 2] - lo[2]) / ext};
      corners[9 * i + 3 * k] = c[k].x;
      corners[9 * i + 3 * k + 1] = c[k].y;
      corners[9 * i + 3 * k + 2] = c[k].z;
    }
    const double area = 0.5 * nrm(crs(sub(c[1], c[0]), sub(c[2], c[0])));
    degen[i] = area < 1e-20;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const double x0 = comp(c[0], a), x1 = comp(c[1], a), x2 = comp(c[2], a);
      const double mn = np_min(np_min(x0, x1), x2), mx = np_max(np_max(x0, x1), x2);
      box[6 * i + a] = mn;
      box[6 * i + 3 + a] = mx;
      const double s = mx - mn;
      side = s > side ? s : side;
    }
  }
  // block max, one atomic per block
  __shared__ unsigned long long red[32];
  unsigned long long o = ord_of(side);
  for (int d = 16; d; d >>= 1) {
    const unsigned long long p = __shfl_down_sync(0xffffffffu, o, d);
    o = p > o ? p : o;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = o;
  __syncthreads();
  if (threadIdx.x < 32) {
    o = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ull;
    for (int d = 16; d; d >>= 1) {
      const unsigned long long p = __shfl_down_sync(0xffffffffu, o, d);
      o = p > o ? p : o;
    }
    if (threadIdx.x == 0) atomicMax(&st[6], o);
  }
}

struct CellGrid {
  double cell;
  int64_t n_side;
};
__device__ __forceinline__ CellGrid cell_grid(const unsigned long long* st) {
  const double span = of_ord(st[6]);
  const double a = span * 1.0001;
  CellGrid g;
  g.cell = a > 1e-9 ? a : 1e-9;
  g.n_side = (int64_t)(1.0 / g.cell) + 3;
  return g;
}
// the <= 8 distinct cell keys of a box (numpy int64 arithmetic wraps)
__device__ __forceinline__ int cell_keys(const double* b, CellGrid g, int64_t* k) {
  int64_t lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    lo[a] = (int64_t)floor(b[a] / g.cell);
    hi[a] = (int64_t)floor(b[3 + a] / g.cell);
  }
  int n = 0;
  for (int c = 0; c < 8; c++) {
    const uint64_t ix = (uint64_t)((c & 4) ? hi[0] : lo[0]), iy = (uint64_t)((c & 2) ? hi[1] : lo[1]),
                   iz = (uint64_t)((c & 1) ? hi[2] : lo[2]);
    const int64_t key = (int64_t)((ix * (uint64_t)g.n_side + iy) * (uint64_t)g.n_side + iz);
    bool dup = false;
    for (int j = 0; j < n; j++) dup |= k[j] == key;
    if (!dup) k[n++] = key;
  }
  return n;
}

__global__ void k_sx_keys(int64_t nt, const unsigned long long* __restrict__ st, const double* __restrict__ box,
                          int64_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  int64_t k[8];
  const int n = cell_keys(box + 6 * i, cell_grid(st), k);
  for (int c = 0; c < 8; c++) {
    keys[8 * i + c] = c < n ? k[c] : INT64_MAX;  // padding sorts last, never paired
    vals[8 * i + c] = (int32_t)i;
  }
}

namespace {
// _tri_tri_cross (mesh.py:300-349) for one pair: bit 0 crossing, bit 1 coplanar
__device__ int tri_tri(const double* P, const double* Q, double tol) {
  const V3 p0{P[0], P[1], P[2]}, p1{P[3], P[4], P[5]}, p2{P[6], P[7], P[8]};
  const V3 q0{Q[0], Q[1], Q[2]}, q1{Q[3], Q[4], Q[5]}, q2{Q[6], Q[7], Q[8]};
  const V3 n1 = crs(sub(p1, p0), sub(p2, p0)), n2 = crs(sub(q1, q0), sub(q2, q0));
  const double dq[3] = {dot_e(sub(q0, p0), n1), dot_e(sub(q1, p0), n1), dot_e(sub(q2, p0), n1)};
  const double dp[3] = {dot_e(sub(p0, q0), n2), dot_e(sub(p1, q0), n2), dot_e(sub(p2, q0), n2)};
  const double s1 = nrm(n1), s2 = nrm(n2);
  const double tq = tol * np_max(s1, 1e-300), tp = tol * np_max(s2, 1e-300);
  const bool sep = (dq[0] > tq && dq[1] > tq && dq[2] > tq) || (dq[0] < -tq && dq[1] < -tq && dq[2] < -tq) ||
                   (dp[0] > tp && dp[1] > tp && dp[2] > tp) || (dp[0] < -tp && dp[1] < -tp && dp[2] < -tp);
  const bool copl = fabs(dq[0]) <= tq && fabs(dq[1]) <= tq && fabs(dq[2]) <= tq && fabs(dp[0]) <= tp &&
                    fabs(dp[1]) <= tp && fabs(dp[2]) <= tp;
  if (sep) return 0;
  if (copl) return 2;
  const V3 d = crs(n1, n2);
  const double ad[3] = {fabs(d.x), fabs(d.y), fabs(d.z)};
  const int ax = (ad[1] > ad[0]) ? ((ad[2] > ad[1]) ? 2 : 1) : ((ad[2] > ad[0]) ? 2 : 0);  // first argmax
  auto interval = [&](V3 a, V3 b, V3 c, const double* dist, double tl, double& lo, double& hi) {
    const double pr[3] = {comp(a, ax), comp(b, ax), comp(c, ax)};
    int sg[3];
#pragma unroll
    for (int i = 0; i < 3; i++) sg[i] = dist[i] > tl ? 1 : -1;
    lo = INFINITY;
    hi = -INFINITY;
#pragma unroll
    for (int i = 0; i < 3; i++) {
      const int j = (i + 1) % 3;
      if (sg[i] * sg[j] < 0) {
        const double df = dist[i] - dist[j];
        const double den = fabs(df) < 1e-300 ? 1.0 : df;
        const double tt = pr[i] + (pr[j] - pr[i]) * (dist[i] / den);
        lo = np_min(lo, tt);
        hi = np_max(hi, tt);
      }
    }
  };
  double lo1, hi1, lo2, hi2;
  interval(q0, q1, q2, dq, tq, lo1, hi1);
  interval(p0, p1, p2, dp, tp, lo2, hi2);
  const double ov = np_min(hi1, hi2) - np_max(lo1, lo2);
  return (ov > tol && isfinite(ov)) ? 1 : 0;
}

struct P2 {
  double x, y;
};
// _clip_polygon (mesh.py:352-365): keep the left side of a -> b
__device__ int clip(const P2* in, int n, P2 a, P2 b, P2* out) {
  int m = 0;
  for (int i = 0; i < n; i++) {
    const P2 cur = in[i], nxt = in[(i + 1) % n];
    const double sc = (b.x - a.x) * (cur.y - a.y) - (b.y - a.y) * (cur.x - a.x);
    const double sn = (b.x - a.x) * (nxt.y - a.y) - (b.y - a.y) * (nxt.x - a.x);
    if (sc >= 0) out[m++] = cur;
    if (sc * sn < 0) {
      const double tt = sc / (sc - sn);
      out[m++] = {cur.x + tt * (nxt.x - cur.x), cur.y + tt * (nxt.y - cur.y)};
    }
  }
  return m;
}
// _coplanar_overlap_area (mesh.py:368-392)
__device__ double coplanar_area(const double* P, const double* Q) {
  const V3 p0{P[0], P[1], P[2]}, p1{P[3], P[4], P[5]}, p2{P[6], P[7], P[8]};
  const V3 n = crs(sub(p1, p0), sub(p2, p0));
  const double an[3] = {fabs(n.x), fabs(n.y), fabs(n.z)};
  const int ax = (an[1] > an[0]) ? ((an[2] > an[1]) ? 2 : 1) : ((an[2] > an[0]) ? 2 : 0);
  const int k0 = ax == 0 ? 1 : 0, k1 = ax == 2 ? 1 : 2;
  P2 a[3], b[3];
  for (int i = 0; i < 3; i++) {
    a[i] = {P[3 * i + k0], P[3 * i + k1]};
    b[i] = {Q[3 * i + k0], Q[3 * i + k1]};
  }
  if (comp(n, ax) < 0) {
    const P2 s = a[0];
    a[0] = a[2];
    a[2] = s;
  }
  const double nb = (b[1].x - b[0].x) * (b[2].y - b[0].y) - (b[1].y - b[0].y) * (b[2].x - b[0].x);
  if (nb < 0) {
    const P2 s = b[0];
    b[0] = b[2];
    b[2] = s;
  }
  P2 buf0[12], buf1[12];
  int m = 3;
  for (int i = 0; i < 3; i++) buf0[i] = b[i];
  P2* cur = buf0;
  P2* nxt = buf1;
  for (int i = 0; i < 3; i++) {
    m = clip(cur, m, a[i], a[(i + 1) % 3], nxt);
    P2* s = cur;
    cur = nxt;
    nxt = s;
    if (m < 3) return 0.0;
  }
  double area = 0.0;
  for (int i = 1; i < m - 1; i++)
    area += 0.5 * fabs((cur[i].x - cur[0].x) * (cur[i + 1].y - cur[0].y) -
                       (cur[i + 1].x - cur[0].x) * (cur[i].y - cur[0].y));
  return area;
}
}  // namespace

// every candidate pair in a cell, tested once (in the smallest shared cell)
__global__ void k_sx_pairs(int64_t n, const int64_t* __restrict__ keys, const int32_t* __restrict__ vals,
                           const unsigned long long* __restrict__ st, const int32_t* __restrict__ tris,
                           const double* __restrict__ corners, const double* __restrict__ box,
                           const uint8_t* __restrict__ degen, double tol, int64_t nt,
                           unsigned long long* __restrict__ n_hits, int64_t* __restrict__ hits, int64_t cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t key = keys[i];
  if (key == INT64_MAX) return;
  const CellGrid g = cell_grid(st);
  const int32_t ti = vals[i];
  for (int64_t j = i + 1; j < n && keys[j] == key; j++) {
    const int32_t tj = vals[j];
    const int32_t a = ti < tj ? ti : tj, b = ti < tj ? tj : ti;
    if (degen[a] || degen[b]) continue;
    bool share = false;
    for (int u = 0; u < 3; u++)
      for (int w = 0; w < 3; w++) share |= tris[3 * (int64_t)a + u] == tris[3 * (int64_t)b + w];
    if (share) continue;
    const double* ba = box + 6 * (int64_t)a;
    const double* bb = box + 6 * (int64_t)b;
    bool ovl = true;
    for (int ax = 0; ax < 3; ax++) ovl &= (ba[ax] <= bb[3 + ax] + tol) && (bb[ax] <= ba[3 + ax] + tol);
    if (!ovl) continue;
    // emitted once: only in the smallest cell key the two triangles share
    int64_t ka[8], kb[8];
    const int na = cell_keys(ba, g, ka), nbk = cell_keys(bb, g, kb);
    int64_t first = INT64_MAX;
    for (int u = 0; u < na; u++)
      for (int w = 0; w < nbk; w++)
        if (ka[u] == kb[w] && ka[u] < first) first = ka[u];
    if (first != key) continue;
    const int r = tri_tri(corners + 9 * (int64_t)a, corners + 9 * (int64_t)b, tol);
    const bool hit = r == 1 || (r == 2 && coplanar_area(corners + 9 * (int64_t)a, corners + 9 * (int64_t)b) > tol);
    if (hit) {
      const unsigned long long slot = atomicAdd(n_hits, 1ull);
      if ((int64_t)slot < cap) hits[slot] = (int64_t)a * nt + b;
    }
  }
}

// Host driver; all buffers from the caller's allocator (workspace callback).
int self_intersections(const double* d_v, int64_t nv, const int32_t* d_t, int64_t nt, double tol,
                       void* (*alloc)(void*, size_t), void* actx, cudaStream_t s, int64_t* d_out_hits,
                       int64_t cap, int64_t* n_hits_host) {
  unsigned long long* st = (unsigned long long*)alloc(actx, 8 * 8);
  double* corners = (double*)alloc(actx, 72 * nt);
  double* box = (double*)alloc(actx, 48 * nt);
  uint8_t* degen = (uint8_t*)alloc(actx, nt);
  int64_t* keys = (int64_t*)alloc(actx, 64 * nt);
  int64_t* keys2 = (int64_t*)alloc(actx, 64 * nt);
  int32_t* vals = (int32_t*)alloc(actx, 32 * nt);
  int32_t* vals2 = (int32_t*)alloc(actx, 32 * nt);
  if (!st || !corners || !box || !degen || !keys || !keys2 || !vals || !vals2) return ODC_E_NOMEM;
  const unsigned long long init[8] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
  if (cudaMemcpyAsync(st, init, sizeof init, cudaMemcpyHostToDevice, s) != cudaSuccess) return ODC_E_CUDA;
  k_sx_bounds<<<592, 256, 0, s>>>(d_v, nv, st);
  k_sx_tris<<<grid_for(nt, 256), 256, 0, s>>>(d_v, d_t, nt, st, corners, box, degen);
  k_sx_keys<<<grid_for(nt, 256), 256, 0, s>>>(nt, st, box, keys, vals);
  const int64_t n = 8 * nt;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, vals, vals2, (int)n, 0, 64, s);
  void* tmp = alloc(actx, tmp_bytes);
  if (!tmp) return ODC_E_NOMEM;
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, vals2, (int)n, 0, 64, s);
  unsigned long long* cnt = st + 7;
  k_sx_pairs<<<grid_for(n, 128), 128, 0, s>>>(n, keys2, vals2, st, d_t, corners, box, degen, tol, nt, cnt,
                                              d_out_hits, cap);
  unsigned long long h = 0;
  if (cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return ODC_E_CUDA;
  *n_hits_host = (int64_t)h;
  if ((int64_t)h > cap) return ODC_OK;  // caller re-runs with a larger buffer
  if (h > 1) {  // sort the hit keys a * nt + b
    int64_t* sorted = (int64_t*)alloc(actx, 8 * h);
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, d_out_hits, sorted, (int)h, 0, 64, s);
    void* t2 = alloc(actx, tb);
    if (!sorted || !t2) return ODC_E_NOMEM;
    cub::DeviceRadixSort::SortKeys(t2, tb, d_out_hits, sorted, (int)h, 0, 64, s);
    if (cudaMemcpyAsync(d_out_hits, sorted, 8 * h, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return ODC_E_CUDA;
  }
  return cudaGetLastError() == cudaSuccess ? ODC_OK : ODC_E_CUDA;
}

}  // namespace odc
