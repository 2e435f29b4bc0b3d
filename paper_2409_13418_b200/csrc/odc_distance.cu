// odc_distance.cu -- exact point-to-mesh distance queries on the device
// (occmesh.mesh.MeshDistanceIndex.query, /root/reference/pkg/src/occmesh/
// mesh.py:202-270, with _closest_point_on_triangles :153-199), the kernel
// behind the distance metrics MD2 / HDD / NIC (metrics.py:26-70).
//
// Broad phase: a uniform grid over the triangles' bounding box; every
// triangle is listed in each cell its box overlaps (CSR).  A query walks
// cubic shells of cells around its own cell and stops once the nearest
// unexplored cell is farther than the best distance found, so the result is
// the exact minimum over all triangles (like the reference's conservative
// KD-tree prune).  The per-triangle closest point is Ericson's region walk
// in numpy's fp64 order (3-term einsum = (p0 + p2) + p1, no FMA: this TU is
// built with --fmad=false), so distances equal the reference's bit for bit,
// and exact ties resolve like the reference's k-nearest-centroid pass.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>

#include "odc_kernels.h"

namespace odc {

namespace {
inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 operator-(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ D3 operator+(D3 a, D3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ D3 operator*(D3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ double ein(D3 a, D3 b) { return (a.x * b.x + a.z * b.z) + a.y * b.y; }
__device__ __forceinline__ double clip01(double t) {
  if (isnan(t)) return t;
  return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
}
__device__ __forceinline__ double nz(double d) { return fabs(d) < 1e-300 ? 1.0 : d; }

// _closest_point_on_triangles for one (point, triangle): first matching region wins
__device__ D3 closest_on_tri(D3 p, D3 a, D3 b, D3 c) {
  const D3 ab = b - a, ac = c - a, ap = p - a;
  const double d1 = ein(ab, ap), d2 = ein(ac, ap);
  const D3 bp = p - b;
  const double d3 = ein(ab, bp), d4 = ein(ac, bp);
  const D3 cp = p - c;
  const double d5 = ein(ab, cp), d6 = ein(ac, cp);
  const double vc = d1 * d4 - d3 * d2, vb = d5 * d2 - d1 * d6, va = d3 * d6 - d5 * d4;
  if (d1 <= 0 && d2 <= 0) return a;
  if (d3 >= 0 && d4 <= d3) return b;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) return a + ab * clip01(d1 / nz(d1 - d3));
  if (d6 >= 0 && d5 <= d6) return c;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) return a + ac * clip01(d2 / nz(d2 - d6));
  const double e43 = d4 - d3, e56 = d5 - d6;
  if (va <= 0 && e43 >= 0 && e56 >= 0) return b + (c - b) * clip01(e43 / nz(e43 + e56));
  const double den = nz((va + vb) + vc);
  const double v = vb / den, w = vc / den;
  return (a + ab * v) + ac * w;
}

__device__ __forceinline__ unsigned long long ord_of(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
}  // namespace

struct DistGrid {
  double lo[3], h;
  int32_t n[3];
};

// bounding box (st[0..5], ord-mapped) and the sum of triangle box max sides (st[6], double bits)
__global__ void k_dist_bounds(const double* __restrict__ v, const int32_t* __restrict__ t, int64_t nt,
                              unsigned long long* __restrict__ st, double* __restrict__ side_sum) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int k = 0; k < 3; k++) {
    const int64_t vi = t[3 * i + k];
    for (int a = 0; a < 3; a++) {
      const double x = v[3 * vi + a];
      lo[a] = fmin(lo[a], x);
      hi[a] = fmax(hi[a], x);
    }
  }
  double side = 0.0;
  for (int a = 0; a < 3; a++) {
    atomicMin(&st[a], ord_of(lo[a]));
    atomicMax(&st[3 + a], ord_of(hi[a]));
    side = fmax(side, hi[a] - lo[a]);
  }
  atomicAdd(side_sum, side);
}

__device__ __forceinline__ void tri_cells(const double* v, const int32_t* t, int64_t i, const DistGrid& g, int c0[3],
                                          int c1[3]) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int k = 0; k < 3; k++) {
    const int64_t vi = t[3 * i + k];
    for (int a = 0; a < 3; a++) {
      const double x = v[3 * vi + a];
      lo[a] = fmin(lo[a], x);
      hi[a] = fmax(hi[a], x);
    }
  }
  for (int a = 0; a < 3; a++) {
    c0[a] = min(max((int)floor((lo[a] - g.lo[a]) / g.h), 0), g.n[a] - 1);
    c1[a] = min(max((int)floor((hi[a] - g.lo[a]) / g.h), 0), g.n[a] - 1);
  }
}

__global__ void k_dist_count(const double* __restrict__ v, const int32_t* __restrict__ t, int64_t nt, DistGrid g,
                             uint32_t* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  int c0[3], c1[3];
  tri_cells(v, t, i, g, c0, c1);
  for (int z = c0[2]; z <= c1[2]; z++)
    for (int y = c0[1]; y <= c1[1]; y++)
      for (int x = c0[0]; x <= c1[0]; x++) atomicAdd(&cnt[((int64_t)z * g.n[1] + y) * g.n[0] + x], 1u);
}

__global__ void k_dist_fill(const double* __restrict__ v, const int32_t* __restrict__ t, int64_t nt, DistGrid g,
                            const uint32_t* __restrict__ off, uint32_t* __restrict__ cursor,
                            int32_t* __restrict__ items) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  int c0[3], c1[3];
  tri_cells(v, t, i, g, c0, c1);
  for (int z = c0[2]; z <= c1[2]; z++)
    for (int y = c0[1]; y <= c1[1]; y++)
      for (int x = c0[0]; x <= c1[0]; x++) {
        const int64_t c = ((int64_t)z * g.n[1] + y) * g.n[0] + x;
        items[off[c] + atomicAdd(&cursor[c], 1u)] = (int32_t)i;
      }
}

__device__ __forceinline__ D3 corner(const double* v, const int32_t* t, int32_t ti, int k) {
  const int64_t vi = t[3 * (int64_t)ti + k];
  return {v[3 * vi], v[3 * vi + 1], v[3 * vi + 2]};
}
__device__ __forceinline__ double tri_dist(D3 p, const double* v, const int32_t* t, int32_t ti, D3& cp) {
  cp = closest_on_tri(p, corner(v, t, ti, 0), corner(v, t, ti, 1), corner(v, t, ti, 2));
  const D3 d = cp - p;
  return sqrt((d.x * d.x + d.y * d.y) + d.z * d.z);
}

// Exact nearest triangle.  The winner among exact distance ties follows the
// reference's two passes (mesh.py:232-268): the first of the k = min(8, T)
// nearest triangle centroids (numpy mean, squared distance summed x, y, z)
// that attains the minimum, else the smallest attaining index.
__global__ void k_dist_query(const double* __restrict__ v, const int32_t* __restrict__ t, int64_t nt, DistGrid g,
                             const uint32_t* __restrict__ off, const int32_t* __restrict__ items,
                             const double* __restrict__ q, int64_t nq, double* __restrict__ dist,
                             int64_t* __restrict__ tri, double* __restrict__ cpo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq) return;
  const D3 p{q[3 * i], q[3 * i + 1], q[3 * i + 2]};
  const double pc[3] = {p.x, p.y, p.z};
  int c[3];
  for (int a = 0; a < 3; a++) c[a] = min(max((int)floor((pc[a] - g.lo[a]) / g.h), 0), g.n[a] - 1);
  const int K = nt < 8 ? (int)nt : 8;
  double kd[8];
  int32_t kt[8];
  int nk = 0;
  double best = INFINITY;
  int32_t bt = -1;
  const int rmax = max(g.n[0], max(g.n[1], g.n[2]));
  for (int r = 0; r <= rmax; r++) {
    for (int z = c[2] - r; z <= c[2] + r; z++) {
      if (z < 0 || z >= g.n[2]) continue;
      for (int y = c[1] - r; y <= c[1] + r; y++) {
        if (y < 0 || y >= g.n[1]) continue;
        const bool face = z == c[2] - r || z == c[2] + r || y == c[1] - r || y == c[1] + r;
        for (int x = c[0] - r; x <= c[0] + r; x += (face ? 1 : 2 * r > 0 ? 2 * r : 1)) {
          if (x < 0 || x >= g.n[0]) continue;
          const int64_t cell = ((int64_t)z * g.n[1] + y) * g.n[0] + x;
          for (uint32_t k = off[cell]; k < off[cell + 1]; k++) {
            const int32_t ti = items[k];
            const D3 A = corner(v, t, ti, 0), B = corner(v, t, ti, 1), C = corner(v, t, ti, 2);
            const D3 cp = closest_on_tri(p, A, B, C);
            const D3 d = cp - p;
            const double dd = sqrt((d.x * d.x + d.y * d.y) + d.z * d.z);
            if (dd < best || (dd == best && ti < bt)) {
              best = dd;
              bt = ti;
            }
            // centroid, counted in its home cell only
            const D3 m{((A.x + B.x) + C.x) / 3.0, ((A.y + B.y) + C.y) / 3.0, ((A.z + B.z) + C.z) / 3.0};
            const double mc[3] = {m.x, m.y, m.z};
            bool home = true;
            const int cc[3] = {x, y, z};
            for (int a = 0; a < 3; a++)
              home &= min(max((int)floor((mc[a] - g.lo[a]) / g.h), 0), g.n[a] - 1) == cc[a];
            if (!home) continue;
            const D3 e = m - p;
            const double d2 = (e.x * e.x + e.y * e.y) + e.z * e.z;
            if (nk < K || d2 < kd[nk - 1] || (d2 == kd[nk - 1] && ti < kt[nk - 1])) {  // ties: lower index first
              int j = nk < K ? nk++ : K - 1;
              while (j > 0 && (kd[j - 1] > d2 || (kd[j - 1] == d2 && kt[j - 1] > ti))) {
                kd[j] = kd[j - 1];
                kt[j] = kt[j - 1];
                j--;
              }
              kd[j] = d2;
              kt[j] = ti;
            }
          }
        }
      }
    }
    // distance from p to the cells not yet explored (open sides only)
    double gap = INFINITY;
    bool all = true;
    for (int a = 0; a < 3; a++) {
      if (c[a] - r > 0) {
        all = false;
        gap = fmin(gap, fmax(0.0, pc[a] - (g.lo[a] + (c[a] - r) * g.h)));
      }
      if (c[a] + r < g.n[a] - 1) {
        all = false;
        gap = fmin(gap, fmax(0.0, (g.lo[a] + (c[a] + r + 1) * g.h) - pc[a]));
      }
    }
    if (all || (best < gap && nk == K && kd[K - 1] < gap * gap)) break;
  }
  int32_t win = bt;
  for (int j = 0; j < nk; j++) {
    D3 cp;
    if (tri_dist(p, v, t, kt[j], cp) == best) {
      win = kt[j];
      break;
    }
  }
  D3 cp;
  dist[i] = tri_dist(p, v, t, win, cp);
  tri[i] = win;
  cpo[3 * i] = cp.x;
  cpo[3 * i + 1] = cp.y;
  cpo[3 * i + 2] = cp.z;
}

// TriangleMesh.areas (mesh.py:57-61): 0.5 * norm(cross(c1 - c0, c2 - c0)),
// numpy's arithmetic order, so the values equal numpy's bit for bit
__global__ void k_tri_areas(const double* __restrict__ v, const int32_t* __restrict__ t, int64_t nt,
                            double* __restrict__ area) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const D3 a = corner(v, t, (int32_t)i, 0), b = corner(v, t, (int32_t)i, 1), c = corner(v, t, (int32_t)i, 2);
  const D3 u = b - a, w = c - a;
  const D3 n{u.y * w.z - u.z * w.y, u.z * w.x - u.x * w.z, u.x * w.y - u.y * w.x};
  area[i] = 0.5 * sqrt((n.x * n.x + n.y * n.y) + n.z * n.z);
}
void launch_tri_areas(const double* v, const int32_t* t, int64_t nt, double* area, cudaStream_t s) {
  if (nt) k_tri_areas<<<grid_for(nt, 256), 256, 0, s>>>(v, t, nt, area);
}

int mesh_distance(const double* d_v, const int32_t* d_t, int64_t nt, const double* d_q, int64_t nq,
                  void* (*alloc)(void*, size_t), void* actx, cudaStream_t s, double* d_dist, int64_t* d_tri,
                  double* d_cp) {
  unsigned long long* st = (unsigned long long*)alloc(actx, 64);
  double* side_sum = (double*)alloc(actx, 8);
  if (!st || !side_sum) return ODC_E_NOMEM;
  const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
  if (cudaMemcpyAsync(st, init, sizeof init, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemsetAsync(side_sum, 0, 8, s) != cudaSuccess)
    return ODC_E_CUDA;
  k_dist_bounds<<<grid_for(nt, 256), 256, 0, s>>>(d_v, d_t, nt, st, side_sum);
  unsigned long long h_st[6];
  double h_side = 0;
  if (cudaMemcpyAsync(h_st, st, sizeof h_st, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(&h_side, side_sum, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return ODC_E_CUDA;
  auto host_of_ord = [](unsigned long long o) {
    const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
    double d;
    memcpy(&d, &b, 8);
    return d;
  };
  DistGrid g;
  double ext = 0;
  for (int a = 0; a < 3; a++) {
    g.lo[a] = host_of_ord(h_st[a]);
    ext = fmax(ext, host_of_ord(h_st[3 + a]) - g.lo[a]);
  }
  // cells about twice the mean triangle size, at most 2^24 cells in all
  double hcell = 2.0 * h_side / (double)nt;
  if (!(hcell > 0)) hcell = ext > 0 ? ext : 1.0;
  for (;;) {
    int64_t total = 1;
    for (int a = 0; a < 3; a++) {
      const double e = host_of_ord(h_st[3 + a]) - g.lo[a];
      g.n[a] = (int32_t)fmin(fmax(ceil(e / hcell), 1.0), 4096.0);
      total *= g.n[a];
    }
    if (total <= (1 << 24)) break;
    hcell *= 1.25;
  }
  g.h = hcell;
  const int64_t ncell = (int64_t)g.n[0] * g.n[1] * g.n[2];
  uint32_t* cnt = (uint32_t*)alloc(actx, 4 * (ncell + 1));
  uint32_t* off = (uint32_t*)alloc(actx, 4 * (ncell + 1));
  uint32_t* cursor = (uint32_t*)alloc(actx, 4 * (ncell + 1));
  uint32_t* tiles = (uint32_t*)alloc(actx, 4 * ((ncell + 1 + 255) / 256 + 1));
  unsigned long long* total = (unsigned long long*)alloc(actx, 8);
  if (!cnt || !off || !cursor || !tiles || !total) return ODC_E_NOMEM;
  if (cudaMemsetAsync(cnt, 0, 4 * (ncell + 1), s) != cudaSuccess ||
      cudaMemsetAsync(cursor, 0, 4 * (ncell + 1), s) != cudaSuccess)
    return ODC_E_CUDA;
  k_dist_count<<<grid_for(nt, 256), 256, 0, s>>>(d_v, d_t, nt, g, cnt);
  const uint32_t* ins[1] = {cnt};
  uint32_t* outs[1] = {off};
  launch_scan_u32(ins, outs, 1, ncell + 1, tiles, total, s);
  unsigned long long h_total = 0;
  if (cudaMemcpyAsync(&h_total, total, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return ODC_E_CUDA;
  if (h_total >= 0xffffffffull) return ODC_E_NOMEM;
  int32_t* items = (int32_t*)alloc(actx, 4 * (h_total + 1));
  if (!items) return ODC_E_NOMEM;
  k_dist_fill<<<grid_for(nt, 256), 256, 0, s>>>(d_v, d_t, nt, g, off, cursor, items);
  k_dist_query<<<grid_for(nq, 128), 128, 0, s>>>(d_v, d_t, nt, g, off, items, d_q, nq, d_dist, d_tri, d_cp);
  return cudaGetLastError() == cudaSuccess ? ODC_OK : ODC_E_CUDA;
}

}  // namespace odc
