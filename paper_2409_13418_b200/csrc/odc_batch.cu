// odc_batch.cu -- the per-shape split of a batched extraction (BASELINE
// config 5, odc_extract_batch).
//
// A batch stacks nb grids of the same resolution along z (GridP::nb): every
// stage runs once over all shapes, and because keys are ordered shape by
// shape (the shape is the high part of the flat index), each shape's crossing
// edges, instances, cells, partitions, fans and triangles are contiguous
// ranges of the stage arrays.  The union mesh is finished (unused-vertex
// removal + repair, polygonize.py:199-214, :253-374) as one mesh: shapes
// share no vertex, so that equals finishing each shape on its own.  Its
// vertex order interleaves the shapes (all partitions, then all fans, then
// each repair pass's duplicates); a stable sort by shape gives every shape
// the reference's own order (partitions, fans, pass 1, pass 2, ... each
// ascending), which is all the split needs.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "odc_kernels.h"

namespace odc {

namespace {
inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* a, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// shape of row r given ascending starts (nb + 1 entries, starts[nb] = total)
__device__ __forceinline__ int shape_of_row(const int64_t* starts, int nb, int64_t r) {
  int lo = 0, hi = nb;  // the last b with starts[b] <= r
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (starts[mid] <= r) lo = mid;
    else hi = mid;
  }
  return lo;
}
}  // namespace

// Per-shape starts (b = 0..nb) of the stage arrays:
//   out[b * kBatchCols + ...] = edges, instances, cells, 4-crossing faces,
//   partitions, triangles, fans
__global__ void k_batch_bounds(GridP g, RecView rec, int64_t A, int64_t K, int64_t Q, int64_t C,
                               const int64_t* __restrict__ f4_key, int64_t F4, const uint32_t* __restrict__ pbase,
                               int64_t P, const uint32_t* __restrict__ toff, const uint32_t* __restrict__ frank,
                               int64_t T, int64_t NF, int64_t* __restrict__ out) {
  const int b = (int)(blockIdx.x * blockDim.x + threadIdx.x);
  if (b > g.nb) return;
  int64_t* o = out + (int64_t)b * kBatchCols;
  int64_t e, q, c;
  if (b == g.nb) {
    e = K;
    q = Q;
    c = C;
  } else {
    const int64_t w = (int64_t)b * g.S * g.S * g.W;  // first word of shape b
    const uint2 oc = rec.occ[w >> 5];
    const int64_t a = (int64_t)oc.y + __popc(oc.x & lowmask((int)(w & 31)));
    if (a < A) {
      e = rec.rec[a].pe;
      q = rec.rec[a].pq;
      c = rec.rec[a].pc;
    } else {
      e = K;
      q = Q;
      c = C;
    }
  }
  o[0] = e;
  o[1] = q;
  o[2] = c;
  o[3] = b == g.nb ? F4 : lower_bound_i64(f4_key, F4, (int64_t)b * g.S3 * 3);
  o[4] = c < C ? (int64_t)pbase[c] : P;
  o[5] = e < K ? (int64_t)toff[e] : T;
  o[6] = e < K ? (int64_t)frank[e] : NF;
}

void launch_batch_bounds(const GridP& g, RecView rec, int64_t A, int64_t K, int64_t Q, int64_t C,
                         const int64_t* f4_key, int64_t F4, const uint32_t* pbase, int64_t P, const uint32_t* toff,
                         const uint32_t* frank, int64_t T, int64_t NF, int64_t* out, cudaStream_t s) {
  k_batch_bounds<<<grid_for(g.nb + 1, 128), 128, 0, s>>>(g, rec, A, K, Q, C, f4_key, F4, pbase, P, toff, frank, T, NF,
                                                         out);
}

// shape of every vertex of the finished union mesh: the shape of a triangle
// holding it (every vertex is referenced after unused-vertex removal)
__global__ void k_vertex_shape(const int32_t* __restrict__ tris, int64_t T, const int64_t* __restrict__ t_start,
                               int nb, uint32_t* __restrict__ vshape) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint32_t b = (uint32_t)shape_of_row(t_start, nb, t);
  vshape[tris[3 * t]] = b;
  vshape[tris[3 * t + 1]] = b;
  vshape[tris[3 * t + 2]] = b;
}

// Per-shape vertex starts in the by-shape order (out[0..nb]) and raw-vertex
// counts (out[nb+1+b]): within a shape's segment the global ids ascend and
// the raw (pre-repair) vertices are the ids below V0, so both are binary
// searches (no same-address atomics over millions of vertices).
__global__ void k_batch_vcounts(const uint32_t* __restrict__ skeys, const int32_t* __restrict__ perm, int64_t V,
                                int64_t V0, int nb, int64_t* __restrict__ out) {
  const int b = (int)(blockIdx.x * blockDim.x + threadIdx.x);
  if (b > nb) return;
  auto first_key = [&](uint32_t key) {  // first i with skeys[i] >= key
    int64_t lo = 0, hi = V;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (skeys[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  const int64_t s0 = first_key((uint32_t)b);
  out[b] = s0;
  if (b == nb) return;
  const int64_t s1 = first_key((uint32_t)b + 1);
  int64_t lo = s0, hi = s1;  // first i in [s0, s1) with perm[i] >= V0
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (perm[mid] < V0) lo = mid + 1;
    else hi = mid;
  }
  out[nb + 1 + b] = lo - s0;
}

// local id of vertex perm[i] = its rank among its shape's vertices
__global__ void k_local_ids(const uint32_t* __restrict__ skeys, const int32_t* __restrict__ perm, int64_t V,
                            const int64_t* __restrict__ v_start, int32_t* __restrict__ local) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  local[perm[i]] = (int32_t)(i - v_start[skeys[i]]);
}

void batch_sort_vertices(const int32_t* tris, int64_t T, int64_t V, int64_t V0, const int64_t* t_start, int nb,
                         uint32_t* vshape, uint32_t* skeys, int32_t* iota, int32_t* perm, void* tmp, size_t* tmp_bytes,
                         int64_t* vcounts, cudaStream_t s) {
  if (!tmp) {  // size query
    cub::DeviceRadixSort::SortPairs(nullptr, *tmp_bytes, vshape, skeys, iota, perm, (int)V, 0, 16, s);
    return;
  }
  if (T) k_vertex_shape<<<grid_for(T, 256), 256, 0, s>>>(tris, T, t_start, nb, vshape);
  int bits = 1;
  while ((1 << bits) < nb && bits < 16) bits++;
  cub::DeviceRadixSort::SortPairs(tmp, *tmp_bytes, vshape, skeys, iota, perm, (int)V, 0, bits, s);
  k_batch_vcounts<<<grid_for(nb + 1, 128), 128, 0, s>>>(skeys, perm, V, V0, nb, vcounts);
}

void launch_local_ids(const uint32_t* skeys, const int32_t* perm, int64_t V, const int64_t* v_start, int32_t* local,
                      cudaStream_t s) {
  if (V) k_local_ids<<<grid_for(V, 256), 256, 0, s>>>(skeys, perm, V, v_start, local);
}

__global__ void k_iota_i32(int32_t* __restrict__ a, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int32_t)i;
}
void launch_iota_i32(int32_t* a, int64_t n, cudaStream_t s) {
  if (n) k_iota_i32<<<grid_for(n, 256), 256, 0, s>>>(a, n);
}

// Per-shape copy-out (shapes concatenated in order): vertices and their
// provenance gathered through perm, refs made shape-local (cell id and edge
// key minus the shape's offset in the stacked grid), triangles renamed to
// local ids.  kind/ref in: provenance of the union mesh's vertices.
__global__ void k_batch_gather(const double* __restrict__ verts, const int32_t* __restrict__ perm,
                               const uint32_t* __restrict__ skeys, int64_t V, const int64_t* __restrict__ kind_in,
                               const int64_t* __restrict__ ref_in, int64_t cell_per_shape, int64_t key_per_shape,
                               double* __restrict__ vout, int64_t* __restrict__ kout, int64_t* __restrict__ rout) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int64_t v = perm[i];
  vout[3 * i] = verts[3 * v];
  vout[3 * i + 1] = verts[3 * v + 1];
  vout[3 * i + 2] = verts[3 * v + 2];
  if (kout) {
    const int64_t k = kind_in[v], b = skeys[i];
    kout[i] = k;
    int64_t r0 = ref_in[2 * v];
    if (k == 0) r0 -= b * cell_per_shape;
    else if (k == 1) r0 -= b * key_per_shape;
    rout[2 * i] = r0;
    rout[2 * i + 1] = ref_in[2 * v + 1];
  }
}
void launch_batch_gather(const double* verts, const int32_t* perm, const uint32_t* skeys, int64_t V,
                         const int64_t* kind_in, const int64_t* ref_in, int64_t cell_per_shape,
                         int64_t key_per_shape, double* vout, int64_t* kout, int64_t* rout, cudaStream_t s) {
  if (V)
    k_batch_gather<<<grid_for(V, 256), 256, 0, s>>>(verts, perm, skeys, V, kind_in, ref_in, cell_per_shape,
                                                    key_per_shape, vout, kout, rout);
}

__global__ void k_batch_tris(const int32_t* __restrict__ tris, int64_t n, const int32_t* __restrict__ local,
                             int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = local[tris[i]];
}
void launch_batch_tris(const int32_t* tris, int64_t T, const int32_t* local, int32_t* out, cudaStream_t s) {
  if (T) k_batch_tris<<<grid_for(3 * T, 256), 256, 0, s>>>(tris, 3 * T, local, out);
}

}  // namespace odc
