// odc_validate.cu -- mesh validation on the device.
//
// validate_manifold (/root/reference/pkg/src/occmesh/mesh.py:91-150):
//   * an undirected edge is non-manifold when more than two triangles use it,
//     a boundary edge when exactly one does;
//   * a vertex is pinched when its incident triangles do not form one
//     component under "share a neighbour vertex" (mesh.py:117-141);
//   * a vertex no triangle uses is isolated.
// Everything is per vertex over its fan (CSR of incident triangles): the
// multiplicity of edge (a, b) is the number of a's fan triangles that
// contain b, so no global edge sort is needed.  Each vertex owns a scratch
// segment proportional to its degree, so fans of any size work.  Outputs are
// compacted in vertex order (and by b within a vertex), which is the
// reference's order: edge keys a*(V+1)+b ascending, vertex ids ascending.
#include <cuda_runtime.h>

#include <cstdint>

#include "odc_kernels.h"

namespace odc {

namespace {
inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t x) {
  while (parent[x] != x) {
    parent[x] = parent[parent[x]];
    x = parent[x];
  }
  return x;
}
}  // namespace

// Per vertex a: neighbour list (vertex, count) in nbv/nbc[2*off[a] ..),
// union-find parents over its fan slots in uf[off[a] ..).
__global__ void k_manifold_vertex(int64_t V, const int32_t* __restrict__ tris, const uint32_t* __restrict__ off,
                                  const int32_t* __restrict__ inc, int32_t* __restrict__ nbv,
                                  uint32_t* __restrict__ nbc, uint32_t* __restrict__ nbt, uint32_t* __restrict__ uf,
                                  uint32_t* __restrict__ n_nb, uint32_t* __restrict__ n_nm,
                                  uint32_t* __restrict__ n_bd, uint32_t* __restrict__ pinched,
                                  uint32_t* __restrict__ isolated) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= V) return;
  const uint32_t o0 = off[a], deg = off[a + 1] - o0;
  int32_t* v = nbv + 2 * (size_t)o0;
  uint32_t* cnt = nbc + 2 * (size_t)o0;
  uint32_t* first = nbt + 2 * (size_t)o0;
  uint32_t* parent = uf + o0;
  uint32_t nn = 0;
  for (uint32_t i = 0; i < deg; i++) {
    parent[i] = i;
    const int32_t t = inc[o0 + i];
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const int32_t b = tris[3 * (size_t)t + k];
      if (b == (int32_t)a) continue;
      uint32_t j = 0;
      while (j < nn && v[j] != b) j++;
      if (j < nn) {  // triangle i shares neighbour b with an earlier fan triangle
        cnt[j]++;
        const uint32_t ra = uf_find(parent, first[j]), rb = uf_find(parent, i);
        if (ra != rb) parent[ra] = rb;
      } else {
        v[nn] = b;
        cnt[nn] = 1;
        first[nn] = i;
        nn++;
      }
    }
  }
  uint32_t nm = 0, bd = 0, roots = 0;
  for (uint32_t j = 0; j < nn; j++)
    if (v[j] > (int32_t)a) {  // each undirected edge counted at its lower end
      nm += cnt[j] > 2;
      bd += cnt[j] == 1;
    }
  for (uint32_t i = 0; i < deg; i++) roots += uf_find(parent, i) == i;
  n_nb[a] = nn;
  n_nm[a] = nm;
  n_bd[a] = bd;
  pinched[a] = roots > 1;
  isolated[a] = deg == 0;
}

// non-manifold edges (a, b), b ascending within a, at nm_off[a]
__global__ void k_manifold_emit(int64_t V, const uint32_t* __restrict__ off, const int32_t* __restrict__ nbv,
                                const uint32_t* __restrict__ nbc, const uint32_t* __restrict__ n_nb,
                                const uint32_t* __restrict__ n_nm, const uint32_t* __restrict__ nm_off,
                                int64_t* __restrict__ edges) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= V || n_nm[a] == 0) return;
  const int32_t* v = nbv + 2 * (size_t)off[a];
  const uint32_t* cnt = nbc + 2 * (size_t)off[a];
  const uint32_t nn = n_nb[a];
  int64_t* out = edges + 2 * (size_t)nm_off[a];
  int32_t last = (int32_t)a;
  for (uint32_t k = 0; k < n_nm[a]; k++) {  // selection in ascending b
    int32_t best = INT32_MAX;
    for (uint32_t j = 0; j < nn; j++)
      if (cnt[j] > 2 && v[j] > last && v[j] < best) best = v[j];
    out[2 * k] = a;
    out[2 * k + 1] = best;
    last = best;
  }
}

// vertex ids whose flag is set, at their exclusive-scan slots
__global__ void k_emit_flagged(int64_t V, const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                               int64_t* __restrict__ out) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a < V && flag[a]) out[pos[a]] = a;
}

__global__ void k_narrow_tris(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out,
                              int64_t V, uint32_t* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t x = in[i];
  if (x < 0 || x >= V) atomicOr(bad, 1u);
  out[i] = (int32_t)x;
}

void launch_manifold_vertex(int64_t V, const int32_t* tris, const uint32_t* off, const int32_t* inc, int32_t* nbv,
                            uint32_t* nbc, uint32_t* nbt, uint32_t* uf, uint32_t* n_nb, uint32_t* n_nm,
                            uint32_t* n_bd, uint32_t* pinched, uint32_t* isolated, cudaStream_t s) {
  if (V)
    k_manifold_vertex<<<grid_for(V, 128), 128, 0, s>>>(V, tris, off, inc, nbv, nbc, nbt, uf, n_nb, n_nm, n_bd,
                                                      pinched, isolated);
}
void launch_manifold_emit(int64_t V, const uint32_t* off, const int32_t* nbv, const uint32_t* nbc,
                          const uint32_t* n_nb, const uint32_t* n_nm, const uint32_t* nm_off, int64_t* edges,
                          cudaStream_t s) {
  if (V) k_manifold_emit<<<grid_for(V, 128), 128, 0, s>>>(V, off, nbv, nbc, n_nb, n_nm, nm_off, edges);
}
void launch_emit_flagged(int64_t V, const uint32_t* flag, const uint32_t* pos, int64_t* out, cudaStream_t s) {
  if (V) k_emit_flagged<<<grid_for(V, 256), 256, 0, s>>>(V, flag, pos, out);
}
void launch_narrow_tris(const int64_t* in, int64_t n, int32_t* out, int64_t V, uint32_t* bad, cudaStream_t s) {
  if (n) k_narrow_tris<<<grid_for(n, 256), 256, 0, s>>>(in, n, out, V, bad);
}

}  // namespace odc
