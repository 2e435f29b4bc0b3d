// odc_slabfin.cu -- kernels of the distributed slab finish.
//
// A z-slab rank owns the partitions of its cell layers and the fans of its
// edges.  Finishing the mesh (polygonize.py:199-214 unused-vertex removal,
// :253-374 repair) needs, per vertex, every triangle that references it.
// Only the partitions of a rank's top cell layer are referenced by another
// rank's triangles (the x/y edges of the next rank's first vertex layer);
// that rank sends those "seam" triangles down, and then every vertex of a
// rank has its whole fan on that rank.  The rank marks its used partitions,
// compacts them, and checks that every fan is one closed disc -- then the
// reference's repair would add nothing and the mesh is final.  Otherwise the
// host falls back to the central finish (slab.py).
#include <cuda_runtime.h>

#include "odc_kernels.h"

namespace odc {

namespace {
inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }
}  // namespace

// seam flag of triangle t: a corner in the halo (ids < n_halo)
__global__ void k_seam_flags(const int32_t* __restrict__ tris, int64_t T, int64_t n_halo,
                             uint32_t* __restrict__ flag) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  flag[t] = (tris[3 * t] < n_halo || tris[3 * t + 1] < n_halo || tris[3 * t + 2] < n_halo) ? 1u : 0u;
}
__global__ void k_seam_take(const int32_t* __restrict__ tris, int64_t T, const uint32_t* __restrict__ flag,
                            const uint32_t* __restrict__ rank, int32_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T || !flag[t]) return;
  const int64_t r = rank[t];
  out[3 * r] = tris[3 * t];
  out[3 * r + 1] = tris[3 * t + 1];
  out[3 * r + 2] = tris[3 * t + 2];
}
void launch_seam_flags(const int32_t* tris, int64_t T, int64_t n_halo, uint32_t* flag, cudaStream_t s) {
  if (T) k_seam_flags<<<grid_for(T, 256), 256, 0, s>>>(tris, T, n_halo, flag);
}
void launch_seam_take(const int32_t* tris, int64_t T, const uint32_t* flag, const uint32_t* rank, int32_t* out,
                      cudaStream_t s) {
  if (T) k_seam_take<<<grid_for(T, 256), 256, 0, s>>>(tris, T, flag, rank, out);
}

// The next rank's seam triangles in this rank's id space: its halo
// partitions are this rank's last n_halo_next owned partitions; its other
// vertices become ghost ids from `ghost` on (they only give fans their
// neighbour identities).
__global__ void k_seam_map(const int32_t* __restrict__ seam, int64_t n, int64_t n_halo_next, int64_t P, int64_t ghost,
                           int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = seam[i];
  out[i] = (int32_t)(v < n_halo_next ? P - n_halo_next + v : ghost + (v - n_halo_next));
}
void launch_seam_map(const int32_t* seam, int64_t n_tris, int64_t n_halo_next, int64_t P, int64_t ghost, int32_t* out,
                     cudaStream_t s) {
  if (n_tris) k_seam_map<<<grid_for(3 * n_tris, 256), 256, 0, s>>>(seam, 3 * n_tris, n_halo_next, P, ghost, out);
}

// owned partitions [P_halo, P) referenced by any corner: the incidence
// count of the fan pass (k_degree_range over the same triangles) is
// non-zero exactly for them.  used (u8, P_own) for odc_slab_final and its
// u32 widening (n >= P_own entries, zero past P_own) for the compaction scan.
__global__ void k_used_from_degree(const uint32_t* __restrict__ deg, int64_t P_halo, int64_t P_own, int64_t n,
                                   uint8_t* __restrict__ used, uint32_t* __restrict__ u32) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t u = i < P_own && deg[P_halo + i] > 0u ? 1u : 0u;
  if (i < P_own) used[i] = (uint8_t)u;
  u32[i] = u;
}
void launch_used_from_degree(const uint32_t* deg, int64_t P_halo, int64_t P_own, int64_t n, uint8_t* used,
                             uint32_t* u32, cudaStream_t s) {
  if (n) k_used_from_degree<<<grid_for(n, 256), 256, 0, s>>>(deg, P_halo, P_own, n, used, u32);
}

// incidence of the vertices in [lo, hi) only
__global__ void k_degree_range(const int32_t* __restrict__ tris, int64_t n, int64_t lo, int64_t hi,
                               uint32_t* __restrict__ deg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = tris[i];
  if (v >= lo && v < hi) atomicAdd(&deg[v], 1u);
}
__global__ void k_fill_range(const int32_t* __restrict__ tris, int64_t n, int64_t lo, int64_t hi,
                             const uint32_t* __restrict__ off, uint32_t* __restrict__ cursor,
                             int32_t* __restrict__ inc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = tris[i];
  if (v < lo || v >= hi) return;
  const uint32_t slot = atomicAdd(&cursor[v], 1u);
  inc[off[v] + slot] = (int32_t)(i / 3);
}
void launch_degree_range(const int32_t* tris, int64_t n_tris, int64_t lo, int64_t hi, uint32_t* deg, cudaStream_t s) {
  if (n_tris) k_degree_range<<<grid_for(3 * n_tris, 256), 256, 0, s>>>(tris, 3 * n_tris, lo, hi, deg);
}
void launch_fill_range(const int32_t* tris, int64_t n_tris, int64_t lo, int64_t hi, const uint32_t* off,
                       uint32_t* cursor, int32_t* inc, cudaStream_t s) {
  if (n_tris) k_fill_range<<<grid_for(3 * n_tris, 256), 256, 0, s>>>(tris, 3 * n_tris, lo, hi, off, cursor, inc);
}

// vertices in [lo, hi) with a fan that is not one closed disc
__global__ void k_count_nondisc(const int32_t* __restrict__ tris, const uint32_t* __restrict__ off,
                                const int32_t* __restrict__ inc, int64_t lo, int64_t hi,
                                unsigned long long* __restrict__ out) {
  const int64_t v = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned bad = 0;
  if (v < hi && off[v + 1] > off[v] && !fan_is_disc(tris, off, inc, v)) bad = 1;
  bad = __reduce_add_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(out, (unsigned long long)bad);
}
void launch_count_nondisc(const int32_t* tris, const uint32_t* off, const int32_t* inc, int64_t lo, int64_t hi,
                          unsigned long long* out, cudaStream_t s) {
  if (hi > lo) k_count_nondisc<<<grid_for(hi - lo, 256), 256, 0, s>>>(tris, off, inc, lo, hi, out);
}

// Final piece: triangles in global ids (halo partitions through the previous
// rank's ids, owned partitions compacted from part_base, fans from
// fan_base) and the compacted owned partition vertices with provenance.
__global__ void k_slab_final_tris(const int32_t* __restrict__ tris, int64_t n, int64_t P_halo, int64_t P,
                                  const int32_t* __restrict__ halo_ids, const uint32_t* __restrict__ newid,
                                  int64_t part_base, int64_t fan_base, int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = tris[i];
  int64_t g;
  if (v < P_halo) g = halo_ids[v];
  else if (v < P) g = part_base + newid[v - P_halo];
  else g = fan_base + (v - P);
  out[i] = (int32_t)g;
}
__global__ void k_slab_final_parts(int64_t P_own, const uint8_t* __restrict__ used, const uint32_t* __restrict__ newid,
                                   const double* __restrict__ verts, const int64_t* __restrict__ pcell,
                                   const int64_t* __restrict__ pidx, double* __restrict__ vout,
                                   int64_t* __restrict__ cout, int64_t* __restrict__ iout) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P_own || !used[i]) return;
  const int64_t o = newid[i];
  vout[3 * o] = verts[3 * i];
  vout[3 * o + 1] = verts[3 * i + 1];
  vout[3 * o + 2] = verts[3 * i + 2];
  cout[o] = pcell[i];
  iout[o] = pidx[i];
}
__global__ void k_slab_top_ids(int64_t P_own, int64_t n_top, const uint32_t* __restrict__ newid, int64_t part_base,
                               int32_t* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_top) return;
  out[j] = (int32_t)(part_base + newid[P_own - n_top + j]);
}
void launch_slab_final_tris(const int32_t* tris, int64_t T, int64_t P_halo, int64_t P, const int32_t* halo_ids,
                            const uint32_t* newid, int64_t part_base, int64_t fan_base, int32_t* out, cudaStream_t s) {
  if (T)
    k_slab_final_tris<<<grid_for(3 * T, 256), 256, 0, s>>>(tris, 3 * T, P_halo, P, halo_ids, newid, part_base,
                                                           fan_base, out);
}
void launch_slab_final_parts(int64_t P_own, const uint8_t* used, const uint32_t* newid, const double* verts,
                             const int64_t* pcell, const int64_t* pidx, double* vout, int64_t* cout, int64_t* iout,
                             cudaStream_t s) {
  if (P_own)
    k_slab_final_parts<<<grid_for(P_own, 256), 256, 0, s>>>(P_own, used, newid, verts, pcell, pidx, vout, cout,
                                                            iout);
}
void launch_slab_top_ids(int64_t P_own, int64_t n_top, const uint32_t* newid, int64_t part_base, int32_t* out,
                         cudaStream_t s) {
  if (n_top) k_slab_top_ids<<<grid_for(n_top, 256), 256, 0, s>>>(P_own, n_top, newid, part_base, out);
}

// Surface probe for slab balancing (analytic fields): one thread per cubic
// box of `box` vertices per side; the box is undecided when the label pass's
// interval bound (field_label_ball, the culling test of k_labels_analytic)
// cannot place the whole ball around it on one side of iso.  counts[bz] =
// undecided boxes in box layer bz -- proportional to the surface area in
// that z-range (thin walls included, which a label-flip probe misses).
__global__ void k_surface_probe(GridP g, FieldP f, int64_t box, int64_t nbx, int64_t nby, int64_t nbz,
                                unsigned long long* __restrict__ counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = nbx * nby * nbz;
  const int64_t bz = i < n ? i / (nbx * nby) : 0;
  unsigned und = 0;
  if (i < n) {
    const int64_t r = i - bz * nbx * nby, by = r / nbx, bx = r - by * nbx;
    const int64_t b[3] = {bx, by, bz};
    double pc[3], r2 = 0.0;
    for (int a = 0; a < 3; a++) {
      const double e = 0.5 * (double)box * g.h[a];  // half extent: vertices [b box, (b + 1) box]
      pc[a] = g.lo[a] + ((double)(b[a] * box) + 0.5 * (double)box) * g.h[a];
      r2 += e * e;
    }
    und = field_label_ball(f, pc, sqrt(r2) * (1.0 + 1e-12) + 1e-300) < 0 ? 1u : 0u;
  }
  // warp aggregate: a warp's boxes share a box layer except at layer ends
  const unsigned lane = threadIdx.x & 31;
  const int64_t bz0 = __shfl_sync(0xffffffffu, bz, 0);
  const bool same = __all_sync(0xffffffffu, bz == bz0 || i >= n);
  if (same) {
    const unsigned t = __reduce_add_sync(0xffffffffu, und);
    if (lane == 0 && t) atomicAdd(&counts[bz0], (unsigned long long)t);
  } else if (und) {
    atomicAdd(&counts[bz], 1ull);
  }
}
void launch_surface_probe(const GridP& g, const FieldP& f, int64_t box, unsigned long long* counts, cudaStream_t s) {
  const int64_t nbx = (g.R + box - 1) / box, nby = nbx, nbz = (g.R + box - 1) / box;
  const int64_t n = nbx * nby * nbz;
  if (n) k_surface_probe<<<grid_for(n, 256), 256, 0, s>>>(g, f, box, nbx, nby, nbz, counts);
}

}  // namespace odc
