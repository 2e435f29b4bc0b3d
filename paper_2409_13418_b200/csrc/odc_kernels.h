// odc_kernels.h -- launch wrappers for the extraction kernels (odc_kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "odc_device.cuh"
#include "odc_tables.h"

namespace odc {

struct Counts5 {  // totals of the active-set scan
  unsigned long long edges, insts, cells, faces, faces4;
};

struct DevStats {  // accumulated on the device, read back once
  unsigned long long boundary_inside;
  unsigned long long status[4];
  unsigned long long rank[4];
  unsigned long long split[4];
  unsigned long long normal_fallbacks;
  unsigned long long skipped;
  unsigned long long max_resid_bits;  // non-negative double, ordered as bits
  unsigned long long used_partitions;
  unsigned long long repair_extra;
  unsigned long long repair_overflow;
  unsigned long long faces_own, faces4_own;  // slab mode: faces with base layer owned
};

struct Stage2D {  // per-instance outputs of the 2D search
  double* pos2;      // (Q,2)
  double* pos3;      // (Q,3)
  uint8_t* status;   // (Q)
  uint8_t* mid;      // (Q)
};

struct OptP {
  int one_d, normals, split, iters_1d, s1_lin, s1_bin, s2_lin, s2_bin, continuous;
  double s1_range, s2_range, qef_trunc, fd_step;
};

// K1: labels of every grid vertex as bit-packed rows (grid.py:109-126)
void launch_labels_analytic(const GridP& g, const FieldP& f, uint32_t* L, cudaStream_t s);
void launch_pack_labels(const GridP& g, const uint8_t* bytes, uint32_t* L, cudaStream_t s);
void launch_unpack_labels(const GridP& g, const uint32_t* L, uint8_t* bytes, cudaStream_t s);
// grid positions in flat vertex order, [begin, begin+n)
void launch_grid_points(const GridP& g, int64_t begin, int64_t n, double* pts, cudaStream_t s);

// K2: crossing edges / faces / cells + ranks + compaction (grid.py:171-296)
int64_t active_tiles(const GridP& g);
int64_t occ_words(const GridP& g);  // uint2 occupancy words of the sparse records
void launch_active_bits(const GridP& g, const uint32_t* L, uint2* occ, uint32_t* tile_sums, DevStats* st,
                        cudaStream_t s);
void launch_scan_tiles(uint32_t* sums, int64_t ntiles, int nch, unsigned long long* totals, cudaStream_t s);
void launch_active_compact(const GridP& g, const uint32_t* L, RecView rec, const uint32_t* tile_sums,
                           int64_t* edge_key, int64_t* inst_key, int64_t* cell_id, int64_t* f4_key, int64_t* face_key,
                           int64_t* face_nc, cudaStream_t s);
// (pe, pq, pc) at word w (any word): slab ownership ranges
void launch_prefix_at(RecView rv, int64_t w, int64_t A, const unsigned long long* totals, unsigned long long* out,
                      cudaStream_t s);
// pbase at the window's owned cell bounds (pre[2], pre[5]) -> out[0..1] (odc_api.cu)
void launch_part_bounds(const uint32_t* pbase, int64_t C, const unsigned long long* pre, bool has_hi,
                        const unsigned long long* totals, unsigned long long* out, cudaStream_t s);

// face-centre probes for 4-crossing faces (dualize.py:59-70)
void launch_face_center_points(const GridP& g, const int64_t* f4_key, int64_t n, double* pts, cudaStream_t s);
void launch_face_center_analytic(const GridP& g, const FieldP& f, const int64_t* f4_key, int64_t n, RecView rec,
                                 cudaStream_t s);
void launch_face_center_scatter(const GridP& g, const int64_t* f4_key, const uint8_t* labels, int64_t n,
                                RecView rec, cudaStream_t s);

// K3: 1D points (search.py:71-94; pipeline.py:94-123)
void launch_search1d_analytic(const GridP& g, const FieldP& f, const OptP& o, const uint32_t* L,
                              const int64_t* edge_key, int64_t K, double* t, double* pos, int64_t* v_in,
                              cudaStream_t s);
// lock-step form for batched fields: state (lo, hi) in t/pos scratch
void launch_search1d_init(const GridP& g, const uint32_t* L, const int64_t* edge_key, int64_t K, double* lo,
                          double* hi, cudaStream_t s);
void launch_search1d_points(const GridP& g, const uint32_t* L, const int64_t* edge_key, int64_t K,
                            const double* lo, const double* hi, double* pts, cudaStream_t s);
void launch_search1d_update(int64_t K, const uint8_t* lab, double* lo, double* hi, cudaStream_t s);
void launch_search1d_finish(const GridP& g, const OptP& o, const uint32_t* L, const int64_t* edge_key, int64_t K,
                            const double* lo, const double* hi, const double* raw_in, const double* raw_out,
                            double* t, double* pos, int64_t* v_in, cudaStream_t s);

// grid positions of the inside (which=0) / outside (which=1) endpoint of each edge
void launch_edge_endpoints(const GridP& g, const uint32_t* L, const int64_t* edge_key, int64_t K, int which,
                           double* pts, cudaStream_t s);

// K5: 2D points (dualize.py:97-129 + search.py:194-322)
void launch_search2d_analytic(const GridP& g, const FieldP& f, const OptP& o, const uint32_t* L,
                              RecView rec, const int64_t* inst_key, int64_t Q, const double* pos1d,
                              Stage2D out, int64_t* inst_edges, DevStats* st, DevStatus* dst, int64_t st_lo,
                              int64_t st_hi, cudaStream_t s);
// lock-step form: 31 batches (1 midpoint + s1_lin + s1_bin + s2_lin + s2_bin)
struct Search2DState;
size_t search2d_state_bytes(int64_t Q);
void launch_search2d_lockstep_init(const GridP& g, const OptP& o, const uint32_t* L, RecView rec,
                                   const int64_t* inst_key, int64_t Q, const double* pos1d, void* state,
                                   int64_t* inst_edges, cudaStream_t s);
// step: 0 = midpoint probe, then step-1 linear/binary, then step-2; returns number of points (Q or 2Q)
int64_t launch_search2d_lockstep_points(const GridP& g, const OptP& o, const int64_t* inst_key, int64_t Q,
                                        int step, const void* state, double* pts, cudaStream_t s);
void launch_search2d_lockstep_update(const GridP& g, const OptP& o, const uint32_t* L, const int64_t* inst_key,
                                     int64_t Q, int step, const uint8_t* lab, void* state, DevStatus* dst,
                                     cudaStream_t s, int64_t q_base = 0);
void launch_search2d_lockstep_finish(const GridP& g, const OptP& o, const uint32_t* L, RecView rec,
                                     const int64_t* inst_key, int64_t Q, const double* pos1d, const void* state,
                                     Stage2D out, DevStats* st, int64_t st_lo, int64_t st_hi, cudaStream_t s);
// fused: fold the labels of ``step`` in and write the points of step + 1; returns their count
// step's labels in, the query points of step + 1 out.  With map != nullptr
// (only when step + 1 is a linear scan step) the points are compacted to the
// instances/rays still scanning: count in cnt2[(step + 1) & 1] (cnt2 is two
// int64, zero before the first step), label slot of point i in map[i]; the
// kernel also resets cnt2[step & 1] and the evaluator's pair counter sched.
bool search2d_step_is_linear(const OptP& o, int step);
int64_t launch_search2d_lockstep_step(const GridP& g, const OptP& o, const uint32_t* L, const int64_t* inst_key,
                                      int64_t Q, int step, const uint8_t* lab, void* state, DevStatus* dst,
                                      double* pts, cudaStream_t s, int32_t* map = nullptr, int64_t* cnt2 = nullptr,
                                      unsigned long long* sched = nullptr, int64_t q_base = 0);
// (q_base: index of the first instance of this batch, for error reports)
int search2d_num_steps(const OptP& o);

// fd-gradient normals (pipeline.py:126-151): 6K raw samples
void launch_fd_points(const GridP& g, const OptP& o, const double* pos1d, int64_t K, double* pts, cudaStream_t s);
void launch_fd_raw_analytic(const FieldP& f, const double* pts, int64_t n, double* raw, cudaStream_t s);
void launch_fd_normals(const GridP& g, const OptP& o, const uint32_t* L, const int64_t* edge_key, int64_t K,
                       const double* raw, double* edge_normals, DevStats* st, int64_t st_lo, int64_t st_hi,
                       cudaStream_t s);

// K6: per-cell partitions, plane samples, QEF (dualize.py:194-444)
void launch_cell_config(const GridP& g, const uint32_t* L, RecView rec, const int64_t* cell_id, int64_t C,
                        const CellTabEntry* table, uint16_t* cfg, uint32_t* ncyc, uint32_t* nsamp, cudaStream_t s);
// single-pass (decoupled look-back) form: status holds 2 * scan_lookback_tiles(n)
// words that are never cleared (epoch: a per-context counter, new per scan, >= 1)
int launch_scan_lookback(const uint32_t* const* in, uint32_t* const* out, int nch, int64_t n,
                         unsigned long long* status, uint32_t epoch, unsigned long long* totals, cudaStream_t s);
int64_t scan_lookback_tiles(int64_t n);
// returns the number of kernels launched
int launch_scan_u32(const uint32_t* const* in, uint32_t* const* out, int nch, int64_t n, uint32_t* tile_buf,
                    unsigned long long* totals, cudaStream_t s);
struct CellOut {
  double* verts;       // (P,3) partition vertices (the first P rows of the mesh)
  int64_t* part_cell;  // (P)
  int64_t* part_index; // (P)
  int64_t* rank;       // (P) (keep only; may be null)
  double* resid;       // (P) (keep only)
  uint64_t* pinfo;     // (C) part_base << 24 | cyc_of_edge
  int64_t* cyc_edges;  // (Ns) keep only
  int64_t* cyc_insts;  // (Ns) keep only
  double* normals;     // (Ns,3) keep only
  int64_t* cyc_len;    // (P) keep only
};
// numpy.linalg.eigh for a batch of symmetric 3x3 matrices (odc_eigh3.cu)
void launch_eigh3_batch(const double* A, int64_t n, double* w, double* V, int32_t* info, cudaStream_t s);
void eigh3_host_batch(const double* A, int64_t n, double* w, double* V, int32_t* info);
// K6 (two kernels, see odc_kernels.cu): snorm (Ns,3) / srow (Ns) sample
// scratch, psoff (P + 1) first sample of every partition (psoff[P] = Ns is
// set by the caller); statistics of cells [st_lo, st_hi) / partitions
// [own_lo, own_hi)
void launch_cell_solve(const GridP& g, const OptP& o, const uint32_t* L, RecView rec, const int64_t* cell_id,
                       int64_t C, const CellTabEntry* table, const uint16_t* cfg, const uint32_t* part_base,
                       const uint32_t* samp_base, const double* pos1d, const double* pos3, const double* edge_normals,
                       CellOut out, double* snorm, int32_t* srow, uint32_t* psoff, int64_t P, DevStats* st,
                       int64_t st_lo, int64_t st_hi, int64_t own_lo, int64_t own_hi, cudaStream_t s);

// K7: polygonization (polygonize.py:110-217)
void launch_poly_classify(const GridP& g, const OptP& o, const uint32_t* L, RecView rec,
                          const int64_t* edge_key, int64_t K, const uint64_t* pinfo, const double* verts,
                          int4* pid4, uint8_t* kase, uint32_t* ntri, uint32_t* nfan, DevStats* st, cudaStream_t s);
void launch_poly_emit(int64_t K, int64_t P, const int64_t* edge_key, const int4* pid4, const uint8_t* kase,
                      const uint32_t* tri_off, const uint32_t* fan_rank, const double* pos1d, double* verts,
                      int32_t* tris, int64_t* fan_edge, uint8_t* used, cudaStream_t s);
void launch_count_used(const uint8_t* used, int64_t P, DevStats* st, cudaStream_t s);
void launch_remap_vertices(int64_t V, int64_t T, const uint8_t* used, const uint32_t* new_id, const double* v_in,
                           double* v_out, int32_t* tris, int64_t* src_of, cudaStream_t s);
void launch_split_cases(int64_t K, const uint8_t* kase, int64_t* out, uint32_t* rank, cudaStream_t s);
void launch_interior_flags(int64_t K, const uint8_t* kase, uint32_t* flag, cudaStream_t s);

// K8: non-manifold repair (polygonize.py:220-374)
// T_dev (optional): the count on the device, T then only bounds the launch
void launch_vertex_degree(const int32_t* tris, int64_t T, uint32_t* deg, cudaStream_t s,
                          const uint8_t* dirty = nullptr, const unsigned long long* T_dev = nullptr);
void launch_vertex_fill(const int32_t* tris, int64_t T, const uint32_t* off, uint32_t* cursor, int32_t* inc,
                        cudaStream_t s, const uint8_t* dirty = nullptr, const unsigned long long* T_dev = nullptr);
// big: per-incidence scratch for fans of more than 64 triangles (nullptr: such
// vertices are counted in DevStats::repair_overflow and skipped; the host
// then re-runs with repair_scratch_bytes(T) of scratch)
void launch_repair_count(const double* verts, const int32_t* tris, int64_t V, const uint32_t* off,
                         const int32_t* inc, uint32_t* extra, char* big, DevStats* st, cudaStream_t s,
                         const uint8_t* dirty = nullptr);
// after a repair pass: flag every corner of the triangles it renamed
void launch_mark_dirty(const int32_t* cur, const int32_t* next, int64_t T, uint8_t* dirty, cudaStream_t s);
size_t repair_scratch_bytes(int64_t T);
void launch_repair_apply(const double* verts, const int32_t* tris, int64_t V, const uint32_t* off,
                         const int32_t* inc, const uint32_t* extra_off, char* big, int32_t* tris_next,
                         int64_t* src_of_new, cudaStream_t s);
void launch_copy_vertices(const double* src, const int64_t* src_of, int64_t base, int64_t n, double* dst,
                          cudaStream_t s);

// slab mode
void launch_count_owned_faces(const GridP& g, RecView rec, DevStats* st, cudaStream_t s);
void launch_globalize_tris(const int32_t* tris, int64_t T, int64_t P_halo, int64_t P_window, int64_t part_base,
                           int64_t P_total, int64_t fan_base, int32_t* out, cudaStream_t s);
void launch_mark_used(const int32_t* tris, int64_t T, uint8_t* used, cudaStream_t s);
void launch_widen_flags(const uint8_t* f, int64_t n, uint32_t* out, cudaStream_t s);
void launch_gather_provenance(int64_t V, const int64_t* src_of, const int64_t* kind_in, const int64_t* ref_in,
                              int64_t* kind, int64_t* ref, cudaStream_t s);

// mesh copy-back: int32 triangles widened to the reference's int64 (mesh.py:28)
void launch_widen_i32(const int32_t* src, int64_t* dst, int64_t n, cudaStream_t s);
// provenance of repair duplicates [V0, V): kind 2, ref (-1, -1) (polygonize.py:348-373)
void launch_dup_provenance(int64_t V0, int64_t V, int64_t* kind, int64_t* ref, cudaStream_t s);

// MeshWindingField (odc_winding.cu; fields.py:281-386): per-triangle terms
struct WindDev {
  double *ta, *tb, *tc, *nhat, *eab, *eac;  // (T,3)
  double *d00, *d01, *d11, *denb;           // (T)
  uint8_t* ok;                              // (T) non-degenerate normal
  int64_t nt;
  double nudge;  // 1e-9 * scale / sqrt(3)
};
void launch_winding_prep(const double* v, const int64_t* t, int64_t nt, const WindDev& w, cudaStream_t s);
struct PointSrc;
// labels (raw > 0.5) and/or raw winding numbers of n query points; sets
// *failed when a query could not be moved off the surface in 8 attempts
void winding_eval(const WindDev& w, const PointSrc& src, int64_t n, uint8_t* labels, double* raw,
                  unsigned int* failed, cudaStream_t s);

// VoxelField (odc_voxel.cu; fields.py:245-278): dense (nx, ny, nz) f64 values
struct VoxDev {
  const double* values;
  int64_t nx, ny, nz;
  double origin[3], spacing[3];
};
void voxel_eval(const VoxDev& w, const PointSrc& src, int64_t n, uint8_t* labels, double* raw, cudaStream_t s);

void launch_instance_edges(const GridP& g, const uint32_t* L, RecView rec, const int64_t* inst_key, int64_t Q,
                           const double* pos1d, int64_t* inst_edges, cudaStream_t s);

// marching-cubes baseline (baseline.py:48-127)
void launch_mc_points(const GridP& g, const uint32_t* L, const int64_t* edge_key, int64_t K, const double* raw_in,
                      const double* raw_out, double iso, double* pos, cudaStream_t s);
void launch_mc_count(int64_t C, const uint32_t* ncyc, const uint32_t* nedge, uint32_t* ntri, cudaStream_t s);
void launch_mc_fans(const GridP& g, const uint32_t* L, RecView rec, const int64_t* cell_id, int64_t C,
                    const CellTabEntry* table, const uint16_t* cfg, const uint32_t* tri_off, const double* pos,
                    int32_t* tris, uint8_t* used, cudaStream_t s);

// mesh validation (odc_validate.cu; mesh.py:91-150)
void launch_manifold_vertex(int64_t V, const int32_t* tris, const uint32_t* off, const int32_t* inc, int32_t* nbv,
                            uint32_t* nbc, uint32_t* nbt, uint32_t* uf, uint32_t* n_nb, uint32_t* n_nm,
                            uint32_t* n_bd, uint32_t* pinched, uint32_t* isolated, cudaStream_t s);
void launch_manifold_emit(int64_t V, const uint32_t* off, const int32_t* nbv, const uint32_t* nbc,
                          const uint32_t* n_nb, const uint32_t* n_nm, const uint32_t* nm_off, int64_t* edges,
                          cudaStream_t s);
void launch_emit_flagged(int64_t V, const uint32_t* flag, const uint32_t* pos, int64_t* out, cudaStream_t s);
void launch_narrow_tris(const int64_t* in, int64_t n, int32_t* out, int64_t V, uint32_t* bad, cudaStream_t s);
// exact point-to-mesh distance (odc_distance.cu; mesh.py:153-270)
int mesh_distance(const double* d_v, const int32_t* d_t, int64_t nt, const double* d_q, int64_t nq,
                  void* (*alloc)(void*, size_t), void* actx, cudaStream_t s, double* d_dist, int64_t* d_tri,
                  double* d_cp);
void launch_tri_areas(const double* v, const int32_t* t, int64_t nt, double* area, cudaStream_t s);
// count_self_intersections (odc_selfx.cu; mesh.py:395-487): hit keys a*nt+b
// sorted into d_out_hits when their number fits cap; *n_hits always set
int self_intersections(const double* d_v, int64_t nv, const int32_t* d_t, int64_t nt, double tol,
                       void* (*alloc)(void*, size_t), void* actx, cudaStream_t s, int64_t* d_out_hits,
                       int64_t cap, int64_t* n_hits);

// provenance (mesh.py:11-20)
void launch_provenance(int64_t V, int64_t P, const int64_t* src_of, const int64_t* part_cell,
                       const int64_t* part_index, const int64_t* fan_edge, int64_t* kind, int64_t* ref,
                       cudaStream_t s);

// shared-field hook
void launch_eval_raw_analytic(const FieldP& f, const double* pts, int64_t n, double* raw, uint8_t* lab,
                              cudaStream_t s);

// ---- batch split (odc_batch.cu): per-shape ranges of a stacked-z batch
constexpr int kBatchCols = 7;  // edges, instances, cells, 4-faces, partitions, triangles, fans
void launch_batch_bounds(const GridP& g, RecView rec, int64_t A, int64_t K, int64_t Q, int64_t C,
                         const int64_t* f4_key, int64_t F4, const uint32_t* pbase, int64_t P, const uint32_t* toff,
                         const uint32_t* frank, int64_t T, int64_t NF, int64_t* out, cudaStream_t s);
// vshape + stable sort by shape (tmp == nullptr: size query into
// *tmp_bytes); vcounts (2 nb + 1): vertex starts per shape (nb + 1), then
// each shape's raw-vertex count
void batch_sort_vertices(const int32_t* tris, int64_t T, int64_t V, int64_t V0, const int64_t* t_start, int nb,
                         uint32_t* vshape, uint32_t* skeys, int32_t* iota, int32_t* perm, void* tmp, size_t* tmp_bytes,
                         int64_t* vcounts, cudaStream_t s);
void launch_iota_i32(int32_t* a, int64_t n, cudaStream_t s);
void launch_local_ids(const uint32_t* skeys, const int32_t* perm, int64_t V, const int64_t* v_start, int32_t* local,
                      cudaStream_t s);
void launch_batch_gather(const double* verts, const int32_t* perm, const uint32_t* skeys, int64_t V,
                         const int64_t* kind_in, const int64_t* ref_in, int64_t cell_per_shape,
                         int64_t key_per_shape, double* vout, int64_t* kout, int64_t* rout, cudaStream_t s);
void launch_batch_tris(const int32_t* tris, int64_t T, const int32_t* local, int32_t* out, cudaStream_t s);

// ---- distributed slab finish (odc_slabfin.cu)
void launch_seam_flags(const int32_t* tris, int64_t T, int64_t n_halo, uint32_t* flag, cudaStream_t s);
void launch_seam_take(const int32_t* tris, int64_t T, const uint32_t* flag, const uint32_t* rank, int32_t* out,
                      cudaStream_t s);
void launch_seam_map(const int32_t* seam, int64_t n_tris, int64_t n_halo_next, int64_t P, int64_t ghost, int32_t* out,
                     cudaStream_t s);
void launch_used_from_degree(const uint32_t* deg, int64_t P_halo, int64_t P_own, int64_t n, uint8_t* used,
                             uint32_t* u32, cudaStream_t s);
void launch_degree_range(const int32_t* tris, int64_t n_tris, int64_t lo, int64_t hi, uint32_t* deg, cudaStream_t s);
void launch_fill_range(const int32_t* tris, int64_t n_tris, int64_t lo, int64_t hi, const uint32_t* off,
                       uint32_t* cursor, int32_t* inc, cudaStream_t s);
void launch_count_nondisc(const int32_t* tris, const uint32_t* off, const int32_t* inc, int64_t lo, int64_t hi,
                          unsigned long long* out, cudaStream_t s);
void launch_slab_final_tris(const int32_t* tris, int64_t T, int64_t P_halo, int64_t P, const int32_t* halo_ids,
                            const uint32_t* newid, int64_t part_base, int64_t fan_base, int32_t* out, cudaStream_t s);
void launch_slab_final_parts(int64_t P_own, const uint8_t* used, const uint32_t* newid, const double* verts,
                             const int64_t* pcell, const int64_t* pidx, double* vout, int64_t* cout, int64_t* iout,
                             cudaStream_t s);
void launch_slab_top_ids(int64_t P_own, int64_t n_top, const uint32_t* newid, int64_t part_base, int32_t* out,
                         cudaStream_t s);
// slab balancing: undecided boxes (of `box` vertices per side) per box layer along z
void launch_surface_probe(const GridP& g, const FieldP& f, int64_t box, unsigned long long* counts, cudaStream_t s);

}  // namespace odc
