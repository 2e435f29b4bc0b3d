/*
 * odc.h -- C-ABI of libodc, the B200-native Occupancy-Based Dual Contouring
 * extraction path.  Plain pointers and sizes only; no torch or CUDA types.
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/pkg/src/occmesh/):
 *
 *   odc_extract        pipeline.contour(field, grid, options, counter)
 *                      pipeline.py:154-240 -- the whole extraction path:
 *                      sample_labels (grid.py:109-126), extract_active
 *                      (grid.py:171-296), find_1d_points (search.py:71-94),
 *                      face_pairings (dualize.py:51-94), partition_cells
 *                      (dualize.py:194-238), find_2d_points (search.py:194-322),
 *                      build_plane_samples/estimate_normals (dualize.py:299-317,
 *                      :402-429), place_3d_points/solve_qef_batch
 *                      (dualize.py:332-372, :432-444), build_mesh
 *                      (polygonize.py:110-217), repair_nonmanifold
 *                      (polygonize.py:253-374).
 *   odc_options        pipeline.ContourOptions + search.SearchBudget/LineBudget
 *                      (pipeline.py:60-78, search.py:29-58).
 *   odc_stats          ContourResult.stats + EvalCounter.snapshot()
 *                      (pipeline.py:30-57, :160-239).
 *   odc_field_*        the field argument: OccupancyField.eval_raw + iso_level +
 *                      continuous (fields.py:51-61), lowered to a device program
 *                      (analytic/CSG/smoothed, fields.py:64-242) or to MLP weights.
 *   odc_eval_raw       EvalCounter.raw / eval_labels on the device (fields.py:35-48);
 *                      also the shared-field hook for the parity oracle.
 *   odc_copy_mesh      ContourResult.mesh / raw_mesh (TriangleMesh, mesh.py:11-76).
 *   odc_copy_array     intermediate stage outputs (LabelVolume.labels, ActiveSets,
 *                      Point1DBatch, Point2DBatch, CellPartitions, ...), for parity.
 *
 * Error codes map onto the reference's exception types (see ODC_E_*).
 * Thread-safety: one odc_ctx per host thread; a context owns its device
 * workspace and its last extraction's outputs.
 */
#ifndef ODC_H
#define ODC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define ODC_OK 0
#define ODC_E_ASSERT 1   /* AssertionError  (grid.py:252-253, search.py:234-238)   */
#define ODC_E_CONTRACT 2 /* InternalContractError (dualize.py:23-24)               */
#define ODC_E_CONFIG 3   /* ConfigurationError (pipeline.py:26-27, :72-78, :128)   */
#define ODC_E_VALUE 4    /* ValueError (grid.py:28-31, fields.py:42-45)           */
#define ODC_E_CUDA 5     /* CUDA runtime failure                                   */
#define ODC_E_NOMEM 6    /* device allocation failure                              */
#define ODC_E_ARG 7      /* bad argument to the C-ABI                              */
#define ODC_E_CALLBACK 8 /* a callback field's function failed (its own exception)  */

/* field program opcodes (postfix; lowering in paper_2409_13418_b200/fields.py) */
#define ODC_OP_END 0
#define ODC_OP_SPHERE_SD 1
#define ODC_OP_BOX_SD 2
#define ODC_OP_TORUS_SD 3
#define ODC_OP_PLANE_SD 4
#define ODC_OP_SD2RAW 5
#define ODC_OP_RAW_MAX 6
#define ODC_OP_RAW_MIN 7
#define ODC_OP_RAW_DIFF 8
#define ODC_OP_RAW_COMPL 9
#define ODC_OP_SD_MIN 10
#define ODC_OP_SD_MAX 11
#define ODC_OP_SD_DIFF 12
#define ODC_OP_SD_NEG 13
#define ODC_OP_XFORM_BEGIN 14
#define ODC_OP_XFORM_END 15
#define ODC_OP_SMOOTH 16
#define ODC_MAX_NODES 256

typedef struct {
  int32_t op;
  int32_t pad;
  double p[16];
} odc_node;

/* MlpField (paper_2409_13418_b200/fields.py): weights as float32 host arrays,
 * already bf16-representable. w0: (d_in, 256) row-major, w1..w7: (256, 256),
 * w_head: (256). */
typedef struct {
  int32_t d_in, width, depth, n_freq;
  const float* w0;
  const float* w_hidden; /* (depth-1, 256, 256) */
  const float* biases;   /* (depth, 256) */
  const float* w_head;   /* (256) */
  double b_head, amplitude, prior_scale, prior_radius;
  double prior_center[3];
} odc_mlp_desc;

typedef struct odc_ctx odc_ctx;
typedef struct odc_field odc_field;

/* ContourOptions (pipeline.py:60-78); enums follow ONE_D_MODES etc. */
#define ODC_ONE_D_MIDPOINT 0
#define ODC_ONE_D_LINEAR 1
#define ODC_ONE_D_BINARY 2
#define ODC_NORMALS_FD 0
#define ODC_NORMALS_2D 1
#define ODC_SPLIT_MDC 0
#define ODC_SPLIT_IC 1
typedef struct {
  int32_t one_d, normals, split, repair;
  int32_t iters_1d, s1_lin, s1_bin, s2_lin, s2_bin;
  int32_t keep_intermediates; /* keep stage outputs for odc_copy_array */
  int32_t method;             /* 0 dual contouring (contour); marching-cubes baseline
                                 (baseline.marching_cubes, baseline.py:48-127): 1 binary, 2 continuous */
  double s1_range, s2_range, qef_truncation, fd_step_factor;
} odc_options;

/* eval categories (EvalCounter, pipeline.py:30-57) */
#define ODC_CAT_LABELS 0
#define ODC_CAT_SEARCH_1D 1
#define ODC_CAT_PROBE_FACE_CENTER 2
#define ODC_CAT_PROBE_FACE_MIDPOINT 3
#define ODC_CAT_SEARCH_2D 4
#define ODC_CAT_FD_GRADIENT 5
#define ODC_N_CAT 6

typedef struct {
  int64_t n_grid_vertices, boundary_inside_vertices;
  int64_t n_crossing_edges, n_crossing_faces, n_face_center_probes, n_crossing_cells;
  int64_t n_2d_points, n_partitions, n_plane_samples;
  int64_t point2d_status_counts[4]; /* exact, midpoint-fallback, clamped, range-exhausted */
  int64_t qef_rank_counts[4];       /* rank 0..3 */
  int64_t split_case_counts[4];     /* index 1..3 */
  double qef_max_residual;
  int64_t normal_fallbacks, skipped_boundary_edges;
  int64_t raw_n_vertices, raw_n_triangles, n_vertices, n_triangles;
  int64_t repair_added_vertices, repair_passes;
  int64_t eval_batches[ODC_N_CAT], eval_evals[ODC_N_CAT];
  int32_t cat_order[ODC_N_CAT]; /* first-record order, -1 terminated */
  int32_t n_kernel_launches;
  float device_ms; /* CUDA-event time of the whole extraction on its stream */
  /* CUDA-event time per stage: 0 labels, 1 active sets, 2 1D points + face
   * probes, 3 normals (2D points / fd), 4 cells + QEF, 5 polygonize, 6 repair,
   * 7 the grid-label evaluation kernel alone (the dominant kernel). */
  float stage_ms[8];
} odc_stats;

int odc_version(void);
int odc_create(int device, odc_ctx** out);
void odc_destroy(odc_ctx* ctx);
const char* odc_last_error(const odc_ctx* ctx);
/* stream: a cudaStream_t passed as void* (NULL = the context's own stream).
 * Synchronises the previous stream first: a context's launches stay ordered
 * (its MLP evaluator takes work from a per-context device counter). */
int odc_set_stream(odc_ctx* ctx, void* stream);
/* Parameters: "mbar_timeout_ms" -- the MLP evaluator's mbarrier waits trap
 * (kernel error) after this long without progress, default 4000, 0 = wait
 * forever (debuggers, MPS/preemption); device-wide.  Profiling only (they
 * affect odc_profile_mlp, never an extraction): "mlp_debug" = timing-
 * experiment bits, "profile_points" = a host pointer to (n, 3) f64 points
 * that odc_profile_mlp evaluates with mlp_debug bit 128 (0 = grid points). */
int odc_set_param(odc_ctx* ctx, const char* name, int64_t value);

int odc_field_analytic(odc_ctx* ctx, const odc_node* nodes, int32_t n_nodes, int32_t continuous,
                       double iso_level, odc_field** out);
int odc_field_mlp(odc_ctx* ctx, const odc_mlp_desc* desc, odc_field** out);
/* MeshWindingField (fields.py:281-386): occupancy from a triangle mesh,
 * raw = generalized winding number (continuous), label = raw > 1/2; queries
 * on the surface are perturbed like the reference's "perturb" mode. */
int odc_field_mesh(odc_ctx* ctx, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                   int64_t n_triangles, odc_field** out);
/* VoxelField (fields.py:245-278): trilinear interpolation of a dense
 * (nx, ny, nz) C-order f64 grid at origin + index * spacing, zero outside;
 * continuous, label = raw > 1/2. */
int odc_field_voxels(odc_ctx* ctx, const double origin[3], const double spacing[3], const double* values, int64_t nx,
                     int64_t ny, int64_t nz, odc_field** out);
/* Any other occupancy function (the reference's field duck type: an object
 * with eval_raw, fields.py:51-61): the pipeline runs on the device and calls
 * fn(user, points, n, labels, raw, stream) for every batch of query points
 * it would pass to eval_raw -- the grid (in chunks), the 1D bisection steps,
 * the face probes, the 2D search steps.  points: device (n,3) f64, complete
 * when fn is called; fn writes labels (device u8, raw > iso) and, when raw is
 * not NULL, raw (device f64), complete when it returns.  Return 0 on
 * success; non-zero aborts the extraction with ODC_E_CALLBACK.  stream is
 * the context's cudaStream_t (fn may enqueue on it and synchronise). */
typedef int (*odc_eval_fn)(void* user, const double* points, int64_t n, uint8_t* labels, double* raw, void* stream);
int odc_field_callback(odc_ctx* ctx, odc_eval_fn fn, void* user, int32_t continuous, double iso_level,
                       odc_field** out);
void odc_field_free(odc_ctx* ctx, odc_field* f);

void odc_default_options(odc_options* o);
int odc_extract(odc_ctx* ctx, const odc_field* field, const double lo[3], const double hi[3], int64_t resolution,
                const odc_options* opt, odc_stats* stats);

/* ---- batches (BASELINE config 5: many analytic shapes, throughput) -------
 * nb analytic fields, shape b on the grid lo[3b..3b+2]..hi[3b..3b+2] at the
 * common resolution R, extracted together: the shapes' grids are stacked
 * along z, so every stage is one launch over all of them (the shape is the
 * high part of the flat index) and the per-extraction host round trips are
 * paid once per batch.  Each shape's result equals odc_extract of that shape
 * alone (the reference runs the shapes one by one, pipeline.py:154-240; the
 * elements of a shape never interact with another's, search.py:1-6).  stats:
 * nb entries.  Dual contouring with two-d-point normals only.
 * Replaces a host loop over occmesh.pipeline.contour (pipeline.py:154). */
int odc_extract_batch(odc_ctx* ctx, const odc_field* const* fields, int32_t nb, const double* lo, const double* hi,
                      int64_t resolution, const odc_options* opt, odc_stats* stats);
/* per-shape layout of the last batch (nb + 1 starts, nb raw counts): shape b
 * owns vertex rows [vertex_start[b], vertex_start[b+1]) (its first
 * raw_vertices[b] rows are the raw mesh's vertices) and triangle rows
 * [triangle_start[b], triangle_start[b+1]) */
int odc_batch_layout(odc_ctx* ctx, int64_t* vertex_start, int64_t* raw_vertices, int64_t* triangle_start);
/* every shape's repaired mesh (vertices, triangles with shape-local vertex
 * ids, provenance with shape-local refs) and raw triangles, concatenated in
 * shape order; any pointer may be NULL.  Raw triangle rows are written only
 * for shapes whose repair added vertices (the others' raw mesh is the
 * repaired one). */
int odc_copy_batch_meshes(odc_ctx* ctx, double* vertices, int64_t* triangles, int64_t* raw_triangles,
                          int64_t* prov_kind, int64_t* prov_ref);

/* ---- z-slab mode (multi-GPU) --------------------------------
 * A rank extracts the owned cell layers [cell_z0, cell_z1) of the global grid
 * plus a recomputed one-layer halo below (no halo data exchange).  Local
 * vertex ids: [0, n_halo) halo-layer partitions (owned by the rank below),
 * [n_halo, n_window) owned partitions, [n_window, n_window + n_fans) fan
 * vertices of owned edges.  After an all-gather of (n_partitions, n_fans)
 * the host calls odc_slab_globalize with the rank's global offsets; rank 0
 * concatenates every rank's owned vertices/triangles in rank order (which is
 * the reference's global order) and calls odc_mesh_finish, which drops
 * unreferenced vertices and repairs (polygonize.py:199-209, :253-374).
 * Device pointers stay valid until the next call on the context. */
typedef struct {
  int64_t n_halo_partitions, n_partitions, n_window_partitions, n_fans, n_triangles;
  const double* partition_vertices; /* device (n_partitions,3) owned partition vertices */
  const double* fan_vertices;       /* device (n_fans,3) */
  const int32_t* triangles;         /* device (n_triangles,3), local ids */
  const int64_t* partition_cell;    /* device (n_partitions) provenance ref[0] */
  const int64_t* partition_index;   /* device (n_partitions) provenance ref[1] */
  const int64_t* fan_edge;          /* device (n_fans) provenance ref[0] of fan vertices */
} odc_slab_info;
int odc_extract_slab(odc_ctx* ctx, const odc_field* field, const double lo[3], const double hi[3],
                     int64_t resolution, const odc_options* opt, int64_t cell_z0, int64_t cell_z1,
                     odc_stats* stats, odc_slab_info* info);
/* rewrite the last slab's local triangle ids to global ids (device int32 (T,3)) */
int odc_slab_globalize(odc_ctx* ctx, int64_t part_base, int64_t n_partitions_total, int64_t fan_base,
                       int32_t* triangles_out);
/* Distributed finish (no gather of the whole mesh to one rank).  Only the
 * partitions of a slab's top cell layer are referenced by another rank's
 * triangles (the next rank's, through its halo); with those "seam"
 * triangles every vertex's whole fan is on its own rank:
 *   1. odc_slab_seam: the last slab's triangles with a halo corner (local ids;
 *      triangles_out NULL = count only) -- sent to the previous rank;
 *   2. odc_slab_local_finish(seam of the next rank, its n_halo): marks and
 *      compacts the used owned partitions (polygonize.py:199-209) and counts
 *      owned vertices whose fan is not one closed disc;
 *   3. if no rank reports such a vertex the reference's repair
 *      (polygonize.py:253-374) adds nothing: with the all-gathered used
 *      counts, odc_slab_top_ids gives the next rank the global ids of this
 *      rank's top-layer partitions, and odc_slab_final writes the final
 *      triangles (global ids) and the compacted partition vertices and
 *      provenance; otherwise the host falls back to odc_mesh_finish. */
int odc_slab_seam(odc_ctx* ctx, int32_t* triangles_out, int64_t* n_triangles);
int odc_slab_local_finish(odc_ctx* ctx, const int32_t* next_seam, int64_t n_seam, int64_t next_n_halo,
                          int64_t* n_used_partitions, int64_t* n_nondisc);
int odc_slab_top_ids(odc_ctx* ctx, int64_t part_base, int64_t n_top, int32_t* ids_out);
int odc_slab_final(odc_ctx* ctx, int64_t part_base, int64_t fan_base, const int32_t* halo_ids, int32_t* triangles_out,
                   double* part_vertices_out, int64_t* part_cell_out, int64_t* part_index_out);
/* finish an assembled mesh (device or host pointers): unused-vertex removal +
 * repair; the result is read back with odc_copy_mesh / odc_mesh_device. */
int odc_mesh_finish(odc_ctx* ctx, const double* vertices, int64_t n_vertices, const int32_t* triangles,
                    int64_t n_triangles, int64_t n_partitions, const int64_t* prov_kind, const int64_t* prov_ref,
                    int32_t repair, odc_stats* stats);

/* which: 0 = repaired mesh, 1 = raw (pre-repair) mesh.  Buffers sized from stats. */
int odc_copy_mesh(odc_ctx* ctx, int32_t which, double* vertices, int64_t* triangles, int64_t* prov_kind,
                  int64_t* prov_ref);
/* the repaired mesh and the raw mesh's triangles in one pipelined transfer
 * (ContourResult.mesh + raw_mesh when repair added vertices: the raw mesh's
 * vertices/provenance are the first raw_n_vertices rows of the repaired one,
 * its triangles differ).  raw_triangles: (raw_n_triangles, 3), may be NULL. */
int odc_copy_mesh_pair(odc_ctx* ctx, double* vertices, int64_t* triangles, int64_t* prov_kind, int64_t* prov_ref,
                       int64_t* raw_triangles);
/* zero-copy device view of the last mesh: vertices (V,3) f64, triangles (T,3) i32 */
int odc_mesh_device(odc_ctx* ctx, int32_t which, const double** vertices, const int32_t** triangles,
                    int64_t* n_vertices, int64_t* n_triangles);

/* intermediate arrays (requires keep_intermediates) */
#define ODC_ARR_LABELS 0         /* u8  (S^3)                          */
#define ODC_ARR_EDGE_KEY 1       /* i64 (K)                            */
#define ODC_ARR_FACE_KEY 2       /* i64 (F)                            */
#define ODC_ARR_FACE_NCROSS 3    /* i64 (F)                            */
#define ODC_ARR_CELLS 4          /* i64 (C)                            */
#define ODC_ARR_INSTANCE_EDGES 5 /* i64 (Q,2)                          */
#define ODC_ARR_T1D 6            /* f64 (K)                            */
#define ODC_ARR_POS1D 7          /* f64 (K,3)                          */
#define ODC_ARR_POS2 8           /* f64 (Q,2)                          */
#define ODC_ARR_STATUS 9         /* u8  (Q)                            */
#define ODC_ARR_PART_CELL 10     /* i64 (P)                            */
#define ODC_ARR_PART_INDEX 11    /* i64 (P)                            */
#define ODC_ARR_CYC_LEN 12       /* i64 (P) cycle length per partition */
#define ODC_ARR_CYC_EDGES 13     /* i64 (Ns)                           */
#define ODC_ARR_CYC_INSTS 14     /* i64 (Ns)                           */
#define ODC_ARR_NORMALS 15       /* f64 (Ns,3)                         */
#define ODC_ARR_QEF_POS 16       /* f64 (P,3)                          */
#define ODC_ARR_QEF_RANK 17      /* i64 (P)                            */
#define ODC_ARR_QEF_RESID 18     /* f64 (P)                            */
#define ODC_ARR_SPLIT_CASES 19   /* i64 (n_interior)                   */
#define ODC_ARR_V_IN 20          /* i64 (K)                            */
#define ODC_ARR_MID_LABEL 21     /* u8  (Q)                            */
#define ODC_ARR_POS3 22          /* f64 (Q,3)                          */
#define ODC_ARR_DUP_SOURCE 23    /* i64 (V-V_raw): raw vertex of each repair duplicate */
#define ODC_N_ARR 24
/* Returns the element count (not bytes) in *n_elems; copies if dst != NULL. */
int odc_copy_array(odc_ctx* ctx, int32_t which, void* dst, int64_t dst_bytes, int64_t* n_elems);

/* Batched field evaluation on the device: raw values (1.0/0.0 for analytic
 * fields and for the MLP in shared-field mode) for host points (n,3) f64. */
int odc_eval_raw(odc_ctx* ctx, const odc_field* field, const double* points, int64_t n, double* raw);
/* Profiling hook (tracing): run the MLP evaluator over n grid points
 * and return CTA 0's clock64 event timeline (trace_len >= 256 int64 slots). */
int odc_profile_mlp(odc_ctx* ctx, const odc_field* field, int64_t n, int64_t* trace, int64_t trace_len);
/* Same, labels only (u8), for host points. */
int odc_eval_labels(odc_ctx* ctx, const odc_field* field, const double* points, int64_t n, uint8_t* labels);

/* Slab balancing probe (SURVEY 8(e) "Balance"; no reference counterpart --
 * the reference has no multi-GPU path): for an analytic field on the grid
 * (lo, hi, R), the number of cubic boxes of `box` vertices per side whose
 * interval bound (the label pass's culling test) cannot exclude the surface,
 * per box layer along z: counts has ceil(R / box) entries.  Proportional to
 * the surface area in each z-range, thin walls included.  ODC_E_ARG for
 * fields without an interval bound (MLP, mesh winding, voxels, callbacks). */
int odc_surface_probe(odc_ctx* ctx, const odc_field* field, const double lo[3], const double hi[3], int64_t R,
                      int64_t box, int64_t* counts);

/* MLP parity hook: the fp32 head dot product h_7 . w_head (before b_head and
 * the fp64 prior) of every point, as the tcgen05 evaluator computes it
 * (bf16 operands, fp32 accumulation) -- compared against a bf16-emulating
 * numpy reference in tests/test_gpu_mlp.py. */
int odc_eval_mlp_dot(odc_ctx* ctx, const odc_field* field, const double* points, int64_t n, float* dot);

/* numpy.linalg.eigh of n symmetric 3x3 matrices (row-major, 9 f64 each), as
 * solve_qef_batch calls it (dualize.py:358): LAPACK dsyevd('V', 'L') of
 * numpy's OpenBLAS, reproduced bit for bit (odc_eigh3.cuh).  w (n,3)
 * ascending, V (n,3,3) = numpy's v (columns are eigenvectors), info (n) =
 * LAPACK's info.  odc_eigh3 runs on ctx's device (host buffers in and out);
 * odc_eigh3_host runs the same code on the calling CPU thread.  The QEF
 * kernel inlines the same solver; these are its test hooks. */
int odc_eigh3(odc_ctx* ctx, const double* A, int64_t n, double* w, double* V, int32_t* info);
int odc_eigh3_host(const double* A, int64_t n, double* w, double* V, int32_t* info);

/* Mesh validation on the device (replaces occmesh.mesh.validate_manifold,
 * mesh.py:91-150).  Triangles are host int64 (n_triangles, 3) indexing
 * n_vertices vertices.  Counts come back in the report; the lists
 * (non-manifold edges (a, b) a < b by key, pinched and isolated vertex ids,
 * all ascending) are then copied with odc_validate_copy into caller buffers
 * of those sizes.  Uses its own workspace: the context's last extraction
 * stays readable. */
typedef struct {
  int32_t manifold, pad;
  int64_t n_nonmanifold_edges, n_pinched_vertices, n_boundary_edges, n_isolated_vertices;
} odc_manifold_report;
int odc_validate_manifold(odc_ctx* ctx, const int64_t* triangles, int64_t n_triangles, int64_t n_vertices,
                          odc_manifold_report* report);
int odc_validate_copy(odc_ctx* ctx, int64_t* nonmanifold_edges, int64_t* pinched_vertices,
                      int64_t* isolated_vertices);

/* Self-intersection count on the device (replaces
 * occmesh.mesh.count_self_intersections(mesh, tolerance, return_pairs),
 * mesh.py:395-487): triangle pairs with positive-measure intersection, pairs
 * sharing a vertex or involving a degenerate triangle excluded, decided in
 * the reference's fp64 arithmetic order.  The sorted (a, b) pairs of the last
 * call are copied with odc_self_intersection_pairs into a (count, 2) buffer. */
int odc_count_self_intersections(odc_ctx* ctx, const double* vertices, int64_t n_vertices,
                                 const int64_t* triangles, int64_t n_triangles, double tolerance, int64_t* count);
int odc_self_intersection_pairs(odc_ctx* ctx, int64_t* pairs);

/* Exact point-to-mesh distances on the device (replaces
 * occmesh.mesh.MeshDistanceIndex(mesh).query(points), mesh.py:202-270):
 * per point the distance, the closest triangle (smallest index on exact
 * ties) and the closest point (n_points, 3); tri / closest may be NULL.
 * The building block of the MD2 / HDD / NIC metrics (metrics.py:26-70). */
int odc_mesh_distance(odc_ctx* ctx, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                      int64_t n_triangles, const double* points, int64_t n_points, double* dist, int64_t* tri,
                      double* closest);

/* Triangle areas (TriangleMesh.areas, mesh.py:57-61), bit-identical to numpy;
 * feeds surface sampling for the metrics. */
int odc_triangle_areas(odc_ctx* ctx, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                       int64_t n_triangles, double* areas);

/* Mesh output formats (replaces occmesh.meshio.export_obj / export_ply,
 * meshio.py:22-28 and :79-98).  Host-only, no context needed; vertices
 * (n_vertices, 3) f64 and triangles (n_triangles, 3) int64, as in
 * TriangleMesh.  OBJ bytes are identical to the reference writer (%.17g,
 * 1-based faces); PLY is binary little-endian float32 / uchar+3 int32. */
int odc_export_obj(const char* path, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                   int64_t n_triangles);
int odc_export_ply(const char* path, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                   int64_t n_triangles);

#ifdef __cplusplus
}
#endif
#endif
