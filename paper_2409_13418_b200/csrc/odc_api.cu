// odc_api.cu -- libodc C-ABI (include/odc.h): contexts, device workspace,
// field upload and the extraction driver (the device counterpart of
// occmesh.pipeline.contour, pipeline.py:154-240).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <chrono>

#include "../../include/odc.h"
#include "odc_kernels.h"
#include "odc_mlp.h"
#include "odc_tables.h"

using namespace odc;

namespace {

// Bump allocator over retained device blocks.  reset() makes the whole
// workspace available again; blocks are merged so a repeated extraction of
// the same size never calls cudaMalloc.
struct Arena {
  struct Block {
    char* p;
    size_t size, used;
  };
  std::vector<Block> blocks;
  size_t high_water = 0, live = 0;

  ~Arena() {
    for (auto& b : blocks) cudaFree(b.p);
  }
  void reset() {
    size_t total = 0;
    for (auto& b : blocks) total += b.size;
    if (blocks.size() > 1) {
      for (auto& b : blocks) cudaFree(b.p);
      blocks.clear();
      Block b{nullptr, total, 0};
      if (cudaMalloc(&b.p, total) == cudaSuccess) blocks.push_back(b);
    }
    for (auto& b : blocks) b.used = 0;
    live = 0;
  }
  void* alloc(size_t n) {
    n = (n + 255) & ~(size_t)255;
    if (n == 0) n = 256;
    for (auto& b : blocks)
      if (b.size - b.used >= n) {
        void* p = b.p + b.used;
        b.used += n;
        live += n;
        high_water = std::max(high_water, live);
        return p;
      }
    size_t want = std::max(n, blocks.empty() ? (size_t)64 << 20 : blocks.back().size * 2);
    Block b{nullptr, want, 0};
    if (cudaMalloc(&b.p, want) != cudaSuccess) {
      cudaGetLastError();
      want = n;
      b.size = n;
      if (cudaMalloc(&b.p, want) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
    }
    blocks.push_back(b);
    return alloc(n);
  }
  template <typename T>
  T* get(int64_t count) {
    return static_cast<T*>(alloc(sizeof(T) * (size_t)std::max<int64_t>(count, 1)));
  }
};

struct OdcError {
  int code;
  std::string msg;
};

}  // namespace

struct odc_field {
  int kind;  // 0 analytic, 1 MLP
  odc_node* nodes = nullptr;
  int32_t n_nodes = 0;
  FieldP fp{};  // the kernels' by-value view (fast-path parameters included)
  int32_t continuous = 0;
  double iso = 0.5;
  // MLP
  uint16_t* w_tc = nullptr;
  float* bias = nullptr;
  float* w_head = nullptr;
  MlpDev mlp{};
  // mesh winding-number field (kind 2)
  WindDev wind{};
  void* wind_buf = nullptr;
  // voxel field (kind 3)
  VoxDev vox{};
  // host callback field (kind 4): the caller's own occupancy function
  odc_eval_fn cb = nullptr;
  void* cb_user = nullptr;
};

struct odc_ctx {
  int device = 0;
  cudaStream_t own = nullptr, stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evs[9] = {};  // stage boundaries
  Arena arena;
  CellTabEntry* table = nullptr;
  // small readback buffer (4 KB): [0, 256) readback() ([8, 32) the
  // statistics block of finish_mesh), [256, 258) the device
  // status (readback_checked), [300, 310) a window's owned ranges and
  // partition bounds, [320] a slab's seam count
  unsigned long long* h_pinned = nullptr;
  unsigned int* d_fail = nullptr;          // device flag: a winding query stayed on the surface
  unsigned long long* d_sched = nullptr;   // MLP evaluator's pair counters: [0] only grows, [1] compacted batches
  unsigned long long sched_next = 0;       // its value when the next launch starts
  // odc_set_param("step_trace"), profiling only: 1 = per-step event timings
  // of the 2D lock-step search to stderr, 2 = also every evaluator launch's
  // per-CTA start/end spread, 3 = 1 after a 300 ms idle (a cool GPU)
  int step_trace = 0;
  unsigned long long* trace_buf = nullptr;
  char* h_stage = nullptr;  // grow-only pinned staging for mesh copy-back
  // mesh validation (its own workspace: the last extraction stays valid)
  Arena varena;
  std::vector<int64_t> v_edges, v_pinched, v_isolated;
  std::vector<int64_t> v_si_pairs;
  size_t h_stage_bytes = 0;
  std::vector<cudaEvent_t> copy_evs;       // one per staged piece of a mesh copy
  std::string err;
  int launches = 0;
  // look-back scan status words (scan1 / scan2)
  unsigned long long* scan_status = nullptr;
  int64_t scan_status_words = 0;
  uint32_t scan_epoch = 0;
  // the statistics block as read back with the used-partition count
  // (finish_mesh): final by then, so finish_stats needs no readback of its own
  DevStats h_stats{};
  bool stats_cached = false;
  int mlp_debug = 0;  // odc_set_param("mlp_debug"): profiling experiments, odc_profile_mlp only
  const double* profile_pts = nullptr;  // odc_set_param("profile_points"): host (n,3) points for odc_profile_mlp
  // last extraction
  bool valid = false;
  GridP g{};
  int64_t K = 0, Q = 0, C = 0, F = 0, F4 = 0, P = 0, Ns = 0, NF = 0, T = 0, V0 = 0, V1 = 0, n_interior = 0;
  bool keep = false;
  uint32_t* L = nullptr;
  RecView rec{};  // sparse word records (active words only)
  int64_t A = 0;  // active words
  int64_t *edge_key = nullptr, *inst_key = nullptr, *cell_id = nullptr, *f4_key = nullptr, *face_key = nullptr,
          *face_nc = nullptr;
  int64_t* v_in = nullptr;
  int64_t* inst_edges = nullptr;
  double *t1d = nullptr, *pos1d = nullptr;
  Stage2D s2{};
  CellOut cells{};
  double* verts0 = nullptr;  // raw mesh vertices
  int32_t* tris0 = nullptr;
  int64_t* src0 = nullptr;   // raw vertex -> pre-compaction index (nullptr = identity)
  double* verts1 = nullptr;  // repaired
  int32_t* tris1 = nullptr;
  int64_t* fan_edge = nullptr;
  uint8_t* kase = nullptr;
  int64_t* split_cases = nullptr;
  // slab mode (z-slab extraction)
  bool slab_mode = false;
  int64_t e_lo = 0, e_hi = 0, c_lo = 0, c_hi = 0, P_halo = 0, P_own = 0;
  double* slab_verts = nullptr;
  int32_t* slab_tris = nullptr;
  // distributed finish of the last slab (odc_slab_local_finish)
  uint8_t* slab_used = nullptr;    // owned partitions referenced by a triangle
  uint32_t* slab_newid = nullptr;  // their compacted index
  int64_t slab_U = -1;
  // seam of the last slab (triangles with a halo corner), flagged and ranked
  // during odc_extract_slab; odc_slab_seam only gathers them
  uint32_t *seam_flag = nullptr, *seam_rank = nullptr;
  int64_t seam_n = 0;
  // mesh assembled by odc_mesh_finish: provenance supplied by the caller
  int64_t* prov_kind_in = nullptr;
  int64_t* prov_ref_in = nullptr;
  struct DupPass {
    const int64_t* src;  // device: source vertex of each new vertex of the pass
    int64_t base, n;
  };
  std::vector<DupPass> dup_passes;  // repair passes (polygonize.py:348-358)
  // scans kept for the batch split
  uint32_t *pbase = nullptr, *toff = nullptr, *frank = nullptr;
  DevStats* dstats = nullptr;
  // last batch extraction (odc_extract_batch): per-shape row starts
  // (nb + 1) x kBatchCols, vertex starts of the repaired mesh, raw counts,
  // and the stable by-shape vertex order
  int nb = 0;
  std::vector<int64_t> b_bounds, b_vstart, b_v0;
  uint32_t* b_skeys = nullptr;
  int32_t *b_perm = nullptr, *b_local = nullptr;
};

namespace {

#define CUDA_TRY(x)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) throw OdcError{ODC_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

template <typename T>
T* need(T* p) {
  if (!p) throw OdcError{ODC_E_NOMEM, "device workspace allocation failed"};
  return p;
}

void check_launch(odc_ctx* c, int n = 1) {
  c->launches += n;
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) throw OdcError{ODC_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

void readback(odc_ctx* c, const void* dev, size_t bytes) {
  CUDA_TRY(cudaMemcpyAsync(c->h_pinned, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
}

void raise_device_status(odc_ctx* c, const DevStatus& s) {
  if (s.code == ODC_E_ASSERT) {
    int64_t q = s.detail;
    std::string where;
    if (c->nb) {  // batch: the shape whose own extraction raises, and its instance index
      unsigned long long* pre = need(c->arena.get<unsigned long long>(3 * (c->nb + 1)));
      unsigned long long* tot = need(c->arena.get<unsigned long long>(3));
      const unsigned long long t3[3] = {(unsigned long long)c->K, (unsigned long long)c->Q, (unsigned long long)c->C};
      CUDA_TRY(cudaMemcpyAsync(tot, t3, sizeof t3, cudaMemcpyHostToDevice, c->stream));
      for (int b = 0; b < c->nb; b++)
        launch_prefix_at(c->rec, (int64_t)b * c->g.S * c->g.S * c->g.W, c->A, tot, pre + 3 * b, c->stream);
      std::vector<unsigned long long> h(3 * c->nb);
      CUDA_TRY(cudaMemcpyAsync(h.data(), pre, sizeof(unsigned long long) * 3 * c->nb, cudaMemcpyDeviceToHost,
                               c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      int b = 0;
      while (b + 1 < c->nb && (int64_t)h[3 * (b + 1) + 1] <= q) b++;
      q -= (int64_t)h[3 * b + 1];
      where = "shape " + std::to_string(b) + ": ";
    }
    throw OdcError{ODC_E_ASSERT, where + "2D search instance " + std::to_string(q) +
                                     ": no corner label differs from the midpoint"};
  }
  if (s.code) throw OdcError{s.code, "device status " + std::to_string(s.code)};
}
// readback of `bytes` at `dev` that also brings the device status (the 2D
// search's assertion, raised first) in the same synchronisation
void readback_checked(odc_ctx* c, const void* dev, size_t bytes, DevStatus* dstat) {
  if (!dstat) {
    readback(c, dev, bytes);
    return;
  }
  char* h = reinterpret_cast<char*>(c->h_pinned);
  CUDA_TRY(cudaMemcpyAsync(h, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaMemcpyAsync(h + 2048, dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  DevStatus st;
  std::memcpy(&st, h + 2048, sizeof st);
  raise_device_status(c, st);
}

// One MLP evaluator launch on this context's stream and pair counter.
// With src.n_dev (a compacted batch, count known only on the device) the
// launch uses a second pair counter that the producing kernel resets to 0.
void run_mlp(odc_ctx* c, const odc_field* f, const PointSrc& src, int64_t n, uint8_t* lab, double* raw,
             cudaStream_t s, const MlpDev* override_md = nullptr) {
  MlpDev md = override_md ? *override_md : f->mlp;
  unsigned long long base0 = 0;
  md.sched = src.n_dev ? c->d_sched + 1 : c->d_sched;
  if (c->trace_buf && !override_md) {
    CUDA_TRY(cudaMemsetAsync(c->trace_buf, 0, 8 * 2048, s));
    md.trace = c->trace_buf;
  }
  const int k = mlp_eval(md, src, n, lab, raw, s, src.n_dev ? &base0 : &c->sched_next);
  if (k < 0)
    throw OdcError{ODC_E_CUDA, "MLP evaluator: no pair counter on this context or no weights"};
  if (k > 1) c->launches += k - 1;  // the caller's check_launch counts one
}

// Evaluate labels (and optionally raw) of n points through the field.
// A callback field: the device points are complete when the caller's
// function runs (stream synchronised), and its labels/raw are complete when
// it returns (its contract), so the pipeline's ordering holds.
void eval_callback(odc_ctx* c, const odc_field* f, const double* pts, int64_t n, uint8_t* lab, double* raw) {
  if (n == 0) return;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const int rc = f->cb(f->cb_user, pts, n, lab, raw, (void*)c->stream);
  if (rc) throw OdcError{ODC_E_CALLBACK, "the field's evaluation callback failed (" + std::to_string(rc) + ")"};
}

void eval_points(odc_ctx* c, const odc_field* f, const double* pts, int64_t n, uint8_t* lab, double* raw,
                 const int64_t* n_dev = nullptr, const int32_t* out_map = nullptr) {
  if (n == 0) return;
  if (f->kind == 0) {
    FieldP fp = f->fp;
    fp.nodes = f->nodes;
    fp.n_nodes = f->n_nodes;
    fp.iso = f->iso;
    launch_eval_raw_analytic(fp, pts, n, raw, lab, c->stream);
  } else if (f->kind == 2) {
    PointSrc src{pts, GridP{}, 0};
    winding_eval(f->wind, src, n, lab, raw, c->d_fail, c->stream);
  } else if (f->kind == 3) {
    PointSrc src{pts, GridP{}, 0};
    voxel_eval(f->vox, src, n, lab, raw, c->stream);
  } else if (f->kind == 4) {
    eval_callback(c, f, pts, n, lab, raw);
    return;
  } else {
    PointSrc src{pts, GridP{}, 0};
    src.n_dev = n_dev;
    src.out_map = out_map;
    run_mlp(c, f, src, n, lab, raw, c->stream);
  }
  check_launch(c);
}

// step_trace (profiling): the evaluator launch of one lock-step -- its span
// from the first CTA start to the last CTA end, and the spread of CTA ends
// (the drain tail)
void trace_spans(odc_ctx* c, int step) {
  std::vector<unsigned long long> tb(2048);
  CUDA_TRY(cudaMemcpyAsync(tb.data(), c->trace_buf, 8 * 2048, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
  for (int i = 0; i < 148; i++) {  // slots 400 + 2b, 401 + 2b: CTA b's start and end
    const unsigned long long a = tb[400 + 2 * i], z = tb[401 + 2 * i];
    if (!a || !z) continue;
    s0 = std::min(s0, a);
    s1 = std::max(s1, a);
    e0 = std::min(e0, z);
    e1 = std::max(e1, z);
  }
  if (s1) fprintf(stderr, "  step %2d evaluator: span %.1f us, CTA starts spread %.1f us, ends spread %.1f us\n", step,
                  (e1 - s0) * 1e-3, (s1 - s0) * 1e-3, (e1 - e0) * 1e-3);
}
// step_trace: per-step evaluation (evaluator + label fix-up), update and gap times
void trace_steps(odc_ctx* c, std::vector<cudaEvent_t>& tev) {
  CUDA_TRY(cudaEventSynchronize(tev.back()));
  const int nsteps = (int)tev.size() / 3;
  double se = 0, su = 0, sg = 0;
  for (int step = 0; step < nsteps; step++) {
    float e = 0, u = 0, gap = 0;
    cudaEventElapsedTime(&e, tev[3 * step], tev[3 * step + 1]);
    cudaEventElapsedTime(&u, tev[3 * step + 1], tev[3 * step + 2]);
    if (step + 1 < nsteps) cudaEventElapsedTime(&gap, tev[3 * step + 2], tev[3 * step + 3]);
    se += e;
    su += u;
    sg += gap;
    fprintf(stderr, "step %2d: eval %.3f ms  update %.3f ms  gap %.3f ms\n", step, e, u, gap);
  }
  fprintf(stderr, "2D search: eval %.3f  update %.3f  gaps %.3f ms\n", se, su, sg);
  for (auto e : tev) cudaEventDestroy(e);
  tev.clear();
  if (c->trace_buf) {
    cudaFree(c->trace_buf);
    c->trace_buf = nullptr;
  }
}

// MeshWindingField "perturb" mode gave up on a query (fields.py:354-355)
void check_surface(odc_ctx* c) {
  if (!c->d_fail) return;
  readback(c, c->d_fail, 4);
  if (((unsigned int*)c->h_pinned)[0]) {
    CUDA_TRY(cudaMemsetAsync(c->d_fail, 0, 4, c->stream));
    throw OdcError{ODC_E_VALUE, "could not perturb queries off the surface"};
  }
}

OptP make_opt(const odc_options* o, int continuous) {
  OptP p{};
  p.one_d = o->one_d;
  p.normals = o->normals;
  p.split = o->split;
  p.iters_1d = o->iters_1d;
  p.s1_lin = o->s1_lin;
  p.s1_bin = o->s1_bin;
  p.s2_lin = o->s2_lin;
  p.s2_bin = o->s2_bin;
  p.continuous = continuous;
  p.s1_range = o->s1_range;
  p.s2_range = o->s2_range;
  p.qef_trunc = o->qef_truncation;
  p.fd_step = o->fd_step_factor;
  return p;
}

void record(odc_stats* st, int cat, int64_t batches, int64_t evals) {
  int i = 0;
  while (i < ODC_N_CAT && st->cat_order[i] >= 0 && st->cat_order[i] != cat) i++;
  if (i < ODC_N_CAT && st->cat_order[i] < 0) st->cat_order[i] = cat;
  st->eval_batches[cat] += batches;
  st->eval_evals[cat] += evals;
}

// The context's look-back status words (grow-only, never cleared: each
// scan takes a new epoch, see launch_scan_lookback)
unsigned long long* scan_status(odc_ctx* c, int64_t n) {
  const int64_t words = 2 * scan_lookback_tiles(n);
  if (words > c->scan_status_words) {
    if (c->scan_status) cudaFree(c->scan_status);
    c->scan_status = nullptr;
    c->scan_status_words = 0;
    const int64_t want = std::max<int64_t>(words, 4096);
    CUDA_TRY(cudaMalloc(&c->scan_status, sizeof(unsigned long long) * want));
    CUDA_TRY(cudaMemset(c->scan_status, 0, sizeof(unsigned long long) * want));  // epoch 0: never current
    c->scan_status_words = want;
  }
  if (++c->scan_epoch >= (1u << 30)) {  // wrapped: clear so no stale word can match
    CUDA_TRY(cudaMemsetAsync(c->scan_status, 0, sizeof(unsigned long long) * c->scan_status_words, c->stream));
    c->scan_epoch = 1;
  }
  return c->scan_status;
}
// The pipeline's scans run single-pass (decoupled look-back, one launch;
// arrays up to one block pass: one block): measured against the tiled
// reduce-then-scan (three launches), equal at 0.6-4 M elements and faster
// below.
void scan_any(odc_ctx* c, const uint32_t* const* ins, uint32_t* const* outs, int nch, int64_t n,
              unsigned long long* totals) {
  unsigned long long* status = scan_status(c, n);
  check_launch(c, launch_scan_lookback(ins, outs, nch, n, status, c->scan_epoch, totals, c->stream));
}
void scan1(odc_ctx* c, const uint32_t* in, uint32_t* out, int64_t n, unsigned long long* totals) {
  const uint32_t* ins[1] = {in};
  uint32_t* outs[1] = {out};
  scan_any(c, ins, outs, 1, n, totals);
}
void scan2(odc_ctx* c, const uint32_t* a, const uint32_t* b, uint32_t* oa, uint32_t* ob, int64_t n,
           unsigned long long* totals) {
  const uint32_t* ins[2] = {a, b};
  uint32_t* outs[2] = {oa, ob};
  scan_any(c, ins, outs, 2, n, totals);
}

// Drop unreferenced partition vertices (polygonize.py:199-209), then repair
// non-manifold fans (polygonize.py:253-374, up to 4 passes).  verts holds P
// partition vertices followed by NF fan vertices; used marks referenced ones.
// tn_dev (optional): the triangle and fan-vertex totals [T, NF] on the device,
// NF and T then being only upper bounds (the caller sized the mesh without
// reading them back); the first synchronisation here brings the exact
// values, with the statistics and (status) the device status to raise.
// Returns the exact T and NF through T_out / NF_out.
void finish_mesh(odc_ctx* c, double* verts, int64_t P, int64_t NF, int32_t* tris, int64_t T, uint8_t* used,
                 bool repair, odc_stats* st, DevStats* dst, unsigned long long* totals,
                 const unsigned long long* tn_dev = nullptr, DevStatus* status = nullptr, int64_t* T_out = nullptr,
                 int64_t* NF_out = nullptr) {
  cudaStream_t s = c->stream;
  launch_count_used(used, P, dst, s);
  check_launch(c);
  c->src0 = nullptr;
  int64_t V0 = P + NF;
  // the first synchronisation's extra payload: exact totals, device status
  auto queue_first = [&]() {
    if (tn_dev)
      CUDA_TRY(cudaMemcpyAsync(c->h_pinned + 40, tn_dev, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    if (status) CUDA_TRY(cudaMemcpyAsync(c->h_pinned + 256, status, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
  };
  auto take_first = [&]() {
    if (status) {
      DevStatus ds;
      std::memcpy(&ds, c->h_pinned + 256, sizeof ds);
      raise_device_status(c, ds);  // before anything trusts the sizes
    }
    if (tn_dev) {
      T = (int64_t)c->h_pinned[40];
      NF = (int64_t)c->h_pinned[41];
      V0 = P + NF;
    }
  };
  // unused-vertex removal: drop partitions no triangle references
  auto compact = [&](int64_t used_p) {
    uint32_t* u32 = need(c->arena.get<uint32_t>(V0));
    uint32_t* nid = need(c->arena.get<uint32_t>(V0));
    launch_widen_flags(used, V0, u32, s);
    check_launch(c);
    scan1(c, u32, nid, V0, totals + 5);
    double* vc = need(c->arena.get<double>(3 * V0));
    c->src0 = need(c->arena.get<int64_t>(V0));
    launch_remap_vertices(V0, T, used, nid, verts, vc, tris, c->src0, s);
    check_launch(c, 2);
    V0 = used_p + NF;
    verts = vc;
  };
  // Every statistic but the repair's is final here.  The used-partition
  // count rides on the first repair pass's readback: that pass runs on the
  // uncompacted ids (an unreferenced vertex has no fan, so it changes
  // nothing); in the rare case that partitions are unused (open boundaries)
  // the mesh is compacted and the repair starts over.
  auto take_stats = [&]() {
    std::memcpy(&c->h_stats, c->h_pinned + 8, sizeof(DevStats));
    c->stats_cached = true;
    return (int64_t)c->h_stats.used_partitions;
  };
  const bool run = repair && T > 0;
  if (!run) {
    CUDA_TRY(cudaMemcpyAsync(c->h_pinned + 8, dst, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
    queue_first();
    CUDA_TRY(cudaStreamSynchronize(s));
    take_first();
    const int64_t used_p = take_stats();
    if (used_p != P) compact(used_p);
  }
  int64_t curV = V0;
  int passes = 0;
  bool stats_pending = run;
  for (bool restart = run; restart;) {
    restart = false;
    c->dup_passes.clear();
    curV = V0;
    const int32_t* cur = tris;  // read only: each pass writes a new triangle array
    double* cv = verts;
    char* big = nullptr;  // scratch for fans of more than 64 triangles, allocated on first need
    uint8_t* dirty = nullptr;  // passes after the first: only vertices whose fan the last pass changed
    passes = 0;
    for (int pass = 0; pass < 4; pass++) {
      passes++;
      uint32_t* deg = need(c->arena.get<uint32_t>(3 * (curV + 1)));  // deg, cursor, extra: one memset
      uint32_t* cursor = deg + (curV + 1);
      uint32_t* extra = cursor + (curV + 1);
      uint32_t* off = need(c->arena.get<uint32_t>(curV + 1));
      int32_t* inc = need(c->arena.get<int32_t>(3 * T));
      uint32_t* eoff = need(c->arena.get<uint32_t>(curV + 1));
      CUDA_TRY(cudaMemsetAsync(deg, 0, sizeof(uint32_t) * 3 * (curV + 1), s));
      launch_vertex_degree(cur, T, deg, s, dirty, stats_pending ? tn_dev : nullptr);
      check_launch(c);
      scan1(c, deg, off, curV + 1, totals + 6);
      launch_vertex_fill(cur, T, off, cursor, inc, s, dirty, stats_pending ? tn_dev : nullptr);
      check_launch(c);
      launch_repair_count(cv, cur, curV, off, inc, extra, big, dst, s, dirty);
      check_launch(c);
      scan1(c, extra, eoff, curV + 1, totals + 7);
      // the added-vertex total, the fan-overflow flag (and, first pass, the
      // statistics) in one synchronisation
      CUDA_TRY(cudaMemcpyAsync(&c->h_pinned[0], totals + 7, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaMemcpyAsync(&c->h_pinned[1], &dst->repair_overflow, sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s));
      if (stats_pending) {
        CUDA_TRY(cudaMemcpyAsync(c->h_pinned + 8, dst, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
        queue_first();
      }
      CUDA_TRY(cudaStreamSynchronize(s));
      if (stats_pending) {
        stats_pending = false;
        take_first();  // exact T, NF: vertex ids below P + NF are the same under the bound
        curV = V0;
        if (T == 0) {  // no triangle after all: nothing to repair
          passes = 0;
          break;
        }
        const int64_t used_p = take_stats();
        if (used_p != P) {  // compact, then repair the compacted mesh from the start
          CUDA_TRY(cudaMemsetAsync(&dst->repair_overflow, 0, sizeof(unsigned long long), s));
          compact(used_p);
          restart = true;
          break;
        }
      }
      if (!big && c->h_pinned[1]) {  // fans of more than 64 triangles need global scratch: re-run with it
        big = need(c->arena.get<char>(repair_scratch_bytes(T)));
        CUDA_TRY(cudaMemsetAsync(&dst->repair_overflow, 0, sizeof(unsigned long long), s));
        launch_repair_count(cv, cur, curV, off, inc, extra, big, dst, s, dirty);
        check_launch(c);
        scan1(c, extra, eoff, curV + 1, totals + 7);
        readback(c, totals + 7, sizeof(unsigned long long));
      }
      const int64_t E = (int64_t)c->h_pinned[0];
      if (E == 0) break;
      int32_t* next = need(c->arena.get<int32_t>(3 * T));
      CUDA_TRY(cudaMemcpyAsync(next, cur, sizeof(int32_t) * 3 * T, cudaMemcpyDeviceToDevice, s));
      int64_t* src_new = need(c->arena.get<int64_t>(E));
      c->dup_passes.push_back({src_new, curV, E});
      launch_repair_apply(cv, cur, curV, off, inc, eoff, big, next, src_new, s);
      check_launch(c);
      double* nv = need(c->arena.get<double>(3 * (curV + E)));
      CUDA_TRY(cudaMemcpyAsync(nv, cv, sizeof(double) * 3 * curV, cudaMemcpyDeviceToDevice, s));
      launch_copy_vertices(cv, src_new, curV, E, nv, s);
      dirty = need(c->arena.get<uint8_t>(curV + E));
      CUDA_TRY(cudaMemsetAsync(dirty, 0, (size_t)(curV + E), s));
      launch_mark_dirty(cur, next, T, dirty, s);
      check_launch(c, 2);
      cur = next;
      cv = nv;
      curV += E;
    }
    if (!restart) {
      c->verts1 = cv;
      c->tris1 = const_cast<int32_t*>(cur);
    }
  }
  c->verts0 = verts;
  c->tris0 = tris;
  c->V0 = V0;
  st->raw_n_vertices = V0;
  st->raw_n_triangles = T;
  if (!run) {
    c->verts1 = verts;
    c->tris1 = tris;
    c->dup_passes.clear();
  } else {
    st->repair_passes = passes;
  }
  c->V1 = curV;
  st->n_vertices = curV;
  st->n_triangles = T;
  st->repair_added_vertices = curV - V0;
  if (T_out) *T_out = T;
  if (NF_out) *NF_out = NF;
}

// z-window of one extraction: owned cell layers [c0, c1) plus a one-layer
// halo below; the full grid is c0 = 0, c1 = R.
struct Window {
  int64_t c0, c1;
  bool slab;  // stop after polygonization (offsets are assigned across ranks)
};

// batch: nb shapes of resolution R stacked along z (GridP::nb), with their
// geometry and fields in device arrays (odc_extract_batch)
struct BatchIn {
  int nb;
  const double* geo;    // device (nb, 6)
  const FieldP* fields;  // device (nb)
};

void extract(odc_ctx* c, const odc_field* f, const double lo[3], const double hi[3], int64_t R,
             const odc_options* o, odc_stats* st, const Window& win, const BatchIn* bin = nullptr) {
  // ---- validation: GridSpec (grid.py:24-31), ContourOptions.validate (pipeline.py:72-78)
  if (R < 2) throw OdcError{ODC_E_VALUE, "resolution must be at least 2"};
  for (int a = 0; a < 3; a++)
    if (!(hi[a] > lo[a])) throw OdcError{ODC_E_VALUE, "grid box must have positive extent"};
  if (o->one_d < 0 || o->one_d > 2) throw OdcError{ODC_E_CONFIG, "unknown 1D mode"};
  if (o->normals < 0 || o->normals > 1) throw OdcError{ODC_E_CONFIG, "unknown normal mode"};
  if (o->split < 0 || o->split > 1) throw OdcError{ODC_E_CONFIG, "unknown split mode"};
  if (R > 1290) throw OdcError{ODC_E_VALUE, "resolution above 1290 exceeds the 32-bit vertex index space"};
  if (win.c0 < 0 || win.c1 > R || win.c0 >= win.c1) throw OdcError{ODC_E_ARG, "bad slab range"};
  if (o->method < 0 || o->method > 2) throw OdcError{ODC_E_CONFIG, "unknown marching-cubes mode"};
  if (o->method && (win.slab || win.c0 != 0 || win.c1 != R))
    throw OdcError{ODC_E_ARG, "marching cubes runs on the whole grid only"};

  std::memset(st, 0, sizeof *st);
  for (int i = 0; i < ODC_N_CAT; i++) st->cat_order[i] = -1;
  c->valid = false;
  c->launches = 0;
  c->stats_cached = false;
  c->slab_U = -1;
  c->seam_n = 0;  // set again by a slab extraction that has triangles
  c->seam_flag = c->seam_rank = nullptr;
  if (c->trace_buf) {  // a step trace cut short by an error: no tracing from here on
    cudaFree(c->trace_buf);
    c->trace_buf = nullptr;
  }
  c->arena.reset();
  c->keep = o->keep_intermediates != 0;
  cudaStream_t s = c->stream;
  CUDA_TRY(cudaEventRecord(c->ev0, s));

  GridP g{};
  g.R = R;
  g.S = R + 1;
  g.S2 = g.S * g.S;
  g.S3 = g.S2 * g.S;
  g.W = (g.S + 31) / 32;
  g.z0 = win.c0 > 0 ? win.c0 - 1 : 0;  // one halo layer below the owned cells
  g.nz = win.c1 - g.z0 + 1;            // through the top vertex layer of the owned cells
  g.own0 = win.c0;
  g.own1 = win.c1 == R ? g.S : win.c1;  // the last slab owns the top vertex layer
  g.NW = g.nz * g.S * g.W;
  c->slab_mode = win.slab;
  for (int a = 0; a < 3; a++) {
    g.lo[a] = lo[a];
    g.h[a] = (hi[a] - lo[a]) / (double)R;  // cell_size (grid.py:37-40)
  }
  if (bin) {  // shapes stacked along z: shape b holds layers [b S, b S + S)
    g.nb = bin->nb;
    g.geo = bin->geo;
    g.z0 = 0;
    g.nz = (int64_t)bin->nb * g.S;
    g.own0 = 0;
    g.own1 = g.nz;
    g.NW = g.nz * g.S * g.W;
  }
  c->nb = bin ? bin->nb : 0;
  set_word_divisors(g);
  c->g = g;
  const OptP op = make_opt(o, f->continuous);
  FieldP fp = f->fp;  // analytic: nodes + fast-path parameters (odc_field_analytic)
  fp.nodes = f->nodes;
  fp.n_nodes = f->n_nodes;
  fp.kind = f->kind;
  fp.iso = f->iso;
  if (bin) fp.batch = bin->fields;
  const bool mlp = f->kind != 0;  // fields evaluated in lock-step batches (MLP, mesh winding)

  const int nst = bin ? bin->nb : 1;  // statistics blocks: one per shape
  DevStats* dst = need(c->arena.get<DevStats>(nst));
  c->dstats = dst;
  DevStatus* dstat = need(c->arena.get<DevStatus>(1));
  unsigned long long* totals = need(c->arena.get<unsigned long long>(8));
  CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(DevStats) * nst, s));
  CUDA_TRY(cudaMemsetAsync(dstat, 0, sizeof(DevStatus), s));
  CUDA_TRY(cudaMemsetAsync(&dstat->detail, 0x7f, sizeof(int64_t), s));  // ~INT64_MAX: min over reporters

  int marks = 0;
  auto mark = [&](int i) {
    CUDA_TRY(cudaEventRecord(c->evs[i], s));
    marks = i + 1;
  };
  // ---- K1: sample_labels (grid.py:109-126)
  mark(0);
  c->L = need(c->arena.get<uint32_t>(g.NW));
  if (!mlp) {
    launch_labels_analytic(g, fp, c->L, s);
    check_launch(c);
    mark(8);
  } else {
    uint8_t* bytes = need(c->arena.get<uint8_t>(g.nz * g.S2));
    PointSrc src{nullptr, g, g.z0 * g.S2};
    if (f->kind == 2) {
      winding_eval(f->wind, src, g.nz * g.S2, bytes, nullptr, c->d_fail, s);
    } else if (f->kind == 3) {
      voxel_eval(f->vox, src, g.nz * g.S2, bytes, nullptr, s);
    } else if (f->kind == 4) {  // the grid's points in flat vertex order, a few million at a time
      const int64_t nall = g.nz * g.S2, chunk = std::min<int64_t>(nall, 1 << 22);
      double* gp = need(c->arena.get<double>(3 * chunk));
      for (int64_t b0 = 0; b0 < nall; b0 += chunk) {
        const int64_t nb = std::min(chunk, nall - b0);
        launch_grid_points(g, g.z0 * g.S2 + b0, nb, gp, s);
        check_launch(c);
        eval_callback(c, f, gp, nb, bytes + b0, nullptr);
      }
    } else {
      run_mlp(c, f, src, g.nz * g.S2, bytes, nullptr, s);
    }
    check_launch(c);
    mark(8);
    launch_pack_labels(g, bytes, c->L, s);
    check_launch(c);
  }
  record(st, ODC_CAT_LABELS, 1, (g.own1 - g.own0) * g.S2);
  st->n_grid_vertices = (g.own1 - g.own0) * g.S2;

  // ---- K2: extract_active (grid.py:171-296)
  mark(1);
  const int64_t nt = active_tiles(g);
  uint32_t* tiles = need(c->arena.get<uint32_t>(6 * nt));
  c->rec.occ = need(c->arena.get<uint2>(occ_words(g)));
  launch_active_bits(g, c->L, const_cast<uint2*>(c->rec.occ), tiles, dst, s);
  launch_scan_tiles(tiles, nt, 6, totals, s);
  check_launch(c, 2);
  readback(c, totals, 6 * sizeof(unsigned long long));
  const int64_t K = (int64_t)c->h_pinned[0], Q = (int64_t)c->h_pinned[1], C = (int64_t)c->h_pinned[2],
                Fn = (int64_t)c->h_pinned[3], F4 = (int64_t)c->h_pinned[4], A = (int64_t)c->h_pinned[5];
  if (K >= (1ll << 31) || Q >= (1ll << 31)) throw OdcError{ODC_E_VALUE, "crossing set exceeds 2^31 elements"};
  c->K = K;
  c->Q = Q;
  c->C = C;
  c->F = Fn;
  c->F4 = F4;
  c->A = A;
  c->rec.rec = need(c->arena.get<WordRec>(A));
  c->edge_key = need(c->arena.get<int64_t>(K));
  c->inst_key = need(c->arena.get<int64_t>(Q));
  c->cell_id = need(c->arena.get<int64_t>(C));
  c->f4_key = need(c->arena.get<int64_t>(F4));
  c->face_key = c->keep ? need(c->arena.get<int64_t>(Fn)) : nullptr;
  c->face_nc = c->keep ? need(c->arena.get<int64_t>(Fn)) : nullptr;
  launch_active_compact(g, c->L, c->rec, tiles, c->edge_key, c->inst_key, c->cell_id, c->f4_key, c->face_key,
                        c->face_nc, s);
  check_launch(c);
  // owned element ranges: rows are in key order, so ownership by base layer
  // is a contiguous row range [lo, hi) read from the word ranks
  int64_t e_lo = 0, e_hi = K, q_lo = 0, q_hi = Q, c_lo = 0, c_hi = C, f_own = Fn, f4_own = F4;
  int64_t K_own = K, Q_own = Q;
  const bool window = !g.nb && (win.slab || g.z0 != 0 || g.nz != g.S);
  const bool win_top = g.own1 <= g.z0 + g.nz - 1;
  unsigned long long* pre = nullptr;
  if (window) {  // read back with the partition totals (window_ranges, one synchronisation)
    pre = need(c->arena.get<unsigned long long>(8));
    launch_prefix_at(c->rec, (g.own0 - g.z0) * g.S * g.W, A, totals, pre, s);
    check_launch(c);
    if (win_top) {
      launch_prefix_at(c->rec, (g.own1 - g.z0) * g.S * g.W, A, totals, pre + 3, s);
      check_launch(c);
    }
    launch_count_owned_faces(g, c->rec, dst, s);
    check_launch(c);
    CUDA_TRY(cudaMemcpyAsync(&c->h_pinned[300], pre, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&c->h_pinned[306], &dst->faces_own, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
  }
  // owned element ranges: rows are in key order, so ownership by base layer
  // is a contiguous row range [lo, hi) read from the word ranks; call after
  // a synchronisation of the stream
  auto window_ranges = [&]() {
    if (window) {
      const unsigned long long* h = c->h_pinned + 300;
      e_lo = (int64_t)h[0];
      q_lo = (int64_t)h[1];
      c_lo = (int64_t)h[2];
      if (win_top) {
        e_hi = (int64_t)h[3];
        q_hi = (int64_t)h[4];
        c_hi = (int64_t)h[5];
      }
      f_own = (int64_t)h[6];
      f4_own = (int64_t)h[7];
    }
    c->e_lo = e_lo;
    c->e_hi = e_hi;
    c->c_lo = c_lo;
    c->c_hi = c_hi;
    K_own = e_hi - e_lo;
    Q_own = q_hi - q_lo;
    st->n_crossing_edges = K_own;
    st->n_crossing_faces = f_own;
    st->n_crossing_cells = c_hi - c_lo;
  };

  auto finish_stats = [&]() {
    if (f->kind == 2) check_surface(c);  // only the winding field raises through d_fail
    DevStats h;
    if (c->stats_cached) {
      h = c->h_stats;
    } else {
      readback(c, dst, sizeof(DevStats));
      std::memcpy(&h, c->h_pinned, sizeof h);
    }
    st->boundary_inside_vertices = (int64_t)h.boundary_inside;
    for (int i = 0; i < 4; i++) {
      st->point2d_status_counts[i] = (int64_t)h.status[i];
      st->qef_rank_counts[i] = (int64_t)h.rank[i];
      st->split_case_counts[i] = (int64_t)h.split[i];
    }
    double mr;
    std::memcpy(&mr, &h.max_resid_bits, 8);
    st->qef_max_residual = mr;
    st->normal_fallbacks = (int64_t)h.normal_fallbacks;
    st->skipped_boundary_edges = (int64_t)h.skipped;
    CUDA_TRY(cudaEventRecord(c->ev1, s));
    CUDA_TRY(cudaEventSynchronize(c->ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    st->device_ms = ms;
    // stage i spans mark i -> mark i+1 (or the end event)
    for (int i = 0; i < 7; i++) {
      float x = 0.f;
      if (i + 1 < marks) cudaEventElapsedTime(&x, c->evs[i], c->evs[i + 1]);
      else if (i < marks) cudaEventElapsedTime(&x, c->evs[i], c->ev1);
      st->stage_ms[i] = x;
    }
    float k1 = 0.f;
    cudaEventElapsedTime(&k1, c->evs[0], c->evs[8]);
    st->stage_ms[7] = k1;
    st->n_kernel_launches = c->launches;
  };

  if (K == 0) {  // pipeline.py:174-179
    if (window) CUDA_TRY(cudaStreamSynchronize(s));
    window_ranges();
    c->P = c->NF = c->T = c->V0 = c->V1 = c->Ns = c->n_interior = 0;
    c->P_halo = c->P_own = 0;
    c->prov_kind_in = c->prov_ref_in = nullptr;
    c->verts0 = c->verts1 = nullptr;
    c->tris0 = c->tris1 = nullptr;
    c->src0 = nullptr;
    finish_stats();
    c->valid = true;
    return;
  }

  // ---- face_pairings probes (dualize.py:59-70)
  // run: the probes themselves (they set the 4-crossing faces' pairing bits
  // in the word records, which the cell configurations read); rec: their
  // eval accounting, in the reference's category order
  auto face_probes = [&](bool run, bool rec) {
    if (run && F4) {
      if (!mlp) {
        launch_face_center_analytic(g, fp, c->f4_key, F4, c->rec, s);
        check_launch(c);
      } else {
        double* pts = need(c->arena.get<double>(3 * F4));
        uint8_t* lab = need(c->arena.get<uint8_t>(F4));
        launch_face_center_points(g, c->f4_key, F4, pts, s);
        check_launch(c);
        eval_points(c, f, pts, F4, lab, nullptr);
        launch_face_center_scatter(g, c->f4_key, lab, F4, c->rec, s);
        check_launch(c);
      }
    }
    if (!rec) return;
    if (f4_own) record(st, ODC_CAT_PROBE_FACE_CENTER, 1, f4_own);
    st->n_face_center_probes = f4_own;
  };

  if (o->method) {  // ---- marching-cubes baseline (baseline.py:48-127)
    window_ranges();  // whole grid (checked above): nothing pending
    mark(2);
    double* mcpos = need(c->arena.get<double>(3 * K));
    double *raw_in = nullptr, *raw_out = nullptr;
    if (o->method == 2) {  // continuous: inverse lerp of the raw grid values (baseline.py:82-89)
      if (!f->continuous)
        throw OdcError{ODC_E_CONFIG, "continuous marching cubes requires a field with raw values"};
      raw_in = need(c->arena.get<double>(K));
      raw_out = need(c->arena.get<double>(K));
      double* pts = need(c->arena.get<double>(3 * K));
      uint8_t* lab = need(c->arena.get<uint8_t>(K));
      launch_edge_endpoints(g, c->L, c->edge_key, K, 0, pts, s);
      eval_points(c, f, pts, K, lab, raw_in);
      launch_edge_endpoints(g, c->L, c->edge_key, K, 1, pts, s);
      eval_points(c, f, pts, K, lab, raw_out);
      check_launch(c, 2);
    }
    launch_mc_points(g, c->L, c->edge_key, K, raw_in, raw_out, f->iso, mcpos, s);
    check_launch(c);
    c->t1d = nullptr;
    c->pos1d = mcpos;
    face_probes(true, true);
    mark(3);
    mark(4);
    uint16_t* cfg = need(c->arena.get<uint16_t>(C));
    uint32_t* ncyc = need(c->arena.get<uint32_t>(C));
    uint32_t* nsamp = need(c->arena.get<uint32_t>(C));
    uint32_t* ntri = need(c->arena.get<uint32_t>(C));
    uint32_t* toff = need(c->arena.get<uint32_t>(C + 1));
    launch_cell_config(g, c->L, c->rec, c->cell_id, C, c->table, cfg, ncyc, nsamp, s);
    launch_mc_count(C, ncyc, nsamp, ntri, s);
    check_launch(c, 2);
    scan1(c, ntri, toff, C, totals);
    readback(c, totals, sizeof(unsigned long long));
    const int64_t T = (int64_t)c->h_pinned[0];
    st->n_partitions = 0;
    mark(5);
    int32_t* tris = need(c->arena.get<int32_t>(3 * T));
    uint8_t* used = need(c->arena.get<uint8_t>(K));
    CUDA_TRY(cudaMemsetAsync(used, 0, (size_t)K, s));
    launch_mc_fans(g, c->L, c->rec, c->cell_id, C, c->table, cfg, toff, mcpos, tris, used, s);
    check_launch(c);
    c->P = K;
    c->NF = 0;
    c->T = T;
    c->Ns = 0;
    c->n_interior = 0;
    c->prov_kind_in = c->prov_ref_in = nullptr;
    c->cells = CellOut{};
    c->fan_edge = nullptr;
    mark(6);
    finish_mesh(c, mcpos, K, 0, tris, T, used, false, st, dst, totals);
    mark(7);
    finish_stats();
    c->valid = true;
    return;
  }

  // ---- K6, first half: per-cell configurations and the partition / plane
  // sample totals (dualize.py:194-238).  They need only the labels and the
  // word records (with the face-centre probes' pairing bits, so the probes
  // run first; their eval accounting stays in the reference's order below),
  // so they run before the searches: their readback also brings the
  // window's owned ranges and the halo / owned partition bounds (one
  // synchronisation instead of three).
  face_probes(true, false);
  uint16_t* cfg = need(c->arena.get<uint16_t>(C));
  uint32_t* ncyc = need(c->arena.get<uint32_t>(C));
  uint32_t* nsamp = need(c->arena.get<uint32_t>(C));
  uint32_t* pbase = need(c->arena.get<uint32_t>(C + 1));
  c->pbase = pbase;
  uint32_t* sbase = need(c->arena.get<uint32_t>(C + 1));
  launch_cell_config(g, c->L, c->rec, c->cell_id, C, c->table, cfg, ncyc, nsamp, s);
  check_launch(c);
  scan2(c, ncyc, nsamp, pbase, sbase, C, totals);
  if (window) {
    launch_part_bounds(pbase, C, pre, win_top, totals, pre + 6, s);
    check_launch(c);
    CUDA_TRY(cudaMemcpyAsync(&c->h_pinned[308], pre + 6, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  }
  readback(c, totals, 2 * sizeof(unsigned long long));
  const int64_t P = (int64_t)c->h_pinned[0], Ns = (int64_t)c->h_pinned[1];
  window_ranges();
  const int64_t P_halo = window ? (int64_t)c->h_pinned[308] : 0, P_end = window ? (int64_t)c->h_pinned[309] : P;

  // ---- K3: 1D points (pipeline.py:94-123, search.py:71-94)
  mark(2);
  c->t1d = need(c->arena.get<double>(K));
  c->pos1d = need(c->arena.get<double>(3 * K));
  c->v_in = c->keep ? need(c->arena.get<int64_t>(K)) : nullptr;
  if (!mlp) {
    launch_search1d_analytic(g, fp, op, c->L, c->edge_key, K, c->t1d, c->pos1d, c->v_in, s);
    check_launch(c);
  } else {
    double* lo1 = need(c->arena.get<double>(K));
    double* hi1 = need(c->arena.get<double>(K));
    double* pts = need(c->arena.get<double>(3 * K));
    uint8_t* lab = need(c->arena.get<uint8_t>(K));
    double *raw_in = nullptr, *raw_out = nullptr;
    launch_search1d_init(g, c->L, c->edge_key, K, lo1, hi1, s);
    check_launch(c);
    if (op.one_d == ODC_ONE_D_BINARY) {
      for (int it = 0; it < op.iters_1d; it++) {
        launch_search1d_points(g, c->L, c->edge_key, K, lo1, hi1, pts, s);
        check_launch(c);
        eval_points(c, f, pts, K, lab, nullptr);
        launch_search1d_update(K, lab, lo1, hi1, s);
        check_launch(c);
      }
    } else if (op.one_d == ODC_ONE_D_LINEAR && f->continuous) {
      // raw grid values at the endpoints (LabelVolume.raw, grid.py:115-123): lo=0 / hi=1 points
      raw_in = need(c->arena.get<double>(K));
      raw_out = need(c->arena.get<double>(K));
      launch_edge_endpoints(g, c->L, c->edge_key, K, 0, pts, s);
      eval_points(c, f, pts, K, lab, raw_in);
      launch_edge_endpoints(g, c->L, c->edge_key, K, 1, pts, s);
      eval_points(c, f, pts, K, lab, raw_out);
      check_launch(c, 2);
    }
    launch_search1d_finish(g, op, c->L, c->edge_key, K, lo1, hi1, raw_in, raw_out, c->t1d, c->pos1d, c->v_in, s);
    check_launch(c);
  }
  if (op.one_d == ODC_ONE_D_BINARY) record(st, ODC_CAT_SEARCH_1D, op.iters_1d, (int64_t)op.iters_1d * K_own);

  face_probes(false, true);

  // ---- normals: 2D points (search.py:194-322) or fd gradient (pipeline.py:126-151)
  mark(3);
  double* edge_normals = nullptr;
  DevStatus* status_pending = nullptr;
  c->inst_edges = c->keep ? need(c->arena.get<int64_t>(2 * Q)) : nullptr;
  c->s2 = Stage2D{};
  if (op.normals == ODC_NORMALS_2D) {
    // line_binary_search_batch (search.py:116-127) with n_linear == 0
    // divides by zero: its bracket is [-inf, nan], the next query is
    // non-finite and eval_labels raises (fields.py:42-45)
    const bool nan1 = op.s1_lin == 0 && (op.s1_bin > 0 || op.s2_lin + op.s2_bin > 0);
    const bool nan2 = op.s2_lin == 0 && op.s2_bin > 0;
    if (Q > 0 && (nan1 || nan2)) throw OdcError{ODC_E_VALUE, "non-finite query point at index 0"};
    c->s2.pos3 = need(c->arena.get<double>(3 * Q));
    if (c->keep) {
      c->s2.pos2 = need(c->arena.get<double>(2 * Q));
      c->s2.status = need(c->arena.get<uint8_t>(Q));
      c->s2.mid = need(c->arena.get<uint8_t>(Q));
    }
    if (!mlp) {
      launch_search2d_analytic(g, fp, op, c->L, c->rec, c->inst_key, Q, c->pos1d, c->s2, c->inst_edges, dst, dstat,
                               q_lo, q_hi, s);
      check_launch(c);
    } else {
      void* state = need(c->arena.alloc(search2d_state_bytes(Q)));
      double* pts = need(c->arena.get<double>(6 * Q));
      uint8_t* lab = need(c->arena.get<uint8_t>(2 * Q));
      launch_search2d_lockstep_init(g, op, c->L, c->rec, c->inst_key, Q, c->pos1d, state, c->inst_edges, s);
      check_launch(c);
      const int nsteps = search2d_num_steps(op);
      int64_t M = launch_search2d_lockstep_points(g, op, c->inst_key, Q, 0, state, pts, s);
      check_launch(c);
      // linear-scan steps evaluate only the instances (rays) still scanning
      // (CTA-pair evaluator only: it takes the count on the device)
      const bool compact = f->kind == 1;
      int32_t* map = compact ? need(c->arena.get<int32_t>(2 * Q)) : nullptr;
      int64_t* cnt2 = compact ? need(c->arena.get<int64_t>(2)) : nullptr;
      bool packed = false;  // this step's points are compacted
      std::vector<cudaEvent_t> tev;  // step_trace: eval start, eval end, step end per step
      if (c->step_trace) {
        if (c->step_trace == 3) {
          CUDA_TRY(cudaStreamSynchronize(s));
          std::this_thread::sleep_for(std::chrono::milliseconds(300));
        }
        if (c->step_trace == 2) CUDA_TRY(cudaMalloc(&c->trace_buf, 8 * 2048));
        tev.resize(3 * nsteps);
        for (auto& e : tev) CUDA_TRY(cudaEventCreate(&e));
      }
      for (int step = 0; step < nsteps; step++) {
        if (!tev.empty()) CUDA_TRY(cudaEventRecord(tev[3 * step], s));
        if (packed) eval_points(c, f, pts, M, lab, nullptr, cnt2 + (step & 1), map);
        else eval_points(c, f, pts, M, lab, nullptr);
        if (!tev.empty()) CUDA_TRY(cudaEventRecord(tev[3 * step + 1], s));
        if (c->trace_buf) trace_spans(c, step);
        if (step + 1 < nsteps) {  // update + the next step's points in one pass
          const bool was = packed;
          // the first step of each linear scan still has every instance scanning
          packed = compact && search2d_step_is_linear(op, step + 1) && search2d_step_is_linear(op, step);
          if (packed && !was) CUDA_TRY(cudaMemsetAsync(cnt2, 0, 2 * sizeof(int64_t), s));  // a run starts
          M = launch_search2d_lockstep_step(g, op, c->L, c->inst_key, Q, step, lab, state, dstat, pts, s,
                                            packed ? map : nullptr, cnt2, c->d_sched + 1);
        } else {
          launch_search2d_lockstep_update(g, op, c->L, c->inst_key, Q, step, lab, state, dstat, s);
        }
        check_launch(c);
        if (!tev.empty()) CUDA_TRY(cudaEventRecord(tev[3 * step + 2], s));
      }
      if (!tev.empty()) trace_steps(c, tev);
      launch_search2d_lockstep_finish(g, op, c->L, c->rec, c->inst_key, Q, c->pos1d, state, c->s2, dst, q_lo, q_hi,
                                      s);
      check_launch(c);
    }
    status_pending = dstat;  // raised at the triangle-total readback, before the mesh is built
    record(st, ODC_CAT_PROBE_FACE_MIDPOINT, 1, Q_own);
    record(st, ODC_CAT_SEARCH_2D, op.s1_lin + op.s1_bin + op.s2_lin + op.s2_bin,
           (int64_t)(op.s1_lin + op.s1_bin) * Q_own + (int64_t)(op.s2_lin + op.s2_bin) * 2 * Q_own);
    st->n_2d_points = Q_own;
  } else {
    if (!f->continuous)
      throw OdcError{ODC_E_CONFIG, "fd-gradient normals require a field with continuous raw values"};
    if (c->inst_edges) {  // kept stage output: the instance pairs exist in this mode too
      launch_instance_edges(g, c->L, c->rec, c->inst_key, Q, c->pos1d, c->inst_edges, s);
      check_launch(c);
    }
    double* pts = need(c->arena.get<double>(18 * K));
    double* raw = need(c->arena.get<double>(6 * K));
    uint8_t* lab = need(c->arena.get<uint8_t>(6 * K));
    launch_fd_points(g, op, c->pos1d, K, pts, s);
    check_launch(c);
    eval_points(c, f, pts, 6 * K, lab, raw);
    edge_normals = need(c->arena.get<double>(3 * K));
    launch_fd_normals(g, op, c->L, c->edge_key, K, raw, edge_normals, dst, e_lo, e_hi, s);
    check_launch(c);
    record(st, ODC_CAT_FD_GRADIENT, 1, 6 * K_own);
    st->n_2d_points = 0;
  }

  // ---- K6: partitions + plane samples + QEF (dualize.py:194-444)
  mark(4);
  c->P = P;
  c->Ns = Ns;
  c->P_halo = P_halo;
  st->n_partitions = P_end - P_halo;
  st->n_plane_samples = Ns;
  // vertex buffer sized for the worst case of fan vertices (one per owned edge)
  double* verts = need(c->arena.get<double>(3 * (P + K_own)));
  CellOut co{};
  co.verts = verts;
  co.part_cell = need(c->arena.get<int64_t>(P));
  co.part_index = need(c->arena.get<int64_t>(P));
  co.pinfo = need(c->arena.get<uint64_t>(C));
  if (c->keep) {
    co.rank = need(c->arena.get<int64_t>(P));
    co.resid = need(c->arena.get<double>(P));
    co.cyc_edges = need(c->arena.get<int64_t>(Ns));
    co.cyc_insts = need(c->arena.get<int64_t>(Ns));
    co.normals = need(c->arena.get<double>(3 * Ns));
    co.cyc_len = need(c->arena.get<int64_t>(P));
  }
  double* snorm = co.normals ? co.normals : need(c->arena.get<double>(3 * Ns));
  int32_t* srow = need(c->arena.get<int32_t>(Ns));
  uint32_t* psoff = need(c->arena.get<uint32_t>(P + 1));
  launch_cell_solve(g, op, c->L, c->rec, c->cell_id, C, c->table, cfg, pbase, sbase, c->pos1d, c->s2.pos3,
                    edge_normals, co, snorm, srow, psoff, P, dst, c_lo, c_hi, P_halo, P_end, s);
  check_launch(c, 2);
  c->cells = co;

  // ---- K7: build_mesh (polygonize.py:110-217) over the owned edges
  mark(5);
  const int64_t* ekey = c->edge_key + e_lo;
  const double* epos = c->pos1d + 3 * e_lo;
  int4* pid4 = need(c->arena.get<int4>(K_own));
  c->kase = need(c->arena.get<uint8_t>(K_own));
  uint32_t* ntri = need(c->arena.get<uint32_t>(K_own));
  uint32_t* nfan = need(c->arena.get<uint32_t>(K_own));
  uint32_t* toff = need(c->arena.get<uint32_t>(K_own));
  uint32_t* frank = need(c->arena.get<uint32_t>(K_own));
  c->toff = toff;
  c->frank = frank;
  launch_poly_classify(g, op, c->L, c->rec, ekey, K_own, co.pinfo, verts, pid4, c->kase, ntri, nfan, dst, s);
  check_launch(c);
  scan2(c, ntri, nfan, toff, frank, K_own, totals);
  // Small whole-grid extractions size the mesh by its bounds (a crossing
  // edge emits at most 4 triangles and 1 fan vertex) and learn the exact
  // totals at the repair's first synchronisation (finish_mesh), one host
  // round trip fewer.  Past ~256 K edges the bounds double the repair's
  // first pass (vertex range P + K instead of P + NF) -- more than a round
  // trip costs -- and slabs and keep_intermediates need the totals here.
  const bool lazy = !win.slab && !c->keep && K_own <= (int64_t(1) << 18);
  int64_t T = 4 * K_own, NF = K_own;
  if (!lazy) {
    readback_checked(c, totals, 2 * sizeof(unsigned long long), status_pending);  // the 2D status is raised first
    T = (int64_t)c->h_pinned[0];
    NF = (int64_t)c->h_pinned[1];
  }
  c->T = T;
  c->NF = NF;
  int32_t* tris = need(c->arena.get<int32_t>(3 * T));
  c->fan_edge = need(c->arena.get<int64_t>(NF));
  uint8_t* used = need(c->arena.get<uint8_t>(P + NF));
  CUDA_TRY(cudaMemsetAsync(used, 0, (size_t)P, s));
  if (NF) CUDA_TRY(cudaMemsetAsync(used + P, 1, (size_t)NF, s));  // fan vertices are always referenced
  launch_poly_emit(K_own, P, ekey, pid4, c->kase, toff, frank, epos, verts, tris, c->fan_edge, used, s);
  check_launch(c);
  if (c->keep) {
    uint32_t* flag = need(c->arena.get<uint32_t>(K_own));
    uint32_t* rank = need(c->arena.get<uint32_t>(K_own));
    launch_interior_flags(K_own, c->kase, flag, s);
    check_launch(c);
    scan1(c, flag, rank, K_own, totals + 4);
    readback(c, totals + 4, sizeof(unsigned long long));
    c->n_interior = (int64_t)c->h_pinned[0];
    c->split_cases = need(c->arena.get<int64_t>(c->n_interior));
    launch_split_cases(K_own, c->kase, c->split_cases, rank, s);
    check_launch(c);
  }
  c->prov_kind_in = c->prov_ref_in = nullptr;
  if (win.slab) {  // offsets across slabs are assigned by the host (odc_slab_globalize)
    c->slab_verts = verts;
    c->slab_tris = tris;
    c->P_own = P_end - P_halo;
    mark(6);
    // the seam (distributed finish): its count comes back with the statistics
    c->seam_n = 0;
    c->seam_flag = c->seam_rank = nullptr;
    const bool seam = T > 0 && P_halo > 0;
    if (seam) {
      c->seam_flag = need(c->arena.get<uint32_t>(T));
      c->seam_rank = need(c->arena.get<uint32_t>(T));
      launch_seam_flags(tris, T, P_halo, c->seam_flag, s);
      check_launch(c);
      scan1(c, c->seam_flag, c->seam_rank, T, totals + 4);
      CUDA_TRY(cudaMemcpyAsync(&c->h_pinned[320], totals + 4, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    }
    mark(7);
    c->V0 = c->V1 = 0;
    st->raw_n_triangles = st->n_triangles = T;
    finish_stats();  // synchronises
    if (seam) c->seam_n = (int64_t)c->h_pinned[320];
    c->valid = true;
    return;
  }
  // ---- unused-vertex removal + K8 repair (polygonize.py:199-209, :253-374)
  mark(6);
  {
    int64_t Tx = T, NFx = NF;
    // totals[0..1] (triangle / fan totals of the scan above) are not touched by
    // finish_mesh's scans (totals + 5..7)
    finish_mesh(c, verts, P, NF, tris, T, used, o->repair != 0, st, dst, totals, lazy ? totals : nullptr,
                lazy ? status_pending : nullptr, &Tx, &NFx);
    c->T = Tx;
    c->NF = NFx;
  }
  mark(7);
  finish_stats();
  c->valid = true;
}

// ---- batch (odc_extract_batch): per-shape statistics and the by-shape
// vertex order of the finished union mesh (odc_batch.cu)
void batch_split(odc_ctx* c, const odc_options* o, const OptP& op, odc_stats* st) {
  const int nb = c->nb;
  cudaStream_t s = c->stream;
  const GridP& g = c->g;
  c->b_bounds.assign((size_t)(nb + 1) * kBatchCols, 0);
  c->b_vstart.assign(nb + 1, 0);
  c->b_v0.assign(nb, 0);
  std::vector<DevStats> ds(nb);
  CUDA_TRY(cudaMemcpyAsync(ds.data(), c->dstats, sizeof(DevStats) * nb, cudaMemcpyDeviceToHost, s));
  if (c->K) {
    int64_t* bd = need(c->arena.get<int64_t>((nb + 1) * kBatchCols));
    launch_batch_bounds(g, c->rec, c->A, c->K, c->Q, c->C, c->f4_key, c->F4, c->pbase, c->P, c->toff, c->frank, c->T,
                        c->NF, bd, s);
    check_launch(c);
    CUDA_TRY(cudaMemcpyAsync(c->b_bounds.data(), bd, sizeof(int64_t) * (nb + 1) * kBatchCols, cudaMemcpyDeviceToHost,
                             s));
    CUDA_TRY(cudaStreamSynchronize(s));
    // by-shape vertex order of the repaired union mesh
    const int64_t V = c->V1, V0 = c->V0, T = c->T;
    std::vector<int64_t> tstart(nb + 1);
    for (int b = 0; b <= nb; b++) tstart[b] = c->b_bounds[(size_t)b * kBatchCols + 5];
    int64_t* dts = need(c->arena.get<int64_t>(nb + 1));
    CUDA_TRY(cudaMemcpyAsync(dts, tstart.data(), sizeof(int64_t) * (nb + 1), cudaMemcpyHostToDevice, s));
    uint32_t* vshape = need(c->arena.get<uint32_t>(V));
    c->b_skeys = need(c->arena.get<uint32_t>(V));
    int32_t* iota = need(c->arena.get<int32_t>(V));
    c->b_perm = need(c->arena.get<int32_t>(V));
    c->b_local = need(c->arena.get<int32_t>(V));
    int64_t* vc = need(c->arena.get<int64_t>(2 * nb + 1));
    size_t tmp_bytes = 0;
    batch_sort_vertices(c->tris1, T, V, V0, dts, nb, vshape, c->b_skeys, iota, c->b_perm, nullptr, &tmp_bytes, vc, s);
    void* tmp = need(c->arena.alloc(tmp_bytes));
    launch_iota_i32(iota, V, s);
    batch_sort_vertices(c->tris1, T, V, V0, dts, nb, vshape, c->b_skeys, iota, c->b_perm, tmp, &tmp_bytes, vc, s);
    check_launch(c, 4);
    std::vector<int64_t> h(2 * nb + 1);
    CUDA_TRY(cudaMemcpyAsync(h.data(), vc, sizeof(int64_t) * (2 * nb + 1), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int b = 0; b <= nb; b++) c->b_vstart[b] = h[b];
    for (int b = 0; b < nb; b++) c->b_v0[b] = h[nb + 1 + b];
    launch_local_ids(c->b_skeys, c->b_perm, V, vc, c->b_local, s);
    check_launch(c);
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  // per-shape statistics, in the reference's accounting (pipeline.py:160-239)
  const float ms = st[0].device_ms;
  const odc_stats uni = st[0];
  for (int b = 0; b < nb; b++) {
    odc_stats& x = st[b];
    std::memset(&x, 0, sizeof x);
    for (int i = 0; i < ODC_N_CAT; i++) x.cat_order[i] = -1;
    const int64_t* lo = &c->b_bounds[(size_t)b * kBatchCols];
    const int64_t* hi = lo + kBatchCols;
    const int64_t K = hi[0] - lo[0], Q = hi[1] - lo[1], C = hi[2] - lo[2], F4 = hi[3] - lo[3];
    x.n_grid_vertices = g.S3;
    record(&x, ODC_CAT_LABELS, 1, g.S3);
    x.boundary_inside_vertices = (int64_t)ds[b].boundary_inside;
    x.n_crossing_edges = K;
    x.n_crossing_cells = C;
    x.device_ms = ms;
    for (int i = 0; i < 8; i++) x.stage_ms[i] = uni.stage_ms[i];
    x.n_kernel_launches = uni.n_kernel_launches;
    if (K == 0) continue;  // pipeline.py:174-179
    x.n_crossing_faces = Q - F4;
    if (op.one_d == ODC_ONE_D_BINARY) record(&x, ODC_CAT_SEARCH_1D, op.iters_1d, (int64_t)op.iters_1d * K);
    if (F4) record(&x, ODC_CAT_PROBE_FACE_CENTER, 1, F4);
    x.n_face_center_probes = F4;
    record(&x, ODC_CAT_PROBE_FACE_MIDPOINT, 1, Q);
    record(&x, ODC_CAT_SEARCH_2D, op.s1_lin + op.s1_bin + op.s2_lin + op.s2_bin,
           (int64_t)(op.s1_lin + op.s1_bin) * Q + (int64_t)(op.s2_lin + op.s2_bin) * 2 * Q);
    x.n_2d_points = Q;
    x.n_partitions = hi[4] - lo[4];
    for (int i = 0; i < 4; i++) {
      x.point2d_status_counts[i] = (int64_t)ds[b].status[i];
      x.qef_rank_counts[i] = (int64_t)ds[b].rank[i];
      x.split_case_counts[i] = (int64_t)ds[b].split[i];
    }
    std::memcpy(&x.qef_max_residual, &ds[b].max_resid_bits, 8);
    x.normal_fallbacks = (int64_t)ds[b].normal_fallbacks;
    x.skipped_boundary_edges = (int64_t)ds[b].skipped;
    const int64_t Tb = hi[5] - lo[5];
    x.raw_n_triangles = x.n_triangles = Tb;
    x.raw_n_vertices = c->b_v0[b];
    x.n_vertices = c->b_vstart[b + 1] - c->b_vstart[b];
    x.repair_added_vertices = x.n_vertices - x.raw_n_vertices;
    x.repair_passes = uni.repair_passes;
  }
  (void)o;
}

int guard(odc_ctx* c, int (*fn)(odc_ctx*, void*), void* arg) {
  try {
    return fn(c, arg);
  } catch (const OdcError& e) {
    c->err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    c->err = "host allocation failed";
    return ODC_E_NOMEM;
  }
}

}  // namespace

extern "C" {

int odc_version(void) { return 1; }

int odc_create(int device, odc_ctx** out) {
  if (!out) return ODC_E_ARG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return ODC_E_CUDA;
  }
  if (device < 0 || device >= n) return ODC_E_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return ODC_E_CUDA;
  odc_ctx* c = new (std::nothrow) odc_ctx();
  if (!c) return ODC_E_NOMEM;
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess || cudaEventCreate(&c->ev0) != cudaSuccess ||
      cudaEventCreate(&c->ev1) != cudaSuccess || cudaMallocHost(&c->h_pinned, 4096) != cudaSuccess ||
      cudaMalloc(&c->d_fail, 4) != cudaSuccess || cudaMemset(c->d_fail, 0, 4) != cudaSuccess ||
      cudaMalloc(&c->d_sched, 16) != cudaSuccess || cudaMemset(c->d_sched, 0, 16) != cudaSuccess) {
    delete c;
    return ODC_E_CUDA;
  }
  c->stream = c->own;
  {  // field buffers come from the stream-ordered pool; keep freed blocks cached
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  for (auto& e : c->evs)
    if (cudaEventCreate(&e) != cudaSuccess) {
      delete c;
      return ODC_E_CUDA;
    }
  std::vector<CellTabEntry> tab(kTableSize);
  if (build_cell_table(tab.data()) != 0) {
    delete c;
    return ODC_E_CONTRACT;
  }
  if (cudaMalloc(&c->table, sizeof(CellTabEntry) * kTableSize) != cudaSuccess ||
      cudaMemcpy(c->table, tab.data(), sizeof(CellTabEntry) * kTableSize, cudaMemcpyHostToDevice) != cudaSuccess) {
    delete c;
    return ODC_E_CUDA;
  }
  *out = c;
  return ODC_OK;
}

void odc_destroy(odc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->table) cudaFree(c->table);
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->d_fail) cudaFree(c->d_fail);
  if (c->d_sched) cudaFree(c->d_sched);
  if (c->trace_buf) cudaFree(c->trace_buf);
  if (c->scan_status) cudaFree(c->scan_status);
  for (auto e : c->copy_evs) cudaEventDestroy(e);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (auto& e : c->evs)
    if (e) cudaEventDestroy(e);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
}

const char* odc_last_error(const odc_ctx* c) { return c ? c->err.c_str() : "null context"; }

int odc_set_param(odc_ctx* c, const char* name, int64_t value) {
  if (!c || !name) return ODC_E_ARG;
  if (std::strcmp(name, "mlp_debug") == 0 && value >= 0 && value <= 255) {
    c->mlp_debug = (int)value;
    return ODC_OK;
  }
  if (std::strcmp(name, "step_trace") == 0 && value >= 0 && value <= 3) {
    c->step_trace = (int)value;
    return ODC_OK;
  }
  if (std::strcmp(name, "mbar_timeout_ms") == 0 && value >= 0) {  // 0: the MLP evaluator's waits never trap
    cudaSetDevice(c->device);
    if (mlp_set_wait_timeout_ns((unsigned long long)value * 1000000ull) != 0) {
      c->err = "mbar_timeout_ms: cudaMemcpyToSymbol failed";
      return ODC_E_CUDA;
    }
    return ODC_OK;
  }
  if (std::strcmp(name, "profile_points") == 0) {  // profiling only: a host pointer, 0 = generated grid points
    c->profile_pts = (const double*)(intptr_t)value;
    return ODC_OK;
  }
  c->err = std::string("unknown parameter ") + name;
  return ODC_E_ARG;
}

int odc_set_stream(odc_ctx* c, void* stream) {
  if (!c) return ODC_E_ARG;
  // the context's launches must stay ordered (the MLP pair counter is per
  // context): drain the old stream before switching
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return ODC_E_CUDA;
  c->stream = stream ? (cudaStream_t)stream : c->own;
  return ODC_OK;
}

void odc_default_options(odc_options* o) {
  std::memset(o, 0, sizeof *o);
  o->one_d = ODC_ONE_D_BINARY;
  o->normals = ODC_NORMALS_2D;
  o->split = ODC_SPLIT_IC;
  o->repair = 1;
  o->iters_1d = 15;
  o->s1_lin = 4;
  o->s1_bin = 11;
  o->s2_lin = 3;
  o->s2_bin = 12;
  o->s1_range = 0.8;
  o->s2_range = 0.70710678118654757;  // math.sqrt(2.0) / 2.0
  o->qef_truncation = 0.1;
  o->fd_step_factor = 0.01;
}

int odc_field_analytic(odc_ctx* c, const odc_node* nodes, int32_t n_nodes, int32_t continuous, double iso,
                       odc_field** out) {
  if (!c || !out || !nodes || n_nodes <= 0 || n_nodes > ODC_MAX_NODES) return ODC_E_ARG;
  cudaSetDevice(c->device);
  odc_field* f = new (std::nothrow) odc_field();
  if (!f) return ODC_E_NOMEM;
  f->kind = 0;
  f->n_nodes = n_nodes;
  f->continuous = continuous;
  f->iso = iso;
  if (cudaMallocAsync((void**)&f->nodes, sizeof(odc_node) * n_nodes, c->stream) != cudaSuccess ||
      cudaMemcpyAsync(f->nodes, nodes, sizeof(odc_node) * n_nodes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess) {
    c->err = "field upload failed";
    delete f;
    return ODC_E_CUDA;
  }
  f->fp.nodes = f->nodes;
  f->fp.n_nodes = n_nodes;
  f->fp.kind = 0;
  f->fp.iso = iso;
  fieldp_set_fast(f->fp, nodes, n_nodes);
  f->fp.ev = ev_mode_of(f->fp);
  *out = f;
  return ODC_OK;
}

int odc_field_mlp(odc_ctx* c, const odc_mlp_desc* d, odc_field** out) {
  if (!c || !d || !out) return ODC_E_ARG;
  if (d->width != 256 || d->depth != 8 || d->d_in != 39 || d->n_freq != 6) {
    c->err = "the device MLP is specialised to d_in=39, 8 x 256";
    return ODC_E_ARG;
  }
  cudaSetDevice(c->device);
  odc_field* f = new (std::nothrow) odc_field();
  if (!f) return ODC_E_NOMEM;
  f->kind = 1;
  f->continuous = 1;
  f->iso = 0.5;
  const size_t nt = mlp_tc_weight_elems();
  std::vector<uint16_t> packed_tc(nt);
  mlp_pack_weights_tc(d->w0, d->d_in, d->w_hidden, packed_tc.data());
  // stream-ordered pool allocations: no driver round trip per field
  cudaStream_t s = c->stream;
  if (cudaMallocAsync((void**)&f->w_tc, nt * 2, s) != cudaSuccess ||
      cudaMallocAsync((void**)&f->bias, 8 * 256 * 4, s) != cudaSuccess ||
      cudaMallocAsync((void**)&f->w_head, 256 * 4, s) != cudaSuccess) {
    c->err = "field upload failed";
    delete f;
    return ODC_E_NOMEM;
  }
  cudaMemcpyAsync(f->w_tc, packed_tc.data(), nt * 2, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(f->bias, d->biases, 8 * 256 * 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(f->w_head, d->w_head, 256 * 4, cudaMemcpyHostToDevice, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) {  // usable from any stream once created
    c->err = "field upload failed";
    delete f;
    return ODC_E_CUDA;
  }
  f->mlp.w_tc = f->w_tc;
  f->mlp.has_bias = 0;
  for (int i = 0; i < 8 * 256; i++)
    if (d->biases[i] != 0.f) f->mlp.has_bias = 1;
  f->mlp.bias = f->bias;
  f->mlp.w_head = f->w_head;
  for (int i = 0; i < 256; i++) f->mlp.w_head_k[i] = d->w_head[i];
  f->mlp.b_head = (float)d->b_head;
  f->mlp.amplitude = d->amplitude;
  f->mlp.prior_scale = d->prior_scale;
  f->mlp.prior_radius = d->prior_radius;
  for (int i = 0; i < 3; i++) f->mlp.prior_center[i] = d->prior_center[i];
  *out = f;
  return ODC_OK;
}

int odc_field_mesh(odc_ctx* c, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                   int64_t n_triangles, odc_field** out) {
  if (!c || !out || n_vertices < 0 || n_triangles < 0 || (n_vertices && !vertices)) return ODC_E_ARG;
  if (n_triangles == 0 || !triangles) {
    c->err = "mesh field needs at least one triangle";
    return ODC_E_VALUE;
  }
  for (int64_t i = 0; i < 3 * n_triangles; i++)
    if (triangles[i] < 0 || triangles[i] >= n_vertices) {
      c->err = "triangle index out of range";
      return ODC_E_VALUE;
    }
  cudaSetDevice(c->device);
  odc_field* f = new (std::nothrow) odc_field();
  if (!f) return ODC_E_NOMEM;
  f->kind = 2;
  f->continuous = 1;
  f->iso = 0.5;
  // nudge = 1e-9 * max(ptp(vertices, axis=0)) / sqrt(3) (fields.py:311-312)
  double scale = 0.0;
  for (int a = 0; a < 3; a++) {
    double lo = vertices[a], hi = vertices[a];
    for (int64_t i = 1; i < n_vertices; i++) {
      lo = std::min(lo, vertices[3 * i + a]);
      hi = std::max(hi, vertices[3 * i + a]);
    }
    scale = std::max(scale, hi - lo);
  }
  if (scale == 0.0) scale = 1.0;
  const int64_t T = n_triangles;
  const size_t bytes = sizeof(double) * (18 * T + 4 * T) + (size_t)T + sizeof(double) * 3 * n_vertices + 24 * T;
  cudaStream_t s = c->stream;
  char* buf = nullptr;
  if (cudaMallocAsync((void**)&buf, bytes + 512, s) != cudaSuccess) {
    delete f;
    c->err = "field upload failed";
    return ODC_E_NOMEM;
  }
  double* d = (double*)buf;
  WindDev& w = f->wind;
  w.ta = d;
  w.tb = d + 3 * T;
  w.tc = d + 6 * T;
  w.nhat = d + 9 * T;
  w.eab = d + 12 * T;
  w.eac = d + 15 * T;
  w.d00 = d + 18 * T;
  w.d01 = d + 19 * T;
  w.d11 = d + 20 * T;
  w.denb = d + 21 * T;
  double* dv = d + 22 * T;
  int64_t* dt = (int64_t*)(dv + 3 * n_vertices);
  w.ok = (uint8_t*)(dt + 3 * T);
  w.nt = T;
  w.nudge = 1e-9 * scale * 1.0 / std::sqrt(3.0);
  f->wind_buf = buf;
  if (cudaMemcpyAsync(dv, vertices, 24 * n_vertices, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(dt, triangles, 24 * T, cudaMemcpyHostToDevice, s) != cudaSuccess) {
    odc_field_free(c, f);
    return ODC_E_CUDA;
  }
  launch_winding_prep(dv, dt, T, w, s);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) {
    odc_field_free(c, f);
    c->err = "mesh field setup failed";
    return ODC_E_CUDA;
  }
  *out = f;
  return ODC_OK;
}

int odc_field_voxels(odc_ctx* c, const double origin[3], const double spacing[3], const double* values, int64_t nx,
                     int64_t ny, int64_t nz, odc_field** out) {
  if (!c || !out || !origin || !spacing || !values) return ODC_E_ARG;
  if (nx < 2 || ny < 2 || nz < 2) {
    c->err = "voxel values must be at least 2 x 2 x 2";
    return ODC_E_VALUE;
  }
  cudaSetDevice(c->device);
  odc_field* f = new (std::nothrow) odc_field();
  if (!f) return ODC_E_NOMEM;
  f->kind = 3;
  f->continuous = 1;
  f->iso = 0.5;
  const size_t bytes = sizeof(double) * (size_t)nx * ny * nz;
  double* d = nullptr;
  if (cudaMallocAsync((void**)&d, bytes, c->stream) != cudaSuccess ||
      cudaMemcpyAsync(d, values, bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess) {
    if (d) cudaFreeAsync(d, c->stream);
    delete f;
    c->err = "field upload failed";
    return ODC_E_NOMEM;
  }
  f->vox.values = d;
  f->vox.nx = nx;
  f->vox.ny = ny;
  f->vox.nz = nz;
  for (int a = 0; a < 3; a++) {
    f->vox.origin[a] = origin[a];
    f->vox.spacing[a] = spacing[a];
  }
  *out = f;
  return ODC_OK;
}

int odc_field_callback(odc_ctx* c, odc_eval_fn fn, void* user, int32_t continuous, double iso, odc_field** out) {
  if (!c || !fn || !out) return ODC_E_ARG;
  odc_field* f = new (std::nothrow) odc_field();
  if (!f) return ODC_E_NOMEM;
  f->kind = 4;
  f->cb = fn;
  f->cb_user = user;
  f->continuous = continuous;
  f->iso = iso;
  f->fp.kind = 4;
  f->fp.iso = iso;
  *out = f;
  return ODC_OK;
}

void odc_field_free(odc_ctx* c, odc_field* f) {
  if (!f) return;
  if (c) {
    cudaStreamSynchronize(c->stream);
    void* bufs[] = {f->nodes, f->w_tc, f->bias, f->w_head, f->wind_buf,
                    (void*)f->vox.values};
    for (void* b : bufs)
      if (b) cudaFreeAsync(b, c->stream);  // back to the pool, no device-wide sync
  } else {
    cudaDeviceSynchronize();
    void* bufs[] = {f->nodes, f->w_tc, f->bias, f->w_head, f->wind_buf,
                    (void*)f->vox.values};
    for (void* b : bufs)
      if (b) cudaFreeAsync(b, 0);
    cudaDeviceSynchronize();
  }
  delete f;
}

struct ExtractArgs {
  const odc_field* f;
  const double* lo;
  const double* hi;
  int64_t R;
  const odc_options* o;
  odc_stats* st;
};

int odc_extract(odc_ctx* c, const odc_field* f, const double lo[3], const double hi[3], int64_t R,
                const odc_options* o, odc_stats* st) {
  if (!c || !f || !lo || !hi || !st) return ODC_E_ARG;
  odc_options def;
  odc_default_options(&def);
  ExtractArgs a{f, lo, hi, R, o ? o : &def, st};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    ExtractArgs* x = (ExtractArgs*)p;
    extract(cc, x->f, x->lo, x->hi, x->R, x->o, x->st, Window{0, x->R, false});
    return (int)ODC_OK;
  }, &a);
}

struct BatchArgs {
  const odc_field* const* f;
  int32_t nb;
  const double* lo;
  const double* hi;
  int64_t R;
  const odc_options* o;
  odc_stats* st;
};

int odc_extract_batch(odc_ctx* c, const odc_field* const* fields, int32_t nb, const double* lo, const double* hi,
                      int64_t R, const odc_options* o, odc_stats* stats) {
  if (!c || !fields || nb < 1 || !lo || !hi || !stats) return ODC_E_ARG;
  odc_options def;
  odc_default_options(&def);
  BatchArgs a{fields, nb, lo, hi, R, o ? o : &def, stats};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    BatchArgs* x = (BatchArgs*)p;
    const int nb = x->nb;
    cc->nb = 0;
    if ((int64_t)nb * (x->R + 1) * (x->R + 1) * (x->R + 1) >= (1ll << 32))
      throw OdcError{ODC_E_VALUE, "batch exceeds 2^32 grid vertices"};
    if (x->o->method != 0) throw OdcError{ODC_E_ARG, "batches run the dual-contouring method only"};
    if (x->o->normals != ODC_NORMALS_2D) throw OdcError{ODC_E_ARG, "batches use two-d-point normals"};
    std::vector<double> geo((size_t)nb * 6);
    std::vector<FieldP> fps(nb);
    for (int b = 0; b < nb; b++) {
      const odc_field* f = x->f[b];
      if (!f || f->kind != 0) throw OdcError{ODC_E_ARG, "batches take analytic fields"};
      if (f->continuous != x->f[0]->continuous)
        throw OdcError{ODC_E_ARG, "batch fields must all be binary or all continuous"};
      for (int a = 0; a < 3; a++) {
        if (!(x->hi[3 * b + a] > x->lo[3 * b + a])) throw OdcError{ODC_E_VALUE, "grid box must have positive extent"};
        geo[6 * b + a] = x->lo[3 * b + a];
        geo[6 * b + 3 + a] = (x->hi[3 * b + a] - x->lo[3 * b + a]) / (double)x->R;  // cell_size (grid.py:37-40)
      }
      FieldP fp = f->fp;
      fp.nodes = f->nodes;
      fp.n_nodes = f->n_nodes;
      fp.kind = f->kind;
      fp.iso = f->iso;
      fps[b] = fp;
    }
    // the geometry and field tables live in the context's field pool (not
    // the arena, which extract() resets)
    cudaStream_t s = cc->stream;
    double* dgeo = nullptr;
    FieldP* dfp = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&dgeo, sizeof(double) * geo.size(), s));
    CUDA_TRY(cudaMallocAsync((void**)&dfp, sizeof(FieldP) * nb, s));
    CUDA_TRY(cudaMemcpyAsync(dgeo, geo.data(), sizeof(double) * geo.size(), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(dfp, fps.data(), sizeof(FieldP) * nb, cudaMemcpyHostToDevice, s));
    BatchIn bin{nb, dgeo, dfp};
    try {
      extract(cc, x->f[0], x->lo, x->hi, x->R, x->o, x->st, Window{0, x->R, false}, &bin);
      batch_split(cc, x->o, make_opt(x->o, x->f[0]->continuous), x->st);
    } catch (...) {
      cudaFreeAsync(dgeo, s);
      cudaFreeAsync(dfp, s);
      cc->nb = 0;
      throw;
    }
    CUDA_TRY(cudaFreeAsync(dgeo, s));
    CUDA_TRY(cudaFreeAsync(dfp, s));
    return (int)ODC_OK;
  }, &a);
}

struct SlabArgs {
  const odc_field* f;
  const double* lo;
  const double* hi;
  int64_t R, z0, z1;
  const odc_options* o;
  odc_stats* st;
  odc_slab_info* info;
};

int odc_extract_slab(odc_ctx* c, const odc_field* f, const double lo[3], const double hi[3], int64_t R,
                     const odc_options* o, int64_t cell_z0, int64_t cell_z1, odc_stats* st, odc_slab_info* info) {
  if (!c || !f || !lo || !hi || !st || !info) return ODC_E_ARG;
  odc_options def;
  odc_default_options(&def);
  SlabArgs a{f, lo, hi, R, cell_z0, cell_z1, o ? o : &def, st, info};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    SlabArgs* x = (SlabArgs*)p;
    extract(cc, x->f, x->lo, x->hi, x->R, x->o, x->st, Window{x->z0, x->z1, true});
    odc_slab_info& I = *x->info;
    std::memset(&I, 0, sizeof I);
    I.n_halo_partitions = cc->P_halo;
    I.n_partitions = cc->P_own;
    I.n_window_partitions = cc->P;
    I.n_fans = cc->NF;
    I.n_triangles = cc->T;
    if (cc->K > 0) {
      I.partition_vertices = cc->slab_verts + 3 * cc->P_halo;
      I.fan_vertices = cc->slab_verts + 3 * cc->P;
      I.triangles = cc->slab_tris;
      I.partition_cell = cc->cells.part_cell + cc->P_halo;
      I.partition_index = cc->cells.part_index + cc->P_halo;
      I.fan_edge = cc->fan_edge;
    }
    return (int)ODC_OK;
  }, &a);
}

int odc_slab_globalize(odc_ctx* c, int64_t part_base, int64_t n_partitions_total, int64_t fan_base,
                       int32_t* triangles_out) {
  if (!c || !c->valid || !c->slab_mode) return ODC_E_ARG;
  if (c->T == 0) return ODC_OK;
  if (!triangles_out) return ODC_E_ARG;
  cudaSetDevice(c->device);
  launch_globalize_tris(c->slab_tris, c->T, c->P_halo, c->P, part_base, n_partitions_total, fan_base, triangles_out,
                        c->stream);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
    c->err = "slab globalize failed";
    return ODC_E_CUDA;
  }
  return ODC_OK;
}

struct FinishArgs {
  const double* v;
  int64_t V;
  const int32_t* t;
  int64_t T, P;
  const int64_t* kind;
  const int64_t* ref;
  int32_t repair;
  odc_stats* st;
};

// ---- distributed slab finish (odc_slabfin.cu, slab.py finish_distributed)
struct SeamArgs {
  int32_t* out;
  int64_t* n;
};
// the last slab's triangles with a halo corner (the previous rank's top
// cell layer), local ids; out == nullptr: count only
int odc_slab_seam(odc_ctx* c, int32_t* out, int64_t* n_out) {
  if (!c || !c->valid || !c->slab_mode || !n_out) return ODC_E_ARG;
  SeamArgs a{out, n_out};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    SeamArgs* x = (SeamArgs*)p;
    cudaStream_t s = cc->stream;
    const int64_t T = cc->T;
    *x->n = cc->seam_n;  // flagged and counted by odc_extract_slab
    if (x->out && *x->n) {
      launch_seam_take(cc->slab_tris, T, cc->seam_flag, cc->seam_rank, x->out, s);
      check_launch(cc);
      CUDA_TRY(cudaStreamSynchronize(s));
    }
    return (int)ODC_OK;
  }, &a);
}

struct LocalFinishArgs {
  const int32_t* seam;
  int64_t n_seam, n_halo_next;
  int64_t *n_used, *n_nondisc;
};

int odc_slab_local_finish(odc_ctx* c, const int32_t* seam, int64_t n_seam, int64_t n_halo_next, int64_t* n_used,
                          int64_t* n_nondisc) {
  if (!c || !c->valid || !c->slab_mode || !n_used || !n_nondisc || n_seam < 0 || (n_seam && !seam))
    return ODC_E_ARG;
  if (n_halo_next < 0 || n_halo_next > c->P_own) return ODC_E_ARG;
  LocalFinishArgs a{seam, n_seam, n_halo_next, n_used, n_nondisc};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    LocalFinishArgs* x = (LocalFinishArgs*)p;
    cudaStream_t s = cc->stream;
    const int64_t T = cc->T, Ts = x->n_seam, P = cc->P, Ph = cc->P_halo, Po = cc->P_own, V = cc->P + cc->NF;
    // this rank's triangles followed by the next rank's seam (mapped)
    int32_t* ext = need(cc->arena.get<int32_t>(3 * (T + Ts)));
    if (T) CUDA_TRY(cudaMemcpyAsync(ext, cc->slab_tris, sizeof(int32_t) * 3 * T, cudaMemcpyDeviceToDevice, s));
    launch_seam_map(x->seam, Ts, x->n_halo_next, P, V, ext + 3 * T, s);
    // incidence of every owned vertex (its whole fan is here), and from it
    // the used owned partitions and their compacted ids (polygonize.py:199-209)
    uint32_t* deg = need(cc->arena.get<uint32_t>(2 * (V + 1)));  // deg, then cursor: one memset
    uint32_t* cursor = deg + (V + 1);
    uint32_t* off = need(cc->arena.get<uint32_t>(V + 1));
    int32_t* inc = need(cc->arena.get<int32_t>(3 * (T + Ts)));
    unsigned long long* cnt = need(cc->arena.get<unsigned long long>(4));
    CUDA_TRY(cudaMemsetAsync(deg, 0, sizeof(uint32_t) * 2 * (V + 1), s));
    CUDA_TRY(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), s));
    launch_degree_range(ext, T + Ts, Ph, V, deg, s);
    cc->slab_used = need(cc->arena.get<uint8_t>(std::max<int64_t>(Po, 1)));
    uint32_t* u32 = need(cc->arena.get<uint32_t>(V + 1));
    cc->slab_newid = need(cc->arena.get<uint32_t>(V + 1));
    launch_used_from_degree(deg, Ph, Po, V + 1, cc->slab_used, u32, s);
    check_launch(cc, 2);
    scan2(cc, u32, deg, cc->slab_newid, off, V + 1, cnt);  // cnt[0] = used partitions
    // every owned vertex's fan: one closed disc?
    launch_fill_range(ext, T + Ts, Ph, V, off, cursor, inc, s);
    launch_count_nondisc(ext, off, inc, Ph, V, cnt + 2, s);
    check_launch(cc, 2);
    readback(cc, cnt, 3 * sizeof(unsigned long long));
    cc->slab_U = (int64_t)cc->h_pinned[0];
    *x->n_used = cc->slab_U;
    *x->n_nondisc = (int64_t)cc->h_pinned[2];
    return (int)ODC_OK;
  }, &a);
}

int odc_slab_top_ids(odc_ctx* c, int64_t part_base, int64_t n_top, int32_t* out) {
  if (!c || !c->valid || !c->slab_mode || c->slab_U < 0 || n_top < 0 || n_top > c->P_own || (n_top && !out))
    return ODC_E_ARG;
  cudaSetDevice(c->device);
  launch_slab_top_ids(c->P_own, n_top, c->slab_newid, part_base, out, c->stream);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
    c->err = "slab top ids failed";
    return ODC_E_CUDA;
  }
  return ODC_OK;
}

int odc_slab_final(odc_ctx* c, int64_t part_base, int64_t fan_base, const int32_t* halo_ids, int32_t* triangles_out,
                   double* part_vertices_out, int64_t* part_cell_out, int64_t* part_index_out) {
  if (!c || !c->valid || !c->slab_mode || c->slab_U < 0) return ODC_E_ARG;
  if ((c->P_halo && !halo_ids) || (c->T && !triangles_out) ||
      (c->slab_U && (!part_vertices_out || !part_cell_out || !part_index_out)))
    return ODC_E_ARG;
  cudaSetDevice(c->device);
  cudaStream_t s = c->stream;
  launch_slab_final_tris(c->slab_tris, c->T, c->P_halo, c->P, halo_ids, c->slab_newid, part_base, fan_base,
                         triangles_out, s);
  launch_slab_final_parts(c->P_own, c->slab_used, c->slab_newid, c->slab_verts + 3 * c->P_halo,
                          c->cells.part_cell + c->P_halo, c->cells.part_index + c->P_halo, part_vertices_out,
                          part_cell_out, part_index_out, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    c->err = "slab final failed";
    return ODC_E_CUDA;
  }
  return ODC_OK;
}

int odc_mesh_finish(odc_ctx* c, const double* vertices, int64_t V, const int32_t* triangles, int64_t T,
                    int64_t n_partitions, const int64_t* prov_kind, const int64_t* prov_ref, int32_t repair,
                    odc_stats* st) {
  if (!c || !st || V < n_partitions || (T && !triangles) || (V && !vertices)) return ODC_E_ARG;
  FinishArgs a{vertices, V, triangles, T, n_partitions, prov_kind, prov_ref, repair, st};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    FinishArgs* x = (FinishArgs*)p;
    cudaStream_t s = cc->stream;
    std::memset(x->st, 0, sizeof *x->st);
    for (int i = 0; i < ODC_N_CAT; i++) x->st->cat_order[i] = -1;
    cc->valid = false;
    cc->launches = 0;
    cc->arena.reset();
    cc->slab_mode = false;
    DevStats* dst = need(cc->arena.get<DevStats>(1));
    unsigned long long* totals = need(cc->arena.get<unsigned long long>(8));
    CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(DevStats), s));
    double* v = need(cc->arena.get<double>(3 * x->V));
    int32_t* t = need(cc->arena.get<int32_t>(3 * x->T));
    if (x->V) CUDA_TRY(cudaMemcpyAsync(v, x->v, sizeof(double) * 3 * x->V, cudaMemcpyDefault, s));
    if (x->T) CUDA_TRY(cudaMemcpyAsync(t, x->t, sizeof(int32_t) * 3 * x->T, cudaMemcpyDefault, s));
    cc->prov_kind_in = cc->prov_ref_in = nullptr;
    if (x->kind && x->ref && x->V) {
      cc->prov_kind_in = need(cc->arena.get<int64_t>(x->V));
      cc->prov_ref_in = need(cc->arena.get<int64_t>(2 * x->V));
      CUDA_TRY(cudaMemcpyAsync(cc->prov_kind_in, x->kind, 8 * x->V, cudaMemcpyDefault, s));
      CUDA_TRY(cudaMemcpyAsync(cc->prov_ref_in, x->ref, 16 * x->V, cudaMemcpyDefault, s));
    }
    uint8_t* used = need(cc->arena.get<uint8_t>(x->V));
    CUDA_TRY(cudaMemsetAsync(used, 0, (size_t)x->V, s));
    launch_mark_used(t, x->T, used, s);
    check_launch(cc);
    cc->T = x->T;
    cc->P = x->P;
    cc->K = 1;  // a mesh exists
    finish_mesh(cc, v, x->P, x->V - x->P, t, x->T, used, x->repair != 0, x->st, dst, totals);
    CUDA_TRY(cudaStreamSynchronize(s));
    cc->valid = true;
    return (int)ODC_OK;
  }, &a);
}

// Device arrays -> the caller's host buffers, pipelined: each segment is
// split into ~4 MB pieces, every piece is copied D2H into pinned staging at
// full link speed and recorded with an event, and host threads spread the
// pieces into the (pageable, first-touch) destinations as soon as their
// event completes -- the D2H of later pieces overlaps the host copies of
// earlier ones.
// One array of a copy-back: `bytes` on the device; widen = the device holds
// int32 that the host receives as int64 (triangles: half the PCIe bytes,
// widened by the copy threads on the way out of the staging buffer).
struct CopySeg {
  const void* dev;
  void* host;
  size_t bytes;
  bool widen = false;
};
bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Destinations in page-locked memory (the Python layer allocates the mesh
// arrays from torch's caching pinned allocator) are written by DMA directly:
// int32 triangles are widened on the device first.  Pageable destinations
// go through the staging pipeline below, whose host side is bound by page
// faults in fresh buffers (~9 GB/s per thread on the B200 hosts).
void copy_out_pipelined(odc_ctx* cc, const std::vector<CopySeg>& segs_in) {
  cudaStream_t s = cc->stream;
  std::vector<CopySeg> segs;
  bool direct = false;
  for (const CopySeg& g : segs_in) {
    if (!g.host || !g.bytes) continue;
    if (!host_pinned(g.host)) {
      segs.push_back(g);
      continue;
    }
    const void* src = g.dev;
    if (g.widen) {
      int64_t* w = need(cc->arena.get<int64_t>(g.bytes / 4));
      launch_widen_i32((const int32_t*)g.dev, w, (int64_t)(g.bytes / 4), s);
      src = w;
    }
    CUDA_TRY(cudaMemcpyAsync(g.host, src, g.widen ? 2 * g.bytes : g.bytes, cudaMemcpyDeviceToHost, s));
    direct = true;
  }
  if (direct && segs.empty()) {
    CUDA_TRY(cudaStreamSynchronize(s));
    return;
  }
  struct Piece {
    const void* dev;
    char* stage;
    char* dst;
    size_t n;
    bool widen;
  };
  const size_t chunk = 4u << 20;
  size_t total = 0;
  for (const CopySeg& g : segs)
    if (g.host && g.bytes) total += (g.bytes + 255) & ~(size_t)255;
  if (!total) return;
  if (total > cc->h_stage_bytes) {
    if (cc->h_stage) cudaFreeHost(cc->h_stage);
    cc->h_stage = nullptr;
    cc->h_stage_bytes = 0;
    const size_t want = total + total / 4;
    CUDA_TRY(cudaHostAlloc((void**)&cc->h_stage, want, cudaHostAllocDefault));
    cc->h_stage_bytes = want;
  }
  std::vector<Piece> pieces;
  size_t off = 0;
  for (const CopySeg& g : segs) {
    if (!g.host || !g.bytes) continue;
    for (size_t o = 0; o < g.bytes; o += chunk)
      pieces.push_back({(const char*)g.dev + o, cc->h_stage + off + o, (char*)g.host + (g.widen ? 2 * o : o),
                        std::min(chunk, g.bytes - o), g.widen});
    off += (g.bytes + 255) & ~(size_t)255;
  }
  while (cc->copy_evs.size() < pieces.size()) {
    cudaEvent_t e;
    // blocking sync: the copy threads sleep until their piece lands instead
    // of spinning (several contexts copy at once in batch mode)
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync));
    cc->copy_evs.push_back(e);
  }
  for (size_t i = 0; i < pieces.size(); i++) {
    CUDA_TRY(cudaMemcpyAsync(pieces[i].stage, pieces[i].dev, pieces[i].n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaEventRecord(cc->copy_evs[i], s));
  }
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  // the host side is first-touch page faults into fresh numpy buffers (the
  // kernel zero-fills ~10 GB/s per thread): as many threads as cores
  const size_t nthr = std::min<size_t>({(size_t)32, (size_t)hw, pieces.size()});
  std::atomic<int> bad{0};
  auto work = [&](size_t t) {
    for (size_t i = t; i < pieces.size(); i += nthr) {
      if (cudaEventSynchronize(cc->copy_evs[i]) != cudaSuccess) {
        bad = 1;
        return;
      }
      if (pieces[i].widen) {
        const int32_t* a = (const int32_t*)pieces[i].stage;
        int64_t* b = (int64_t*)pieces[i].dst;
        const size_t m = pieces[i].n / 4;
        for (size_t j = 0; j < m; j++) b[j] = a[j];
      } else {
        std::memcpy(pieces[i].dst, pieces[i].stage, pieces[i].n);
      }
    }
  };
  if (nthr <= 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (size_t t = 1; t < nthr; t++) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
  }
  if (bad) throw OdcError{ODC_E_CUDA, "mesh copy failed"};
}

struct CopyMeshArgs {
  int32_t which;
  double* v;
  int64_t* t;
  int64_t* kind;
  int64_t* ref;
  int64_t* raw_t;  // odc_copy_mesh_pair: the pre-repair triangles too
};

// Everything is produced in its final host type on the device (triangles
// widened to int64, duplicate provenance filled in) and copied out with
// copy_out_pipelined.
int copy_mesh_impl(odc_ctx* c, CopyMeshArgs* a) {
  if (!c) return ODC_E_ARG;
  if (!c->valid) {
    c->err = "no extraction result";
    return ODC_E_ARG;
  }
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    CopyMeshArgs* x = (CopyMeshArgs*)p;
    const bool raw = x->which == 1;
    const int64_t V = raw ? cc->V0 : cc->V1, T = cc->T;
    const double* dv = raw ? cc->verts0 : cc->verts1;
    const int32_t* dt = raw ? cc->tris0 : cc->tris1;
    cudaStream_t s = cc->stream;
    std::vector<CopySeg> segs;
    segs.push_back({dv, x->v, sizeof(double) * 3 * V});
    if (x->t && T) segs.push_back({dt, x->t, sizeof(int32_t) * 3 * T, true});
    if ((x->kind || x->ref) && V) {
      int64_t* dk = need(cc->arena.get<int64_t>(V));
      int64_t* dr = need(cc->arena.get<int64_t>(2 * V));
      const int64_t V0 = cc->V0;
      if (cc->prov_kind_in)
        launch_gather_provenance(V0, cc->src0, cc->prov_kind_in, cc->prov_ref_in, dk, dr, s);
      else
        launch_provenance(V0, cc->P, cc->src0, cc->cells.part_cell, cc->cells.part_index, cc->fan_edge, dk, dr, s);
      launch_dup_provenance(V0, V, dk, dr, s);
      segs.push_back({dk, x->kind, sizeof(int64_t) * V});
      segs.push_back({dr, x->ref, sizeof(int64_t) * 2 * V});
    }
    if (x->raw_t && T)  // pre-repair triangles (same count, corners not renamed)
      segs.push_back({cc->tris0, x->raw_t, sizeof(int32_t) * 3 * T, true});
    CUDA_TRY(cudaGetLastError());
    copy_out_pipelined(cc, segs);
    return (int)ODC_OK;
  }, a);
}

int odc_copy_mesh(odc_ctx* c, int32_t which, double* vertices, int64_t* triangles, int64_t* prov_kind,
                  int64_t* prov_ref) {
  CopyMeshArgs a{which, vertices, triangles, prov_kind, prov_ref, nullptr};
  return copy_mesh_impl(c, &a);
}

int odc_copy_mesh_pair(odc_ctx* c, double* vertices, int64_t* triangles, int64_t* prov_kind, int64_t* prov_ref,
                       int64_t* raw_triangles) {
  CopyMeshArgs a{0, vertices, triangles, prov_kind, prov_ref, raw_triangles};
  return copy_mesh_impl(c, &a);
}

struct BatchCopyArgs {
  double* v;
  int64_t* t;
  int64_t* raw_t;
  int64_t* kind;
  int64_t* ref;
};

int odc_copy_batch_meshes(odc_ctx* c, double* vertices, int64_t* triangles, int64_t* raw_triangles,
                          int64_t* prov_kind, int64_t* prov_ref) {
  if (!c) return ODC_E_ARG;
  if (!c->valid || !c->nb) {
    c->err = "no batch extraction result";
    return ODC_E_ARG;
  }
  BatchCopyArgs a{vertices, triangles, raw_triangles, prov_kind, prov_ref};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    BatchCopyArgs* x = (BatchCopyArgs*)p;
    const int64_t V = cc->V1, V0 = cc->V0, T = cc->T;
    if (!cc->K || !V) return (int)ODC_OK;
    cudaStream_t s = cc->stream;
    std::vector<CopySeg> segs;
    int64_t *dk = nullptr, *dr = nullptr, *ok = nullptr, *orf = nullptr;
    if (x->kind || x->ref) {  // union provenance, then gathered shape by shape
      dk = need(cc->arena.get<int64_t>(V));
      dr = need(cc->arena.get<int64_t>(2 * V));
      launch_provenance(V0, cc->P, cc->src0, cc->cells.part_cell, cc->cells.part_index, cc->fan_edge, dk, dr, s);
      launch_dup_provenance(V0, V, dk, dr, s);
      ok = need(cc->arena.get<int64_t>(V));
      orf = need(cc->arena.get<int64_t>(2 * V));
    }
    double* ov = need(cc->arena.get<double>(3 * V));
    const GridP& g = cc->g;
    launch_batch_gather(cc->verts1, cc->b_perm, cc->b_skeys, V, dk, dr, g.S * g.R * g.R, 3 * g.S3, ov, ok, orf, s);
    segs.push_back({ov, x->v, sizeof(double) * 3 * V});
    if (ok) {
      segs.push_back({ok, x->kind, sizeof(int64_t) * V});
      segs.push_back({orf, x->ref, sizeof(int64_t) * 2 * V});
    }
    if (x->t && T) {
      int32_t* t32 = need(cc->arena.get<int32_t>(3 * T));
      launch_batch_tris(cc->tris1, T, cc->b_local, t32, s);
      segs.push_back({t32, x->t, sizeof(int32_t) * 3 * T, true});
    }
    if (x->raw_t && T && V != V0) {  // pre-repair triangles: only shapes the repair changed
      int32_t* r32 = need(cc->arena.get<int32_t>(3 * T));
      launch_batch_tris(cc->tris0, T, cc->b_local, r32, s);
      for (int b = 0; b < cc->nb; b++) {
        const int64_t t0 = cc->b_bounds[(size_t)b * kBatchCols + 5], t1 = cc->b_bounds[(size_t)(b + 1) * kBatchCols + 5];
        if (cc->b_vstart[b + 1] - cc->b_vstart[b] != cc->b_v0[b] && t1 > t0)
          segs.push_back({r32 + 3 * t0, x->raw_t + 3 * t0, sizeof(int32_t) * 3 * (t1 - t0), true});
      }
    }
    CUDA_TRY(cudaGetLastError());
    copy_out_pipelined(cc, segs);
    return (int)ODC_OK;
  }, &a);
}

int odc_batch_layout(odc_ctx* c, int64_t* vertex_start, int64_t* raw_vertices, int64_t* triangle_start) {
  if (!c || !vertex_start || !raw_vertices || !triangle_start) return ODC_E_ARG;
  if (!c->valid || !c->nb) {
    c->err = "no batch extraction result";
    return ODC_E_ARG;
  }
  for (int b = 0; b <= c->nb; b++) {
    vertex_start[b] = c->b_vstart.empty() ? 0 : c->b_vstart[b];
    triangle_start[b] = c->b_bounds[(size_t)b * kBatchCols + 5];
    if (b < c->nb) raw_vertices[b] = c->b_v0[b];
  }
  return ODC_OK;
}


struct ValidateArgs {
  const int64_t* tris;
  int64_t T, V;
  odc_manifold_report* out;
};

int odc_validate_manifold(odc_ctx* c, const int64_t* triangles, int64_t n_triangles, int64_t n_vertices,
                          odc_manifold_report* out) {
  if (!c || !out || n_triangles < 0 || n_vertices < 0 || (n_triangles && !triangles)) return ODC_E_ARG;
  if (n_vertices >= INT32_MAX || 3 * n_triangles >= INT32_MAX) {
    c->err = "validate_manifold: mesh too large for 32-bit fans";
    return ODC_E_ARG;
  }
  ValidateArgs a{triangles, n_triangles, n_vertices, out};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    ValidateArgs* x = (ValidateArgs*)p;
    std::memset(x->out, 0, sizeof *x->out);
    cc->v_edges.clear();
    cc->v_pinched.clear();
    cc->v_isolated.clear();
    if (x->T == 0) {  // mesh.py:97-98: an empty mesh is reported manifold, nothing else
      x->out->manifold = 1;
      return (int)ODC_OK;
    }
    Arena& A = cc->varena;
    A.reset();
    cudaStream_t s = cc->stream;
    const int64_t T = x->T, V = x->V, n3 = 3 * T;
    int64_t* t64 = need(A.get<int64_t>(n3));
    int32_t* t = need(A.get<int32_t>(n3));
    uint32_t* bad = need(A.get<uint32_t>(2));
    unsigned long long* totals = need(A.get<unsigned long long>(8));
    CUDA_TRY(cudaMemcpyAsync(t64, x->tris, 8 * n3, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(bad, 0, 8, s));
    launch_narrow_tris(t64, n3, t, V, bad, s);
    check_launch(cc);
    readback(cc, bad, 4);
    if (((uint32_t*)cc->h_pinned)[0]) throw OdcError{ODC_E_VALUE, "triangle index out of range"};
    uint32_t* deg = need(A.get<uint32_t>(V + 1));
    uint32_t* off = need(A.get<uint32_t>(V + 1));
    uint32_t* cursor = need(A.get<uint32_t>(V));
    int32_t* inc = need(A.get<int32_t>(n3));
    CUDA_TRY(cudaMemsetAsync(deg, 0, 4 * (V + 1), s));
    CUDA_TRY(cudaMemsetAsync(cursor, 0, 4 * V, s));
    launch_vertex_degree(t, T, deg, s);
    check_launch(cc);
    auto scan = [&](const uint32_t* in, uint32_t* o, int64_t n, unsigned long long* tot) {
      const uint32_t* ins[1] = {in};
      uint32_t* outs[1] = {o};
      uint32_t* tiles = need(A.get<uint32_t>((n + 255) / 256 + 1));
      check_launch(cc, launch_scan_u32(ins, outs, 1, n, tiles, tot, s));
    };
    scan(deg, off, V + 1, totals + 0);
    launch_vertex_fill(t, T, off, cursor, inc, s);
    check_launch(cc);
    int32_t* nbv = need(A.get<int32_t>(2 * n3));
    uint32_t* nbc = need(A.get<uint32_t>(2 * n3));
    uint32_t* nbt = need(A.get<uint32_t>(2 * n3));
    uint32_t* uf = need(A.get<uint32_t>(n3));
    uint32_t* per[5];
    for (auto& q : per) q = need(A.get<uint32_t>(V + 1));
    uint32_t *n_nb = per[0], *n_nm = per[1], *n_bd = per[2], *pin = per[3], *iso = per[4];
    launch_manifold_vertex(V, t, off, inc, nbv, nbc, nbt, uf, n_nb, n_nm, n_bd, pin, iso, s);
    check_launch(cc);
    uint32_t* nm_off = need(A.get<uint32_t>(V + 1));
    uint32_t* bd_off = need(A.get<uint32_t>(V + 1));
    uint32_t* pin_off = need(A.get<uint32_t>(V + 1));
    uint32_t* iso_off = need(A.get<uint32_t>(V + 1));
    scan(n_nm, nm_off, V, totals + 1);
    scan(n_bd, bd_off, V, totals + 2);
    scan(pin, pin_off, V, totals + 3);
    scan(iso, iso_off, V, totals + 4);
    readback(cc, totals + 1, 4 * sizeof(unsigned long long));
    const int64_t n_nm_t = (int64_t)cc->h_pinned[0], n_bd_t = (int64_t)cc->h_pinned[1],
                  n_pin_t = (int64_t)cc->h_pinned[2], n_iso_t = (int64_t)cc->h_pinned[3];
    int64_t* e_out = need(A.get<int64_t>(2 * n_nm_t + 1));
    int64_t* p_out = need(A.get<int64_t>(n_pin_t + 1));
    int64_t* i_out = need(A.get<int64_t>(n_iso_t + 1));
    launch_manifold_emit(V, off, nbv, nbc, n_nb, n_nm, nm_off, e_out, s);
    launch_emit_flagged(V, pin, pin_off, p_out, s);
    launch_emit_flagged(V, iso, iso_off, i_out, s);
    check_launch(cc, 3);
    cc->v_edges.resize(2 * n_nm_t);
    cc->v_pinched.resize(n_pin_t);
    cc->v_isolated.resize(n_iso_t);
    if (n_nm_t) CUDA_TRY(cudaMemcpyAsync(cc->v_edges.data(), e_out, 16 * n_nm_t, cudaMemcpyDeviceToHost, s));
    if (n_pin_t) CUDA_TRY(cudaMemcpyAsync(cc->v_pinched.data(), p_out, 8 * n_pin_t, cudaMemcpyDeviceToHost, s));
    if (n_iso_t) CUDA_TRY(cudaMemcpyAsync(cc->v_isolated.data(), i_out, 8 * n_iso_t, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    x->out->manifold = n_nm_t == 0 && n_pin_t == 0;
    x->out->n_nonmanifold_edges = n_nm_t;
    x->out->n_pinched_vertices = n_pin_t;
    x->out->n_boundary_edges = n_bd_t;
    x->out->n_isolated_vertices = n_iso_t;
    return (int)ODC_OK;
  }, &a);
}

int odc_validate_copy(odc_ctx* c, int64_t* nonmanifold_edges, int64_t* pinched_vertices, int64_t* isolated_vertices) {
  if (!c) return ODC_E_ARG;
  if (nonmanifold_edges && !c->v_edges.empty())
    std::memcpy(nonmanifold_edges, c->v_edges.data(), 8 * c->v_edges.size());
  if (pinched_vertices && !c->v_pinched.empty())
    std::memcpy(pinched_vertices, c->v_pinched.data(), 8 * c->v_pinched.size());
  if (isolated_vertices && !c->v_isolated.empty())
    std::memcpy(isolated_vertices, c->v_isolated.data(), 8 * c->v_isolated.size());
  return ODC_OK;
}

struct SelfxArgs {
  const double* v;
  int64_t nv;
  const int64_t* t;
  int64_t nt;
  double tol;
  int64_t* count;
};

int odc_count_self_intersections(odc_ctx* c, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                                 int64_t n_triangles, double tolerance, int64_t* count) {
  if (!c || !count || n_vertices < 0 || n_triangles < 0 || (n_vertices && !vertices) || (n_triangles && !triangles))
    return ODC_E_ARG;
  if (n_vertices >= INT32_MAX || n_triangles >= INT32_MAX / 8) {
    c->err = "count_self_intersections: mesh too large";
    return ODC_E_ARG;
  }
  SelfxArgs a{vertices, n_vertices, triangles, n_triangles, tolerance, count};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    SelfxArgs* x = (SelfxArgs*)p;
    *x->count = 0;
    cc->v_si_pairs.clear();
    if (x->nt < 2) return (int)ODC_OK;  // mesh.py:423-424
    Arena& A = cc->varena;
    cudaStream_t s = cc->stream;
    const int64_t n3 = 3 * x->nt;
    double* dv = nullptr;
    int32_t* t = nullptr;
    auto upload = [&]() {
      A.reset();
      dv = need(A.get<double>(3 * x->nv));
      int64_t* t64 = need(A.get<int64_t>(n3));
      t = need(A.get<int32_t>(n3));
      uint32_t* bad = need(A.get<uint32_t>(2));
      CUDA_TRY(cudaMemcpyAsync(dv, x->v, 24 * x->nv, cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(t64, x->t, 8 * n3, cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaMemsetAsync(bad, 0, 8, s));
      launch_narrow_tris(t64, n3, t, x->nv, bad, s);
      check_launch(cc);
      readback(cc, bad, 4);
      if (((uint32_t*)cc->h_pinned)[0]) throw OdcError{ODC_E_VALUE, "triangle index out of range"};
    };
    auto alloc = [](void* ar, size_t n) -> void* { return ((Arena*)ar)->alloc(n); };
    int64_t cap = 1 << 20, n_hits = 0;
    for (;;) {
      upload();
      int64_t* hits = need(A.get<int64_t>(cap));
      const int rc = self_intersections(dv, x->nv, t, x->nt, x->tol, alloc, &A, s, hits, cap, &n_hits);
      if (rc != ODC_OK) throw OdcError{rc, "count_self_intersections failed"};
      if (n_hits > cap) {  // rerun with room for every hit
        cap = n_hits;
        continue;
      }
      cc->v_si_pairs.resize(2 * n_hits);
      std::vector<int64_t> keys(n_hits);
      if (n_hits) CUDA_TRY(cudaMemcpyAsync(keys.data(), hits, 8 * n_hits, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      for (int64_t i = 0; i < n_hits; i++) {
        cc->v_si_pairs[2 * i] = keys[i] / x->nt;
        cc->v_si_pairs[2 * i + 1] = keys[i] % x->nt;
      }
      break;
    }
    *x->count = n_hits;
    return (int)ODC_OK;
  }, &a);
}

struct DistArgs {
  const double* v;
  int64_t nv;
  const int64_t* t;
  int64_t nt;
  const double* q;
  int64_t nq;
  double* dist;
  int64_t* tri;
  double* cp;
};

int odc_mesh_distance(odc_ctx* c, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                      int64_t n_triangles, const double* points, int64_t n_points, double* dist, int64_t* tri,
                      double* closest) {
  if (!c || n_vertices < 0 || n_triangles < 0 || n_points < 0 || (n_points && (!points || !dist))) return ODC_E_ARG;
  if (n_triangles == 0 || !vertices || !triangles) {
    c->err = "distance index needs a non-empty mesh";
    return ODC_E_VALUE;
  }
  if (n_vertices >= INT32_MAX || 3 * n_triangles >= INT32_MAX) {
    c->err = "mesh_distance: mesh too large";
    return ODC_E_ARG;
  }
  DistArgs a{vertices, n_vertices, triangles, n_triangles, points, n_points, dist, tri, closest};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    DistArgs* x = (DistArgs*)p;
    if (x->nq == 0) return (int)ODC_OK;
    Arena& A = cc->varena;
    A.reset();
    cudaStream_t s = cc->stream;
    const int64_t n3 = 3 * x->nt;
    double* dv = need(A.get<double>(3 * x->nv));
    int64_t* t64 = need(A.get<int64_t>(n3));
    int32_t* t = need(A.get<int32_t>(n3));
    uint32_t* bad = need(A.get<uint32_t>(2));
    double* dq = need(A.get<double>(3 * x->nq));
    double* dd = need(A.get<double>(x->nq));
    int64_t* dt = need(A.get<int64_t>(x->nq));
    double* dc = need(A.get<double>(3 * x->nq));
    CUDA_TRY(cudaMemcpyAsync(dv, x->v, 24 * x->nv, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(t64, x->t, 8 * n3, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(dq, x->q, 24 * x->nq, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(bad, 0, 8, s));
    launch_narrow_tris(t64, n3, t, x->nv, bad, s);
    check_launch(cc);
    readback(cc, bad, 4);
    if (((uint32_t*)cc->h_pinned)[0]) throw OdcError{ODC_E_VALUE, "triangle index out of range"};
    auto alloc = [](void* ar, size_t n) -> void* { return ((Arena*)ar)->alloc(n); };
    const int rc = mesh_distance(dv, t, x->nt, dq, x->nq, alloc, &A, s, dd, dt, dc);
    if (rc != ODC_OK) throw OdcError{rc, "mesh_distance failed"};
    cc->launches += 5;
    CUDA_TRY(cudaMemcpyAsync(x->dist, dd, 8 * x->nq, cudaMemcpyDeviceToHost, s));
    if (x->tri) CUDA_TRY(cudaMemcpyAsync(x->tri, dt, 8 * x->nq, cudaMemcpyDeviceToHost, s));
    if (x->cp) CUDA_TRY(cudaMemcpyAsync(x->cp, dc, 24 * x->nq, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return (int)ODC_OK;
  }, &a);
}

int odc_triangle_areas(odc_ctx* c, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                       int64_t n_triangles, double* areas) {
  if (!c || n_vertices < 0 || n_triangles < 0 || (n_triangles && (!triangles || !areas || !vertices)))
    return ODC_E_ARG;
  if (n_vertices >= INT32_MAX || 3 * n_triangles >= INT32_MAX) return ODC_E_ARG;
  DistArgs a{vertices, n_vertices, triangles, n_triangles, nullptr, 0, areas, nullptr, nullptr};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    DistArgs* x = (DistArgs*)p;
    if (x->nt == 0) return (int)ODC_OK;
    Arena& A = cc->varena;
    A.reset();
    cudaStream_t s = cc->stream;
    const int64_t n3 = 3 * x->nt;
    double* dv = need(A.get<double>(3 * x->nv));
    int64_t* t64 = need(A.get<int64_t>(n3));
    int32_t* t = need(A.get<int32_t>(n3));
    uint32_t* bad = need(A.get<uint32_t>(2));
    double* da = need(A.get<double>(x->nt));
    CUDA_TRY(cudaMemcpyAsync(dv, x->v, 24 * x->nv, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(t64, x->t, 8 * n3, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(bad, 0, 8, s));
    launch_narrow_tris(t64, n3, t, x->nv, bad, s);
    launch_tri_areas(dv, t, x->nt, da, s);
    check_launch(cc, 2);
    readback(cc, bad, 4);
    if (((uint32_t*)cc->h_pinned)[0]) throw OdcError{ODC_E_VALUE, "triangle index out of range"};
    CUDA_TRY(cudaMemcpyAsync(x->dist, da, 8 * x->nt, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return (int)ODC_OK;
  }, &a);
}

int odc_self_intersection_pairs(odc_ctx* c, int64_t* pairs) {
  if (!c) return ODC_E_ARG;
  if (pairs && !c->v_si_pairs.empty()) std::memcpy(pairs, c->v_si_pairs.data(), 8 * c->v_si_pairs.size());
  return ODC_OK;
}

int odc_mesh_device(odc_ctx* c, int32_t which, const double** v, const int32_t** t, int64_t* nv, int64_t* nt) {
  if (!c || !c->valid) return ODC_E_ARG;
  const bool raw = which == 1;
  if (v) *v = raw ? c->verts0 : c->verts1;
  if (t) *t = raw ? c->tris0 : c->tris1;
  if (nv) *nv = raw ? c->V0 : c->V1;
  if (nt) *nt = c->T;
  return ODC_OK;
}

struct CopyArrArgs {
  int32_t which;
  void* dst;
  int64_t bytes;
  int64_t* n;
};

int odc_copy_array(odc_ctx* c, int32_t which, void* dst, int64_t dst_bytes, int64_t* n_elems) {
  if (!c || !n_elems) return ODC_E_ARG;
  if (!c->valid) {
    c->err = "no extraction result";
    return ODC_E_ARG;
  }
  CopyArrArgs a{which, dst, dst_bytes, n_elems};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    CopyArrArgs* x = (CopyArrArgs*)p;
    const void* src = nullptr;
    int64_t n = 0, esize = 8;
    const bool has1d = cc->K > 0;
    std::vector<uint8_t> unpack;
    switch (x->which) {
      case ODC_ARR_LABELS: {
        n = cc->g.S3;
        esize = 1;
        if (x->dst) {
          uint8_t* b = need(cc->arena.get<uint8_t>(n));
          launch_unpack_labels(cc->g, cc->L, b, cc->stream);
          src = b;
        }
        break;
      }
      case ODC_ARR_EDGE_KEY: src = cc->edge_key; n = cc->K; break;
      case ODC_ARR_V_IN: src = cc->v_in; n = cc->v_in ? cc->K : 0; break;
      case ODC_ARR_FACE_KEY: src = cc->face_key; n = cc->face_key ? cc->F : 0; break;
      case ODC_ARR_FACE_NCROSS: src = cc->face_nc; n = cc->face_nc ? cc->F : 0; break;
      case ODC_ARR_CELLS: src = cc->cell_id; n = cc->C; break;
      case ODC_ARR_INSTANCE_EDGES: src = cc->inst_edges; n = (cc->inst_edges && has1d) ? 2 * cc->Q : 0; break;
      case ODC_ARR_T1D: src = cc->t1d; n = has1d ? cc->K : 0; break;
      case ODC_ARR_POS1D: src = cc->pos1d; n = has1d ? 3 * cc->K : 0; break;
      case ODC_ARR_POS2: src = cc->s2.pos2; n = (cc->s2.pos2 && has1d) ? 2 * cc->Q : 0; break;
      case ODC_ARR_POS3: src = cc->s2.pos3; n = (cc->s2.pos3 && has1d) ? 3 * cc->Q : 0; break;
      case ODC_ARR_STATUS: src = cc->s2.status; n = (cc->s2.status && has1d) ? cc->Q : 0; esize = 1; break;
      case ODC_ARR_MID_LABEL: src = cc->s2.mid; n = (cc->s2.mid && has1d) ? cc->Q : 0; esize = 1; break;
      case ODC_ARR_PART_CELL: src = cc->cells.part_cell; n = has1d ? cc->P : 0; break;
      case ODC_ARR_PART_INDEX: src = cc->cells.part_index; n = has1d ? cc->P : 0; break;
      case ODC_ARR_CYC_EDGES: src = cc->cells.cyc_edges; n = (cc->cells.cyc_edges && has1d) ? cc->Ns : 0; break;
      case ODC_ARR_CYC_INSTS: src = cc->cells.cyc_insts; n = (cc->cells.cyc_insts && has1d) ? cc->Ns : 0; break;
      case ODC_ARR_NORMALS: src = cc->cells.normals; n = (cc->cells.normals && has1d) ? 3 * cc->Ns : 0; break;
      case ODC_ARR_QEF_POS: src = cc->cells.verts; n = has1d ? 3 * cc->P : 0; break;
      case ODC_ARR_QEF_RANK: src = cc->cells.rank; n = (cc->cells.rank && has1d) ? cc->P : 0; break;
      case ODC_ARR_QEF_RESID: src = cc->cells.resid; n = (cc->cells.resid && has1d) ? cc->P : 0; break;
      case ODC_ARR_SPLIT_CASES: src = cc->split_cases; n = (cc->split_cases && has1d) ? cc->n_interior : 0; break;
      case ODC_ARR_DUP_SOURCE: {
        // original (raw-mesh) vertex of every repair duplicate, resolved across passes
        n = cc->V1 - cc->V0;
        if (x->dst && n) {
          if (x->bytes < 8 * n) throw OdcError{ODC_E_ARG, "destination too small"};
          int64_t* out = (int64_t*)x->dst;
          for (const auto& dp : cc->dup_passes) {
            std::vector<int64_t> s(dp.n);
            CUDA_TRY(cudaMemcpyAsync(s.data(), dp.src, 8 * dp.n, cudaMemcpyDeviceToHost, cc->stream));
            CUDA_TRY(cudaStreamSynchronize(cc->stream));
            for (int64_t i = 0; i < dp.n; i++) {
              int64_t v = s[i];
              out[dp.base - cc->V0 + i] = v >= cc->V0 ? out[v - cc->V0] : v;
            }
          }
        }
        *x->n = n;
        return (int)ODC_OK;
      }
      case ODC_ARR_CYC_LEN: src = cc->cells.cyc_len; n = (cc->cells.cyc_len && has1d) ? cc->P : 0; break;
      default: throw OdcError{ODC_E_ARG, "unknown array id"};
    }
    *x->n = n;
    if (x->dst && n) {
      if (!src) throw OdcError{ODC_E_ARG, "array not kept (set keep_intermediates)"};
      if (x->bytes < esize * n) throw OdcError{ODC_E_ARG, "destination too small"};
      CUDA_TRY(cudaMemcpyAsync(x->dst, src, (size_t)(esize * n), cudaMemcpyDeviceToHost, cc->stream));
      CUDA_TRY(cudaStreamSynchronize(cc->stream));
    }
    return (int)ODC_OK;
  }, &a);
}

struct EvalArgs {
  const odc_field* f;
  const double* pts;
  int64_t n;
  double* raw;
  uint8_t* lab;
};

static int eval_common(odc_ctx* c, const odc_field* f, const double* pts, int64_t n, double* raw, uint8_t* lab) {
  if (!c || !f || (!pts && n)) return ODC_E_ARG;
  EvalArgs a{f, pts, n, raw, lab};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    EvalArgs* x = (EvalArgs*)p;
    if (x->n == 0) return (int)ODC_OK;
    // eval_labels rejects non-finite points (fields.py:42-45)
    for (int64_t i = 0; i < 3 * x->n; i++)
      if (!std::isfinite(x->pts[i])) throw OdcError{ODC_E_VALUE, "non-finite query point at index " + std::to_string(i / 3)};
    cc->valid = false;  // the evaluation reuses the workspace
    cc->arena.reset();
    double* dp = need(cc->arena.get<double>(3 * x->n));
    double* dr = x->raw ? need(cc->arena.get<double>(x->n)) : nullptr;
    uint8_t* dl = need(cc->arena.get<uint8_t>(x->n));
    CUDA_TRY(cudaMemcpyAsync(dp, x->pts, sizeof(double) * 3 * x->n, cudaMemcpyHostToDevice, cc->stream));
    eval_points(cc, x->f, dp, x->n, dl, dr);
    check_surface(cc);
    if (x->raw) CUDA_TRY(cudaMemcpyAsync(x->raw, dr, sizeof(double) * x->n, cudaMemcpyDeviceToHost, cc->stream));
    if (x->lab) CUDA_TRY(cudaMemcpyAsync(x->lab, dl, x->n, cudaMemcpyDeviceToHost, cc->stream));
    CUDA_TRY(cudaStreamSynchronize(cc->stream));
    return (int)ODC_OK;
  }, &a);
}

int odc_profile_mlp(odc_ctx* c, const odc_field* f, int64_t n, int64_t* trace, int64_t trace_len) {
  if (!c || !f || f->kind != 1 || !trace || trace_len < 256) return ODC_E_ARG;
  cudaSetDevice(c->device);
  c->valid = false;
  c->arena.reset();
  // the kernels' trace slots reach index ~1,200: the device buffer is at
  // least 2,048 entries whatever the caller reads back
  unsigned long long* dt = c->arena.get<unsigned long long>(trace_len > 2048 ? trace_len : 2048);
  uint8_t* lab = c->arena.get<uint8_t>(n);
  if (!dt || !lab) return ODC_E_NOMEM;
  cudaMemsetAsync(dt, 0, 8 * (trace_len > 2048 ? trace_len : 2048), c->stream);
  GridP g{};
  const int64_t S = 1 + (int64_t)std::ceil(std::cbrt((double)n));
  g.R = S - 1;
  g.S = S;
  g.S2 = S * S;
  g.S3 = S * S * S;
  g.W = (S + 31) / 32;
  g.z0 = 0;
  g.nz = S;
  for (int a = 0; a < 3; a++) {
    g.lo[a] = 0.0;
    g.h[a] = 1.0 / (double)g.R;
  }
  MlpDev md = f->mlp;
  md.debug = c->mlp_debug & 63;
  md.trace = (c->mlp_debug & 64) ? nullptr : dt;  // 64: time the kernel without the trace hooks
  const int64_t np = n < g.S3 ? n : g.S3;
  PointSrc src{nullptr, g, 0};
  if (c->mlp_debug & 128) {  // 128: explicit points (the search batches' path): the grid's, or the caller's
    double* pts = c->arena.get<double>(3 * np);
    if (!pts) return ODC_E_NOMEM;
    if (c->profile_pts) cudaMemcpyAsync(pts, c->profile_pts, 24 * np, cudaMemcpyHostToDevice, c->stream);
    else launch_grid_points(g, 0, np, pts, c->stream);
    src.pts = pts;
  }
  cudaEventRecord(c->ev0, c->stream);
  try {
    run_mlp(c, f, src, np, lab, nullptr, c->stream, &md);
  } catch (const OdcError& e) {
    c->err = e.msg;
    return e.code;
  }
  cudaEventRecord(c->ev1, c->stream);
  if (cudaMemcpyAsync(trace, dt, 8 * trace_len, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess) {
    c->err = "profile run failed";
    return ODC_E_CUDA;
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  trace[trace_len - 1] = (int64_t)(ms * 1e6f);  // kernel time, ns
  return ODC_OK;
}

int odc_eval_raw(odc_ctx* c, const odc_field* f, const double* pts, int64_t n, double* raw) {
  return eval_common(c, f, pts, n, raw, nullptr);
}
int odc_eval_labels(odc_ctx* c, const odc_field* f, const double* pts, int64_t n, uint8_t* labels) {
  return eval_common(c, f, pts, n, nullptr, labels);
}

int odc_surface_probe(odc_ctx* c, const odc_field* f, const double lo[3], const double hi[3], int64_t R,
                      int64_t box, int64_t* counts) {
  if (!c || !f || !lo || !hi || !counts || R < 1 || box < 1) return ODC_E_ARG;
  if (f->kind != 0) {
    c->err = "surface probe: only analytic fields have an interval bound";
    return ODC_E_ARG;
  }
  struct A {
    const odc_field* f;
    const double *lo, *hi;
    int64_t R, box;
    int64_t* counts;
  } a{f, lo, hi, R, box, counts};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    A* x = (A*)p;
    GridP g{};
    g.R = x->R;
    g.S = x->R + 1;
    for (int k = 0; k < 3; k++) {
      g.lo[k] = x->lo[k];
      g.h[k] = (x->hi[k] - x->lo[k]) / (double)x->R;
    }
    FieldP fp = x->f->fp;
    fp.nodes = x->f->nodes;
    fp.n_nodes = x->f->n_nodes;
    fp.iso = x->f->iso;
    const int64_t nbz = (x->R + x->box - 1) / x->box;
    // stream-ordered scratch: the last extraction's workspace stays valid
    unsigned long long* d = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&d, sizeof(unsigned long long) * nbz, cc->stream));
    CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * nbz, cc->stream));
    launch_surface_probe(g, fp, x->box, d, cc->stream);
    const cudaError_t e = cudaPeekAtLastError();
    cudaMemcpyAsync(x->counts, d, sizeof(int64_t) * nbz, cudaMemcpyDeviceToHost, cc->stream);
    cudaFreeAsync(d, cc->stream);
    CUDA_TRY(e);
    CUDA_TRY(cudaStreamSynchronize(cc->stream));
    return (int)ODC_OK;
  }, &a);
}

struct DotArgs {
  const odc_field* f;
  const double* pts;
  int64_t n;
  float* dot;
};
int odc_eval_mlp_dot(odc_ctx* c, const odc_field* f, const double* pts, int64_t n, float* dot) {
  if (!c || !f || f->kind != 1 || n < 0 || (n && (!pts || !dot))) return ODC_E_ARG;
  DotArgs a{f, pts, n, dot};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    DotArgs* x = (DotArgs*)p;
    if (x->n == 0) return (int)ODC_OK;
    cc->valid = false;
    cc->arena.reset();
    double* dp = need(cc->arena.get<double>(3 * x->n));
    uint8_t* dl = need(cc->arena.get<uint8_t>(x->n));
    float* dd = need(cc->arena.get<float>(x->n));
    CUDA_TRY(cudaMemcpyAsync(dp, x->pts, sizeof(double) * 3 * x->n, cudaMemcpyHostToDevice, cc->stream));
    PointSrc src{dp, GridP{}, 0};
    src.dot_out = dd;
    run_mlp(cc, x->f, src, x->n, dl, nullptr, cc->stream);
    check_launch(cc);
    CUDA_TRY(cudaMemcpyAsync(x->dot, dd, sizeof(float) * x->n, cudaMemcpyDeviceToHost, cc->stream));
    CUDA_TRY(cudaStreamSynchronize(cc->stream));
    return (int)ODC_OK;
  }, &a);
}

struct Eigh3Args {
  const double* A;
  int64_t n;
  double *w, *V;
  int32_t* info;
};
int odc_eigh3(odc_ctx* c, const double* A, int64_t n, double* w, double* V, int32_t* info) {
  if (!c || n < 0 || (n && (!A || !w || !V || !info))) return ODC_E_ARG;
  Eigh3Args a{A, n, w, V, info};
  cudaSetDevice(c->device);
  return guard(c, [](odc_ctx* cc, void* p) {
    Eigh3Args* x = (Eigh3Args*)p;
    if (x->n == 0) return (int)ODC_OK;
    cc->valid = false;  // reuses the workspace
    cc->arena.reset();
    double* dA = need(cc->arena.get<double>(9 * x->n));
    double* dw = need(cc->arena.get<double>(3 * x->n));
    double* dV = need(cc->arena.get<double>(9 * x->n));
    int32_t* di = need(cc->arena.get<int32_t>(x->n));
    CUDA_TRY(cudaMemcpyAsync(dA, x->A, sizeof(double) * 9 * x->n, cudaMemcpyHostToDevice, cc->stream));
    launch_eigh3_batch(dA, x->n, dw, dV, di, cc->stream);
    cc->launches++;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(x->w, dw, sizeof(double) * 3 * x->n, cudaMemcpyDeviceToHost, cc->stream));
    CUDA_TRY(cudaMemcpyAsync(x->V, dV, sizeof(double) * 9 * x->n, cudaMemcpyDeviceToHost, cc->stream));
    CUDA_TRY(cudaMemcpyAsync(x->info, di, sizeof(int32_t) * x->n, cudaMemcpyDeviceToHost, cc->stream));
    CUDA_TRY(cudaStreamSynchronize(cc->stream));
    return (int)ODC_OK;
  }, &a);
}
int odc_eigh3_host(const double* A, int64_t n, double* w, double* V, int32_t* info) {
  if (n < 0 || (n && (!A || !w || !V || !info))) return ODC_E_ARG;
  eigh3_host_batch(A, n, w, V, info);
  return ODC_OK;
}

}  // extern "C"
