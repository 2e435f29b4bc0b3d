/*
 * odc_oracle.c -- CPU oracle (TEST INFRASTRUCTURE ONLY; see odc_oracle.h).
 *
 * A lock-step, single-threaded C restatement of occmesh.pipeline.contour.
 * Each section cites the reference function it restates
 * (paths relative to /root/reference/pkg/src/occmesh/).  Floating-point
 * expressions follow numpy's evaluation order, measured on the reference
 * host and re-checked by tests/test_oracle_golden.py:
 *   - separate ufuncs never fuse (compile with -ffp-contract=off);
 *   - norm(x, axis=1) of (N,3)      = sqrt((x0*x0 + x1*x1) + x2*x2);
 *   - einsum('ij,ij->i') (3 terms)  = (p0 + p2) + p1;
 *   - einsum('pij,pi->pj')          = (t0 + t1) + t2;
 *   - einsum('pij,pj->pi')          = (t0 + t2) + t1;
 *   - (N,3) @ (3,3) (OpenBLAS dgemm) and 1-D x @ y (ddot) = fma chain
 *     fma(a2, b2, fma(a1, b1, a0*b0));
 *   - np.add.at accumulates sequentially in index order.
 * The QEF eigensolve (np.linalg.eigh, dualize.py:358) calls numpy's own
 * LAPACK dsyevd through a function pointer the caller supplies, so the whole
 * result -- positions, split cases, mesh -- is the reference's bit for bit
 * (tests/test_oracle_golden.py).
 */
#include "odc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_E_ASSERT 1
#define ORC_E_CONTRACT 2
#define ORC_E_CONFIG 3
#define ORC_E_VALUE 4
#define ORC_E_ALLOC 5

int orc_version(void) { return 1; }

/* ------------------------------------------------------------------------ */
/* helpers                                                                  */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t S, R, S2, S3;
  double lo[3], h[3];
} grid_t;

static inline double gpos(const grid_t* g, int a, int64_t c) { return g->lo[a] + (double)c * g->h[a]; }
static inline void vcoords(const grid_t* g, int64_t vid, int64_t c[3]) {
  c[0] = vid % g->S;
  c[1] = (vid / g->S) % g->S;
  c[2] = vid / g->S2;
}
static inline void vposition(const grid_t* g, int64_t vid, double p[3]) {
  int64_t c[3];
  vcoords(g, vid, c);
  for (int a = 0; a < 3; a++) p[a] = gpos(g, a, c[a]);
}
static inline int64_t vstep(const grid_t* g, int a) { return a == 0 ? 1 : (a == 1 ? g->S : g->S2); }

static void* xalloc(size_t n) {
  void* p = calloc(n ? n : 1, 1);
  return p;
}

static int64_t lower_bound_i64(const int64_t* a, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

static inline double dot3_fma(const double* a, const double* b) { return fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0])); }
static inline double einsum3(const double* a, const double* b) {
  /* einsum('ij,ij->i') with 3 terms: (p0 + p2) + p1 */
  double p0 = a[0] * b[0], p1 = a[1] * b[1], p2 = a[2] * b[2];
  return (p0 + p2) + p1;
}
static inline double norm3_rows(const double* x) { return sqrt((x[0] * x[0] + x[1] * x[1]) + x[2] * x[2]); }
static inline void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

/* ------------------------------------------------------------------------ */
/* Field evaluation: fields.py:35-242 (raw value semantics)                 */
/* ------------------------------------------------------------------------ */
/* (p - c) @ R with OpenBLAS's fma chain (fields.py:107, :179). */
static inline void rot_rows(const double* l, const double* R, double* o) {
  for (int j = 0; j < 3; j++) o[j] = fma(l[2], R[6 + j], fma(l[1], R[3 + j], l[0] * R[j]));
}

static double eval_prog_point(const orc_node* prog, int32_t n_nodes, const double* pt) {
  double st[64];
  double pst[16][3];
  int sp = 0, pp = 0;
  double p[3] = {pt[0], pt[1], pt[2]};
  for (int i = 0; i < n_nodes; i++) {
    const orc_node* nd = &prog[i];
    const double* q = nd->p;
    switch (nd->op) {
      case ORC_OP_SPHERE_SD: { /* fields.py:80-82 */
        double d[3] = {p[0] - q[0], p[1] - q[1], p[2] - q[2]};
        st[sp++] = norm3_rows(d) - q[3];
        break;
      }
      case ORC_OP_BOX_SD: { /* fields.py:103-111 */
        double l[3] = {p[0] - q[0], p[1] - q[1], p[2] - q[2]};
        if (q[6] != 0.0) {
          double o[3];
          rot_rows(l, q + 7, o);
          l[0] = o[0]; l[1] = o[1]; l[2] = o[2];
        }
        double qq[3], mq[3];
        for (int a = 0; a < 3; a++) {
          qq[a] = fabs(l[a]) - q[3 + a];
          mq[a] = qq[a] > 0.0 ? qq[a] : 0.0;
        }
        double outside = norm3_rows(mq);
        double mx = qq[0];
        if (qq[1] > mx) mx = qq[1];
        if (qq[2] > mx) mx = qq[2];
        double inside = mx < 0.0 ? mx : 0.0;
        st[sp++] = outside + inside;
        break;
      }
      case ORC_OP_TORUS_SD: { /* fields.py:122-126 */
        double l[3] = {p[0] - q[0], p[1] - q[1], p[2] - q[2]};
        double ring = hypot(l[0], l[1]) - q[3];
        st[sp++] = hypot(ring, l[2]) - q[4];
        break;
      }
      case ORC_OP_PLANE_SD: { /* fields.py:138-139 (dgemv; order tolerance-only) */
        double l[3] = {p[0] - q[0], p[1] - q[1], p[2] - q[2]};
        st[sp++] = dot3_fma(l, q + 3);
        break;
      }
      case ORC_OP_SD2RAW: /* fields.py:70-72 */
        st[sp - 1] = st[sp - 1] < 0.0 ? 1.0 : 0.0;
        break;
      case ORC_OP_RAW_MAX: case ORC_OP_SD_MAX: {
        double b = st[--sp], a = st[sp - 1];
        st[sp - 1] = (a >= b) ? a : b;
        break;
      }
      case ORC_OP_RAW_MIN: case ORC_OP_SD_MIN: {
        double b = st[--sp], a = st[sp - 1];
        st[sp - 1] = (a <= b) ? a : b;
        break;
      }
      case ORC_OP_RAW_DIFF: { /* fields.py:197 */
        double b = 1.0 - st[--sp], a = st[sp - 1];
        st[sp - 1] = (a <= b) ? a : b;
        break;
      }
      case ORC_OP_RAW_COMPL: st[sp - 1] = 1.0 - st[sp - 1]; break;
      case ORC_OP_SD_DIFF: { /* fields.py:216 */
        double b = -st[--sp], a = st[sp - 1];
        st[sp - 1] = (a >= b) ? a : b;
        break;
      }
      case ORC_OP_SD_NEG: st[sp - 1] = -st[sp - 1]; break;
      case ORC_OP_XFORM_BEGIN: { /* fields.py:176-180 */
        pst[pp][0] = p[0]; pst[pp][1] = p[1]; pst[pp][2] = p[2]; pp++;
        double l[3] = {p[0] - q[0], p[1] - q[1], p[2] - q[2]};
        if (q[6] != 0.0) {
          double o[3];
          rot_rows(l, q + 7, o);
          l[0] = o[0]; l[1] = o[1]; l[2] = o[2];
        }
        p[0] = l[0]; p[1] = l[1]; p[2] = l[2];
        break;
      }
      case ORC_OP_XFORM_END:
        pp--;
        p[0] = pst[pp][0]; p[1] = pst[pp][1]; p[2] = pst[pp][2];
        break;
      case ORC_OP_SMOOTH: { /* fields.py:239-242 */
        double kd = q[0] * st[sp - 1];
        if (kd < -500.0) kd = -500.0;
        if (kd > 500.0) kd = 500.0;
        st[sp - 1] = 1.0 / (1.0 + exp(kd));
        break;
      }
      default: break;
    }
  }
  return sp > 0 ? st[sp - 1] : 0.0;
}

int orc_eval_raw(const orc_node* prog, int32_t n_nodes, const double* pts, int64_t n, double* raw) {
  for (int64_t i = 0; i < n; i++) raw[i] = eval_prog_point(prog, n_nodes, pts + 3 * i);
  return 0;
}

typedef struct {
  const orc_node* prog;
  int32_t n_nodes;
  orc_raw_cb cb;
  void* user;
  double iso;
  orc_result* res;
  int n_order;
} field_t;

static void record(field_t* f, int cat, int64_t batches, int64_t evals) {
  orc_result* r = f->res;
  int seen = 0;
  for (int i = 0; i < f->n_order; i++)
    if (r->cat_order[i] == cat) seen = 1;
  if (!seen) r->cat_order[f->n_order++] = cat;
  r->eval_batches[cat] += batches;
  r->eval_evals[cat] += evals;
}

/* One logical batch -> raw values (pipeline.py:46-48 EvalCounter.raw). */
static void batch_raw(field_t* f, const double* pts, int64_t n, double* raw, int cat) {
  if (f->cb) {
    f->cb(pts, n, raw, cat, f->user);
  } else {
    orc_eval_raw(f->prog, f->n_nodes, pts, n, raw);
  }
}

/* One logical batch -> labels (pipeline.py:42-44; fields.py:35-48). */
static void batch_labels(field_t* f, const double* pts, int64_t n, uint8_t* lab, int cat) {
  record(f, cat, 1, n);
  double* raw = (double*)malloc(sizeof(double) * (n ? n : 1));
  batch_raw(f, pts, n, raw, cat);
  for (int64_t i = 0; i < n; i++) lab[i] = raw[i] > f->iso ? 1 : 0;
  free(raw);
}

/* numpy.linalg.eigh(UPLO='L') through numpy's own LAPACK dsyevd (the call
   solve_qef_batch makes, dualize.py:358), so QEF positions are the reference's. */
typedef void (*dsyevd_fn)(const char*, const char*, const int64_t*, double*, const int64_t*, double*,
                          double*, const int64_t*, int64_t*, const int64_t*, int64_t*, size_t, size_t);
static void lapack_eigh3(void* fn, const double Ain[9], double w[3], double V[9]) {
  double a[9];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) a[i + 3 * j] = Ain[3 * i + j]; /* column-major */
  int64_t n = 3, lda = 3, info = 0, lwork = 64, liwork = 32;
  double work[64];
  int64_t iwork[32];
  ((dsyevd_fn)fn)("V", "L", &n, a, &lda, w, work, &lwork, iwork, &liwork, &info, 1, 1);
  for (int i = 0; i < 3; i++)
    for (int k = 0; k < 3; k++) V[3 * i + k] = a[i + 3 * k];
}

/* ------------------------------------------------------------------------ */
/* main pipeline                                                            */
/* ------------------------------------------------------------------------ */
#define FAIL(code, ...) do { r->error = (code); snprintf(r->errmsg, sizeof r->errmsg, __VA_ARGS__); goto done; } while (0)

/* partitions lookup (dualize.py:180-188) */
typedef struct { int64_t key, pid; } kv_t;
static int kv_cmp(const void* a, const void* b) {
  int64_t x = ((const kv_t*)a)->key, y = ((const kv_t*)b)->key;
  return x < y ? -1 : (x > y);
}

typedef struct { int64_t key, slot; } ks_t;
static int ks_cmp(const void* a, const void* b) {
  const ks_t *x = (const ks_t*)a, *y = (const ks_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->slot < y->slot ? -1 : (x->slot > y->slot);
}

typedef struct { double th; int64_t idx; } th_t;
static int th_cmp(const void* a, const void* b) {
  const th_t *x = (const th_t*)a, *y = (const th_t*)b;
  if (x->th != y->th) return x->th < y->th ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static int repair_nonmanifold(const double* v_in, int64_t V, const int64_t* t_in, int64_t T,
                              const int64_t* kind_in, const int64_t* ref_in, orc_result* r);

int orc_contour(const orc_node* prog, int32_t n_nodes, orc_raw_cb cb, void* user,
                const double lo[3], const double hi[3], int64_t R,
                const orc_options* opt, orc_result* out) {
  orc_result* r = out;
  memset(r, 0, sizeof *r);
  if (!opt->dsyevd) return ORC_E_CONFIG; /* numpy's LAPACK dsyevd is required */
  for (int i = 0; i < ORC_N_CAT; i++) r->cat_order[i] = -1;
  field_t F = {prog, n_nodes, cb, user, opt->iso_level, r, 0};
  field_t* f = &F;

  /* scratch freed at done: */
  double* pts = NULL;
  uint8_t* lab = NULL;
  uint8_t* crossing = NULL;
  int64_t* inst_start = NULL;
  uint8_t* center_lab = NULL;
  double *lo1 = NULL, *hi1 = NULL;
  kv_t* lookup = NULL;
  double* part_pos_tmp = NULL;
  int64_t* sample_part = NULL;
  int64_t* sample_edge = NULL;
  double* sample_pe = NULL;
  double* edge_normals = NULL;

  /* ---- GridSpec (grid.py:17-91) ---- */
  if (R < 2) FAIL(ORC_E_VALUE, "resolution must be at least 2");
  for (int a = 0; a < 3; a++)
    if (!(hi[a] > lo[a])) FAIL(ORC_E_VALUE, "grid box must have positive extent");
  if (opt->one_d < 0 || opt->one_d > 2) FAIL(ORC_E_CONFIG, "unknown 1D mode");
  if (opt->normals < 0 || opt->normals > 1) FAIL(ORC_E_CONFIG, "unknown normal mode");
  if (opt->split < 0 || opt->split > 1) FAIL(ORC_E_CONFIG, "unknown split mode");
  grid_t G;
  G.R = R; G.S = R + 1; G.S2 = G.S * G.S; G.S3 = G.S2 * G.S;
  for (int a = 0; a < 3; a++) { G.lo[a] = lo[a]; G.h[a] = (hi[a] - lo[a]) / (double)R; r->h[a] = G.h[a]; }
  grid_t* g = &G;
  r->S = G.S; r->R = R;
  const int64_t S = G.S, S3 = G.S3;

  /* ---- sample_labels (grid.py:109-126) ---- */
  r->labels = (uint8_t*)xalloc(S3);
  if (opt->continuous) r->raw = (double*)xalloc(sizeof(double) * S3);
  {
    const int64_t CH = 1 << 20;
    pts = (double*)malloc(sizeof(double) * 3 * CH);
    double* rw = (double*)malloc(sizeof(double) * CH);
    for (int64_t s0 = 0; s0 < S3; s0 += CH) {
      int64_t n = (S3 - s0 < CH) ? S3 - s0 : CH;
      for (int64_t i = 0; i < n; i++) vposition(g, s0 + i, pts + 3 * i);
      batch_raw(f, pts, n, rw, ORC_CAT_LABELS);
      for (int64_t i = 0; i < n; i++) {
        r->labels[s0 + i] = rw[i] > f->iso ? 1 : 0;
        if (r->raw) r->raw[s0 + i] = rw[i];
      }
    }
    free(rw);
    free(pts); pts = NULL;
    record(f, ORC_CAT_LABELS, 1, S3);
  }
  const uint8_t* L = r->labels;
  /* boundary_inside_count (grid.py:102-106) */
  {
    int64_t shell = 0;
    for (int64_t vid = 0; vid < S3; vid++) {
      if (!L[vid]) continue;
      int64_t c[3];
      vcoords(g, vid, c);
      int on = 0;
      for (int a = 0; a < 3; a++) on |= (c[a] == 0 || c[a] == R);
      shell += on;
    }
    r->boundary_inside = shell;
  }

  /* ---- extract_active (grid.py:171-296) ---- */
  crossing = (uint8_t*)xalloc(S3);
  {
    int64_t K = 0;
    for (int64_t vid = 0; vid < S3; vid++) {
      int64_t c[3];
      vcoords(g, vid, c);
      for (int a = 0; a < 3; a++)
        if (c[a] < R && L[vid] != L[vid + vstep(g, a)]) { crossing[vid] |= (uint8_t)(1 << a); K++; }
    }
    r->K = K;
    r->edge_key = (int64_t*)xalloc(8 * K);
    r->v_in = (int64_t*)xalloc(8 * K);
    r->v_out = (int64_t*)xalloc(8 * K);
    int64_t k = 0;
    for (int64_t vid = 0; vid < S3; vid++) {
      if (!crossing[vid]) continue;
      for (int a = 0; a < 3; a++) {
        if (!(crossing[vid] >> a & 1)) continue;
        int64_t other = vid + vstep(g, a);
        r->edge_key[k] = vid * 3 + a;
        int base_in = L[vid] == 1;
        r->v_in[k] = base_in ? vid : other;
        r->v_out[k] = base_in ? other : vid;
        k++;
      }
    }
  }
  const int64_t K = r->K;
#define CROSS(key) ((crossing[(key) / 3] >> ((key) % 3)) & 1)
  {
    /* faces: every face whose in-plane coordinates are < R and that has >= 2
       crossing boundary edges (the reference's candidate set is exactly these,
       grid.py:212-260) */
    int64_t Fc = 0, F4 = 0;
    for (int pass = 0; pass < 2; pass++) {
      int64_t fr = 0;
      for (int64_t vid = 0; vid < S3; vid++) {
        int64_t c[3];
        vcoords(g, vid, c);
        for (int n = 0; n < 3; n++) {
          int b = (n + 1) % 3, cc = (n + 2) % 3;
          if (!(c[b] < R && c[cc] < R)) continue;
          int64_t w0 = vid, w1 = vid + vstep(g, b), w3 = vid + vstep(g, cc);
          int64_t e[4] = {w0 * 3 + b, w1 * 3 + cc, w3 * 3 + b, w0 * 3 + cc};
          int nc = 0;
          for (int j = 0; j < 4; j++) nc += CROSS(e[j]);
          if (nc % 2) FAIL(ORC_E_ASSERT, "face crossing-edge parity violated");
          if (nc < 2) continue;
          if (pass == 0) { Fc++; if (nc == 4) F4++; }
          else { r->face_key[fr] = vid * 3 + n; r->face_ncross[fr] = nc; fr++; }
        }
      }
      if (pass == 0) {
        r->F = Fc; r->F4 = F4;
        r->face_key = (int64_t*)xalloc(8 * Fc);
        r->face_ncross = (int64_t*)xalloc(8 * Fc);
      }
    }
    /* cells: union of the cells around crossing edges (grid.py:263-278) */
    int64_t Cc = 0;
    for (int pass = 0; pass < 2; pass++) {
      int64_t ci = 0;
      for (int64_t z = 0; z < R; z++)
        for (int64_t y = 0; y < R; y++)
          for (int64_t x = 0; x < R; x++) {
            int64_t base = x + y * S + z * G.S2;
            int any = 0;
            /* the cell's 12 edges */
            for (int i = 0; i < 8 && !any; i++) {
              int64_t v = base + (i & 1) + ((i >> 1) & 1) * S + ((i >> 2) & 1) * G.S2;
              for (int a = 0; a < 3; a++)
                if (!((i >> a) & 1) && (crossing[v] >> a & 1)) any = 1;
            }
            if (!any) continue;
            if (pass == 1) r->cells[ci] = x + y * R + z * R * R;
            ci++;
          }
      if (pass == 0) { Cc = ci; r->C = Cc; r->cells = (int64_t*)xalloc(8 * Cc); }
    }
  }
  const int64_t Fn = r->F;
  if (K == 0) goto done; /* pipeline.py:174-179 */

  /* ---- _edge_points / find_1d_points (pipeline.py:94-123, search.py:71-94) ---- */
  r->t1d = (double*)xalloc(8 * K);
  r->pos1d = (double*)xalloc(24 * K);
  {
    double* pin = (double*)malloc(24 * K);
    double* span = (double*)malloc(24 * K);
    for (int64_t k = 0; k < K; k++) {
      double a[3], b[3];
      vposition(g, r->v_in[k], a);
      vposition(g, r->v_out[k], b);
      for (int j = 0; j < 3; j++) { pin[3 * k + j] = a[j]; span[3 * k + j] = b[j] - a[j]; }
    }
    if (opt->one_d == 0) {
      lo1 = (double*)malloc(8 * K);
      hi1 = (double*)malloc(8 * K);
      pts = (double*)malloc(24 * K);
      lab = (uint8_t*)malloc(K);
      for (int64_t k = 0; k < K; k++) { lo1[k] = 0.0; hi1[k] = 1.0; }
      for (int it = 0; it < opt->iters_1d; it++) {
        for (int64_t k = 0; k < K; k++) {
          double tm = 0.5 * (lo1[k] + hi1[k]);
          for (int j = 0; j < 3; j++) pts[3 * k + j] = pin[3 * k + j] + tm * span[3 * k + j];
        }
        batch_labels(f, pts, K, lab, ORC_CAT_SEARCH_1D);
        for (int64_t k = 0; k < K; k++) {
          double tm = 0.5 * (lo1[k] + hi1[k]);
          if (lab[k] == 1) lo1[k] = tm; else hi1[k] = tm;
        }
      }
      double eps = ldexp(1.0, -opt->iters_1d);
      double upper = 1.0 - eps;
      for (int64_t k = 0; k < K; k++) {
        double t = 0.5 * (lo1[k] + hi1[k]);
        t = t < eps ? eps : t;
        t = t > upper ? upper : t;
        r->t1d[k] = t;
      }
      free(pts); pts = NULL;
      free(lab); lab = NULL;
    } else if (opt->one_d == 1) {
      for (int64_t k = 0; k < K; k++) r->t1d[k] = 0.5;
    } else {
      for (int64_t k = 0; k < K; k++) {
        double ri, ro;
        if (r->raw) { ri = r->raw[r->v_in[k]]; ro = r->raw[r->v_out[k]]; }
        else { ri = (double)L[r->v_in[k]]; ro = (double)L[r->v_out[k]]; }
        double pi = ri - opt->iso_level, po = ro - opt->iso_level;
        double den = pi - po;
        double t = fabs(den) < 1e-300 ? 0.5 : pi / (den == 0.0 ? 1.0 : den);
        t = t < 0.0 ? 0.0 : t;
        t = t > 1.0 ? 1.0 : t;
        r->t1d[k] = t;
      }
    }
    for (int64_t k = 0; k < K; k++)
      for (int j = 0; j < 3; j++) r->pos1d[3 * k + j] = pin[3 * k + j] + r->t1d[k] * span[3 * k + j];
    free(pin);
    free(span);
  }

  /* ---- face_pairings (dualize.py:51-94) ---- */
  {
    center_lab = (uint8_t*)xalloc(Fn);
    int64_t F4 = r->F4;
    if (F4) {
      pts = (double*)malloc(24 * F4);
      lab = (uint8_t*)malloc(F4);
      int64_t j = 0;
      for (int64_t fr = 0; fr < Fn; fr++) {
        if (r->face_ncross[fr] != 4) continue;
        int64_t vid = r->face_key[fr] / 3;
        int n = (int)(r->face_key[fr] % 3), b = (n + 1) % 3, c = (n + 2) % 3;
        double p[3];
        vposition(g, vid, p);
        p[b] += 0.5 * G.h[b];
        p[c] += 0.5 * G.h[c];
        memcpy(pts + 3 * j, p, 24);
        j++;
      }
      batch_labels(f, pts, F4, lab, ORC_CAT_PROBE_FACE_CENTER);
      j = 0;
      for (int64_t fr = 0; fr < Fn; fr++)
        if (r->face_ncross[fr] == 4) center_lab[fr] = lab[j++];
      free(pts); pts = NULL;
      free(lab); lab = NULL;
    }
    int64_t Q = Fn + F4;
    r->Q = Q;
    r->inst_face_row = (int64_t*)xalloc(8 * Q);
    r->inst_edges = (int64_t*)xalloc(16 * Q);
    inst_start = (int64_t*)xalloc(8 * (Fn + 1));
    int64_t q = 0;
    for (int64_t fr = 0; fr < Fn; fr++) {
      inst_start[fr] = q;
      int64_t vid = r->face_key[fr] / 3;
      int n = (int)(r->face_key[fr] % 3), b = (n + 1) % 3, c = (n + 2) % 3;
      int64_t w0 = vid, w1 = vid + vstep(g, b), w3 = vid + vstep(g, c);
      int64_t e[4] = {w0 * 3 + b, w1 * 3 + c, w3 * 3 + b, w0 * 3 + c};
      int64_t pairs[2][2];
      int np_ = 0;
      if (r->face_ncross[fr] == 2) {
        int64_t sel[2];
        int ns = 0;
        for (int j = 0; j < 4; j++)
          if (CROSS(e[j])) sel[ns++] = e[j];
        pairs[0][0] = sel[0]; pairs[0][1] = sel[1]; np_ = 1;
      } else { /* _pair_rule, dualize.py:37-48 */
        if (center_lab[fr] == L[w0]) {
          pairs[0][0] = e[0]; pairs[0][1] = e[1]; pairs[1][0] = e[2]; pairs[1][1] = e[3];
        } else {
          pairs[0][0] = e[3]; pairs[0][1] = e[0]; pairs[1][0] = e[1]; pairs[1][1] = e[2];
        }
        np_ = 2;
      }
      for (int j = 0; j < np_; j++) {
        int64_t a = pairs[j][0], bb = pairs[j][1];
        if (!(a < bb)) { int64_t t = a; a = bb; bb = t; }
        r->inst_face_row[q] = fr;
        r->inst_edges[2 * q] = a;
        r->inst_edges[2 * q + 1] = bb;
        q++;
      }
    }
    inst_start[Fn] = q;
  }
  const int64_t Q = r->Q;

  /* ---- partition_cells + trace_cycles (dualize.py:132-238) ---- */
  {
    int64_t Cn = r->C;
    int64_t cap = 16, P = 0, Ns = 0;
    int64_t capE = 64;
    r->part_cell = (int64_t*)malloc(8 * cap);
    r->part_index = (int64_t*)malloc(8 * cap);
    r->cyc_off = (int64_t*)malloc(8 * (cap + 1));
    r->cyc_edges = (int64_t*)malloc(8 * capE);
    r->cyc_insts = (int64_t*)malloc(8 * capE);
    r->cyc_off[0] = 0;
    for (int64_t ci = 0; ci < Cn; ci++) {
      int64_t cell = r->cells[ci];
      int64_t cx = cell % R, cy = (cell / R) % R, cz = cell / (R * R);
      int64_t base = cx + cy * S + cz * G.S2;
      /* cell_edge_keys (grid.py:315-322) then sorted (trace_cycles) */
      int64_t ek[12];
      int ne = 0;
      for (int a = 0; a < 3; a++)
        for (int i = 0; i < 8; i++) {
          if ((i >> a) & 1) continue;
          int64_t v = base + (i & 1) + ((i >> 1) & 1) * S + ((i >> 2) & 1) * G.S2;
          int64_t key = v * 3 + a;
          if (CROSS(key)) ek[ne++] = key;
        }
      for (int i = 0; i < ne; i++)
        for (int j = i + 1; j < ne; j++)
          if (ek[j] < ek[i]) { int64_t t = ek[i]; ek[i] = ek[j]; ek[j] = t; }
      /* joins[k]: up to 2 entries (inst, other) */
      int64_t jinst[12][4], joth[12][4];
      int jn[12] = {0};
      /* cell_face_keys (grid.py:325-334) */
      for (int a = 0; a < 3; a++)
        for (int side = 0; side < 2; side++) {
          int64_t fkey = (base + side * vstep(g, a)) * 3 + a;
          int64_t fr = lower_bound_i64(r->face_key, Fn, fkey);
          if (fr >= Fn || r->face_key[fr] != fkey) continue;
          for (int64_t qq = inst_start[fr]; qq < inst_start[fr + 1]; qq++) {
            int64_t ea = r->inst_edges[2 * qq], eb = r->inst_edges[2 * qq + 1];
            for (int i = 0; i < ne; i++) {
              if (ek[i] == ea && jn[i] < 4) { jinst[i][jn[i]] = qq; joth[i][jn[i]] = eb; jn[i]++; }
              if (ek[i] == eb && jn[i] < 4) { jinst[i][jn[i]] = qq; joth[i][jn[i]] = ea; jn[i]++; }
            }
          }
        }
      int visited[12] = {0};
      int cyc_idx = 0;
      for (int si = 0; si < ne; si++) {
        if (visited[si]) continue;
        if (jn[si] != 2) FAIL(ORC_E_CONTRACT, "edge %lld has %d joins, expected 2", (long long)ek[si], jn[si]);
        if (P + 1 >= cap) {
          cap *= 2;
          r->part_cell = (int64_t*)realloc(r->part_cell, 8 * cap);
          r->part_index = (int64_t*)realloc(r->part_index, 8 * cap);
          r->cyc_off = (int64_t*)realloc(r->cyc_off, 8 * (cap + 1));
        }
        /* min(joins[start]) over (inst, other) */
        int m = 0;
        if (jinst[si][1] < jinst[si][0] || (jinst[si][1] == jinst[si][0] && joth[si][1] < joth[si][0])) m = 1;
        int64_t inst = jinst[si][m], nxt = joth[si][m];
        int64_t start = ek[si];
        int64_t prev = inst;
        visited[si] = 1;
        int64_t ce[16], cinst[16];
        int len = 0;
        ce[len] = start; cinst[len] = inst; len++;
        while (nxt != start) {
          int ni = -1;
          for (int i = 0; i < ne; i++) if (ek[i] == nxt) ni = i;
          if (ni < 0 || len >= 12) FAIL(ORC_E_CONTRACT, "broken join cycle at edge %lld", (long long)nxt);
          visited[ni] = 1;
          int nopt = 0, pick = -1;
          for (int j = 0; j < jn[ni]; j++) if (jinst[ni][j] != prev) { nopt++; pick = j; }
          if (nopt != 1) FAIL(ORC_E_CONTRACT, "broken join cycle at edge %lld", (long long)nxt);
          ce[len] = nxt;
          inst = jinst[ni][pick];
          cinst[len] = inst;
          len++;
          prev = inst;
          nxt = joth[ni][pick];
        }
        if (Ns + len >= capE) {
          while (Ns + len >= capE) capE *= 2;
          r->cyc_edges = (int64_t*)realloc(r->cyc_edges, 8 * capE);
          r->cyc_insts = (int64_t*)realloc(r->cyc_insts, 8 * capE);
        }
        for (int i = 0; i < len; i++) { r->cyc_edges[Ns + i] = ce[i]; r->cyc_insts[Ns + i] = cinst[i]; }
        Ns += len;
        r->part_cell[P] = cell;
        r->part_index[P] = cyc_idx++;
        P++;
        r->cyc_off[P] = Ns;
      }
    }
    r->P = P;
    r->Ns = Ns;
    lookup = (kv_t*)xalloc(sizeof(kv_t) * Ns);
    int64_t stride = S3 * 3;
    for (int64_t p = 0; p < P; p++)
      for (int64_t s = r->cyc_off[p]; s < r->cyc_off[p + 1]; s++) {
        lookup[s].key = r->part_cell[p] * stride + r->cyc_edges[s];
        lookup[s].pid = p;
      }
    qsort(lookup, Ns, sizeof(kv_t), kv_cmp);
  }
  const int64_t P = r->P, Ns = r->Ns;

  /* ---- normals: two-d-points (search.py:194-322, dualize.py:97-129, :299-317, :402-429) ---- */
  sample_part = (int64_t*)xalloc(8 * Ns);
  sample_edge = (int64_t*)xalloc(8 * Ns);
  sample_pe = (double*)xalloc(24 * Ns);
  r->normals = (double*)xalloc(24 * Ns);
  for (int64_t p = 0; p < P; p++)
    for (int64_t s = r->cyc_off[p]; s < r->cyc_off[p + 1]; s++) {
      sample_part[s] = p;
      int64_t row = lower_bound_i64(r->edge_key, K, r->cyc_edges[s]);
      if (row >= K || r->edge_key[row] != r->cyc_edges[s]) FAIL(ORC_E_CONTRACT, "edge key not in the crossing set");
      sample_edge[s] = row;
      memcpy(sample_pe + 3 * s, r->pos1d + 3 * row, 24);
    }
  double hmin = G.h[0];
  if (G.h[1] < hmin) hmin = G.h[1];
  if (G.h[2] < hmin) hmin = G.h[2];

  if (opt->normals == 0) {
    /* build_face_batch (dualize.py:97-129) */
    double* org = (double*)malloc(24 * Q);
    int* bax = (int*)malloc(sizeof(int) * Q);
    int* cax = (int*)malloc(sizeof(int) * Q);
    double *hu = (double*)malloc(8 * Q), *hv = (double*)malloc(8 * Q);
    double *p1 = (double*)malloc(16 * Q), *p2 = (double*)malloc(16 * Q);
    uint8_t* cl = (uint8_t*)malloc(4 * Q);
    for (int64_t q = 0; q < Q; q++) {
      int64_t fr = r->inst_face_row[q];
      int64_t vid = r->face_key[fr] / 3;
      int n = (int)(r->face_key[fr] % 3), b = (n + 1) % 3, c = (n + 2) % 3;
      vposition(g, vid, org + 3 * q);
      bax[q] = b; cax[q] = c;
      hu[q] = G.h[b]; hv[q] = G.h[c];
      for (int j = 0; j < 2; j++) {
        int64_t key = r->inst_edges[2 * q + j];
        int64_t row = lower_bound_i64(r->edge_key, K, key);
        double* pp = (j == 0) ? p1 + 2 * q : p2 + 2 * q;
        pp[0] = r->pos1d[3 * row + b] - org[3 * q + b];
        pp[1] = r->pos1d[3 * row + c] - org[3 * q + c];
      }
      int64_t w0 = vid, w1 = vid + vstep(g, b), w3 = vid + vstep(g, c), w2 = w1 + vstep(g, c);
      cl[4 * q + 0] = L[w0]; cl[4 * q + 1] = L[w1]; cl[4 * q + 2] = L[w2]; cl[4 * q + 3] = L[w3];
    }
    /* find_2d_points (search.py:194-322) */
    double *mid = (double*)malloc(16 * Q), *dl = (double*)malloc(16 * Q), *ray = (double*)malloc(16 * Q);
    double* hmq = (double*)malloc(8 * Q);
    uint8_t* degen = (uint8_t*)malloc(Q);
    r->mid_label = (uint8_t*)xalloc(Q);
    pts = (double*)malloc(48 * Q);
    lab = (uint8_t*)malloc(2 * Q);
#define LIFT(q, u, v, out) do { (out)[0] = org[3*(q)]; (out)[1] = org[3*(q)+1]; (out)[2] = org[3*(q)+2]; \
      (out)[bax[q]] = org[3*(q)+bax[q]] + (u); (out)[cax[q]] = org[3*(q)+cax[q]] + (v); } while (0)
    for (int64_t q = 0; q < Q; q++) {
      double hm = hu[q] < hv[q] ? hu[q] : hv[q];
      hmq[q] = hm;
      mid[2 * q] = 0.5 * (p1[2 * q] + p2[2 * q]);
      mid[2 * q + 1] = 0.5 * (p1[2 * q + 1] + p2[2 * q + 1]);
      double ch0 = p2[2 * q] - p1[2 * q], ch1 = p2[2 * q + 1] - p1[2 * q + 1];
      double clen = sqrt(ch0 * ch0 + ch1 * ch1);
      degen[q] = clen < 1e-12 * hm;
      double safe = degen[q] ? 1.0 : clen;
      dl[2 * q] = ch0 / safe;
      dl[2 * q + 1] = ch1 / safe;
      LIFT(q, mid[2 * q], mid[2 * q + 1], pts + 3 * q);
    }
    batch_labels(f, pts, Q, r->mid_label, ORC_CAT_PROBE_FACE_MIDPOINT);
    for (int64_t q = 0; q < Q; q++) {
      double perp0 = -dl[2 * q + 1], perp1 = dl[2 * q];
      double cu[4] = {0.0, hu[q], hu[q], 0.0}, cv[4] = {0.0, 0.0, hv[q], hv[q]};
      double plus_d = INFINITY, minus_d = INFINITY;
      for (int c = 0; c < 4; c++) {
        double r0 = cu[c] - mid[2 * q], r1 = cv[c] - mid[2 * q + 1];
        double side = r0 * perp0 + r1 * perp1;
        double dist = sqrt(r0 * r0 + r1 * r1);
        if (cl[4 * q + c] == r->mid_label[q]) continue;
        if (side > 0 && dist < plus_d) plus_d = dist;
        if (side < 0 && dist < minus_d) minus_d = dist;
      }
      if (isinf(plus_d) && isinf(minus_d))
        FAIL(ORC_E_ASSERT, "2D search instance %lld: no corner label differs from the midpoint", (long long)q);
      if (plus_d <= minus_d) { ray[2 * q] = perp0; ray[2 * q + 1] = perp1; }
      else { ray[2 * q] = -perp0; ray[2 * q + 1] = -perp1; }
    }
    /* step 1: line_binary_search_batch (search.py:97-133) */
    double *q2 = (double*)malloc(16 * Q), *dist_r = (double*)malloc(8 * Q);
    uint8_t* found_r = (uint8_t*)xalloc(Q);
    {
      int N = opt->s1_lin, NB = opt->s1_bin;
      int64_t* first = (int64_t*)malloc(8 * Q);
      double *A = (double*)malloc(8 * Q), *B = (double*)malloc(8 * Q), *mr = (double*)malloc(8 * Q);
      for (int64_t q = 0; q < Q; q++) { first[q] = N; mr[q] = opt->s1_range * hmq[q]; }
      for (int i = 1; i <= N; i++) {
        double fr = (double)i / (double)N;
        for (int64_t q = 0; q < Q; q++) {
          double s = mr[q] * fr;
          LIFT(q, mid[2 * q] + s * ray[2 * q], mid[2 * q + 1] + s * ray[2 * q + 1], pts + 3 * q);
        }
        batch_labels(f, pts, Q, lab, ORC_CAT_SEARCH_2D);
        for (int64_t q = 0; q < Q; q++)
          if (lab[q] != r->mid_label[q] && !found_r[q]) { first[q] = i; found_r[q] = 1; }
      }
      for (int64_t q = 0; q < Q; q++) {
        A[q] = mr[q] * ((double)(first[q] - 1) / (double)N);
        B[q] = mr[q] * ((double)first[q] / (double)N);
      }
      for (int it = 0; it < NB; it++) {
        for (int64_t q = 0; q < Q; q++) {
          double m = 0.5 * (A[q] + B[q]);
          LIFT(q, mid[2 * q] + m * ray[2 * q], mid[2 * q + 1] + m * ray[2 * q + 1], pts + 3 * q);
        }
        batch_labels(f, pts, Q, lab, ORC_CAT_SEARCH_2D);
        for (int64_t q = 0; q < Q; q++) {
          double m = 0.5 * (A[q] + B[q]);
          if (lab[q] == r->mid_label[q]) A[q] = m; else B[q] = m;
        }
      }
      for (int64_t q = 0; q < Q; q++) {
        q2[2 * q] = mid[2 * q] + A[q] * ray[2 * q];
        q2[2 * q + 1] = mid[2 * q + 1] + A[q] * ray[2 * q + 1];
        dist_r[q] = A[q];
      }
      free(first); free(A); free(B); free(mr);
    }
    /* step 2: both rays in one lock-step batch of 2Q */
    double* q12 = (double*)malloc(32 * Q);
    uint8_t* found12 = (uint8_t*)xalloc(2 * Q);
    {
      int N = opt->s2_lin, NB = opt->s2_bin;
      int64_t M = 2 * Q;
      int64_t* first = (int64_t*)malloc(8 * M);
      double *A = (double*)malloc(8 * M), *B = (double*)malloc(8 * M), *mr = (double*)malloc(8 * M);
      double* dir = (double*)malloc(16 * M);
      for (int64_t m = 0; m < M; m++) {
        int64_t q = m < Q ? m : m - Q;
        first[m] = N;
        mr[m] = opt->s2_range * hmq[q];
        double sg = m < Q ? -1.0 : 1.0;
        dir[2 * m] = m < Q ? -dl[2 * q] : dl[2 * q];
        dir[2 * m + 1] = m < Q ? -dl[2 * q + 1] : dl[2 * q + 1];
        (void)sg;
      }
      for (int i = 1; i <= N; i++) {
        double fr = (double)i / (double)N;
        for (int64_t m = 0; m < M; m++) {
          int64_t q = m < Q ? m : m - Q;
          double s = mr[m] * fr;
          LIFT(q, q2[2 * q] + s * dir[2 * m], q2[2 * q + 1] + s * dir[2 * m + 1], pts + 3 * m);
        }
        batch_labels(f, pts, M, lab, ORC_CAT_SEARCH_2D);
        for (int64_t m = 0; m < M; m++) {
          int64_t q = m < Q ? m : m - Q;
          if (lab[m] != r->mid_label[q] && !found12[m]) { first[m] = i; found12[m] = 1; }
        }
      }
      for (int64_t m = 0; m < M; m++) {
        A[m] = mr[m] * ((double)(first[m] - 1) / (double)N);
        B[m] = mr[m] * ((double)first[m] / (double)N);
      }
      for (int it = 0; it < NB; it++) {
        for (int64_t m = 0; m < M; m++) {
          int64_t q = m < Q ? m : m - Q;
          double mm = 0.5 * (A[m] + B[m]);
          LIFT(q, q2[2 * q] + mm * dir[2 * m], q2[2 * q + 1] + mm * dir[2 * m + 1], pts + 3 * m);
        }
        batch_labels(f, pts, M, lab, ORC_CAT_SEARCH_2D);
        for (int64_t m = 0; m < M; m++) {
          int64_t q = m < Q ? m : m - Q;
          double mm = 0.5 * (A[m] + B[m]);
          if (lab[m] == r->mid_label[q]) A[m] = mm; else B[m] = mm;
        }
      }
      for (int64_t m = 0; m < M; m++) {
        int64_t q = m < Q ? m : m - Q;
        q12[2 * m] = q2[2 * q] + A[m] * dir[2 * m];
        q12[2 * m + 1] = q2[2 * q + 1] + A[m] * dir[2 * m + 1];
      }
      free(first); free(A); free(B); free(mr); free(dir);
    }
    /* intersection, clamp, status (search.py:278-322) */
    r->pos2 = (double*)xalloc(16 * Q);
    r->pos3 = (double*)xalloc(24 * Q);
    r->status = (uint8_t*)xalloc(Q);
    for (int64_t q = 0; q < Q; q++) {
      double hm = hmq[q];
      const double *P1 = p1 + 2 * q, *P2 = p2 + 2 * q, *M = mid + 2 * q;
      double qa[2] = {q12[2 * q], q12[2 * q + 1]}, qb[2] = {q12[2 * (q + Q)], q12[2 * (q + Q) + 1]};
      double a1[2] = {qa[0] - P1[0], qa[1] - P1[1]}, a2[2] = {qb[0] - P2[0], qb[1] - P2[1]};
      double l1 = sqrt(a1[0] * a1[0] + a1[1] * a1[1]), l2 = sqrt(a2[0] * a2[0] + a2[1] * a2[1]);
      double cr = a1[0] * a2[1] - a1[1] * a2[0];
      int exact = dist_r[q] <= 1e-4 * hm;
      int parallel = (fabs(cr) <= 1e-6 * l1 * l2) || (l1 < 1e-12 * hm) || (l2 < 1e-12 * hm) || degen[q];
      double sc = parallel ? 1.0 : cr;
      double d21[2] = {P2[0] - P1[0], P2[1] - P1[1]};
      double tpar = (d21[0] * a2[1] - d21[1] * a2[0]) / sc;
      double pf[2] = {P1[0] + tpar * a1[0], P1[1] + tpar * a1[1]};
      double pos[2];
      if (exact || parallel) { pos[0] = M[0]; pos[1] = M[1]; }
      else { pos[0] = pf[0]; pos[1] = pf[1]; }
      double lov[2] = {-0.5 * hu[q], -0.5 * hv[q]}, hiv[2] = {1.5 * hu[q], 1.5 * hv[q]};
      double delta[2] = {pos[0] - M[0], pos[1] - M[1]};
      double smin = INFINITY;
      for (int i = 0; i < 2; i++) {
        double shi = delta[i] > 0 ? (hiv[i] - M[i]) / delta[i] : INFINITY;
        double slo = delta[i] < 0 ? (lov[i] - M[i]) / delta[i] : INFINITY;
        double m2 = shi < slo ? shi : slo; /* np.minimum (no NaNs possible) */
        if (m2 < smin) smin = m2;
      }
      double s = smin < 1.0 ? smin : 1.0;
      int clamped = s < 1.0;
      double fin[2] = {M[0] + s * delta[0], M[1] + s * delta[1]};
      uint8_t st = 0;
      int unfound = !(found_r[q] && found12[q] && found12[q + Q]);
      if (unfound) st = 3;
      if (clamped) st = 2;
      if (parallel && !exact) st = 1;
      if (exact) st = 0;
      r->status[q] = st;
      r->pos2[2 * q] = fin[0];
      r->pos2[2 * q + 1] = fin[1];
      LIFT(q, fin[0], fin[1], r->pos3 + 3 * q);
    }
#undef LIFT
    free(org); free(bax); free(cax); free(hu); free(hv); free(p1); free(p2); free(cl);
    free(mid); free(dl); free(ray); free(hmq); free(degen);
    free(q2); free(dist_r); free(found_r); free(q12); free(found12);
    free(pts); pts = NULL;
    free(lab); lab = NULL;

    /* build_plane_samples + estimate_normals (dualize.py:299-317, :402-429) */
    int64_t nfb = 0;
    for (int64_t p = 0; p < P; p++) {
      int64_t s0 = r->cyc_off[p], len = r->cyc_off[p + 1] - s0;
      for (int64_t j = 0; j < len; j++) {
        int64_t s = s0 + j;
        int64_t ia = r->cyc_insts[s0 + (j - 1 + len) % len], ib = r->cyc_insts[s];
        const double* pe = sample_pe + 3 * s;
        double da[3], db[3], n[3];
        for (int c = 0; c < 3; c++) { da[c] = r->pos3[3 * ia + c] - pe[c]; db[c] = r->pos3[3 * ib + c] - pe[c]; }
        cross3(da, db, n);
        double nn = norm3_rows(n);
        int fb = nn <= 1e-9 * hmin * hmin;
        int64_t row = sample_edge[s];
        double pi[3], po[3], ed[3];
        vposition(g, r->v_in[row], pi);
        vposition(g, r->v_out[row], po);
        for (int c = 0; c < 3; c++) ed[c] = po[c] - pi[c];
        double el = norm3_rows(ed);
        double safe = fb ? 1.0 : nn;
        for (int c = 0; c < 3; c++) n[c] = n[c] / safe;
        if (fb) for (int c = 0; c < 3; c++) n[c] = ed[c] / el;
        if (einsum3(n, ed) < 0.0) for (int c = 0; c < 3; c++) n[c] = -n[c];
        memcpy(r->normals + 3 * s, n, 24);
        nfb += fb;
      }
    }
    r->n_fallback = nfb;
  } else {
    /* _fd_normals (pipeline.py:126-151) */
    if (!opt->continuous) FAIL(ORC_E_CONFIG, "fd-gradient normals require a field with continuous raw values");
    double step = opt->fd_step_factor * hmin;
    int64_t M = 6 * K;
    pts = (double*)malloc(24 * M);
    double* vals = (double*)malloc(8 * M);
    for (int i = 0; i < 6; i++)
      for (int64_t k = 0; k < K; k++)
        for (int c = 0; c < 3; c++) {
          double e = (c == i % 3) ? step : 0.0;
          pts[3 * (i * K + k) + c] = i < 3 ? r->pos1d[3 * k + c] + e : r->pos1d[3 * k + c] - e;
        }
    record(f, ORC_CAT_FD_GRADIENT, 1, M);
    batch_raw(f, pts, M, vals, ORC_CAT_FD_GRADIENT);
    edge_normals = (double*)malloc(24 * K);
    int64_t nbad = 0;
    for (int64_t k = 0; k < K; k++) {
      double gr[3], n[3];
      for (int i = 0; i < 3; i++) gr[i] = (vals[i * K + k] - vals[(i + 3) * K + k]) / (2.0 * step);
      double nr = norm3_rows(gr);
      double pi[3], po[3], ed[3];
      vposition(g, r->v_in[k], pi);
      vposition(g, r->v_out[k], po);
      for (int c = 0; c < 3; c++) ed[c] = po[c] - pi[c];
      double el = norm3_rows(ed);
      int bad = nr < 1e-30;
      double sn = bad ? 1.0 : nr;
      for (int c = 0; c < 3; c++) n[c] = bad ? ed[c] / el : -gr[c] / sn;
      if (einsum3(n, ed) < 0.0) for (int c = 0; c < 3; c++) n[c] = -n[c];
      memcpy(edge_normals + 3 * k, n, 24);
      nbad += bad;
    }
    for (int64_t s = 0; s < Ns; s++) memcpy(r->normals + 3 * s, edge_normals + 3 * sample_edge[s], 24);
    r->n_fallback = nbad;
    free(vals);
    free(pts); pts = NULL;
  }

  /* ---- place_3d_points / solve_qef_batch (dualize.py:332-372, :432-444) ---- */
  r->qef_pos = (double*)xalloc(24 * P);
  r->qef_rank = (int64_t*)xalloc(8 * P);
  r->qef_resid = (double*)xalloc(8 * P);
  for (int64_t p = 0; p < P; p++) {
    int64_t s0 = r->cyc_off[p], s1 = r->cyc_off[p + 1];
    double cnt = (double)(s1 - s0);
    if (cnt < 1.0) cnt = 1.0;
    double cen[3] = {0, 0, 0};
    for (int64_t s = s0; s < s1; s++)
      for (int c = 0; c < 3; c++) cen[c] += sample_pe[3 * s + c];
    for (int c = 0; c < 3; c++) cen[c] /= cnt;
    double A[9] = {0}, b[3] = {0, 0, 0};
    for (int64_t s = s0; s < s1; s++) {
      const double* n = r->normals + 3 * s;
      for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) A[3 * i + j] += n[i] * n[j];
    }
    for (int64_t s = s0; s < s1; s++) {
      const double* n = r->normals + 3 * s;
      double d[3] = {sample_pe[3 * s] - cen[0], sample_pe[3 * s + 1] - cen[1], sample_pe[3 * s + 2] - cen[2]};
      double off = einsum3(n, d);
      for (int c = 0; c < 3; c++) b[c] += n[c] * off;
    }
    double w[3], V[9];
    lapack_eigh3(opt->dsyevd, A, w, V);
    double sv[3];
    for (int k = 0; k < 3; k++) sv[k] = sqrt(w[k] > 0.0 ? w[k] : 0.0);
    double smax = sv[2];
    double thr = opt->qef_truncation * (smax > 1e-300 ? smax : 1e-300);
    int keep[3], rank = 0;
    for (int k = 0; k < 3; k++) { keep[k] = (sv[k] >= thr) && (smax > 0.0); rank += keep[k]; }
    double coef[3], y[3], sol[3];
    for (int j = 0; j < 3; j++) coef[j] = (V[0 + j] * b[0] + V[3 + j] * b[1]) + V[6 + j] * b[2];
    for (int j = 0; j < 3; j++) y[j] = keep[j] ? coef[j] / w[j] : 0.0;
    for (int i = 0; i < 3; i++) sol[i] = (V[3 * i] * y[0] + V[3 * i + 2] * y[2]) + V[3 * i + 1] * y[1];
    int64_t cell = r->part_cell[p];
    int64_t cc[3] = {cell % R, (cell / R) % R, cell / (R * R)};
    double pos[3];
    for (int c = 0; c < 3; c++) {
      double blo = G.lo[c] + (double)cc[c] * G.h[c];
      double bhi = blo + G.h[c];
      double x = cen[c] + sol[c];
      x = x > blo ? x : blo;
      x = x < bhi ? x : bhi;
      pos[c] = x;
    }
    double res = 0.0;
    for (int64_t s = s0; s < s1; s++) {
      double d[3] = {pos[0] - sample_pe[3 * s], pos[1] - sample_pe[3 * s + 1], pos[2] - sample_pe[3 * s + 2]};
      double e = einsum3(r->normals + 3 * s, d);
      res += e * e;
    }
    memcpy(r->qef_pos + 3 * p, pos, 24);
    r->qef_rank[p] = rank;
    r->qef_resid[p] = res;
  }

  /* ---- build_mesh (polygonize.py:110-217) ---- */
  {
    static const int RING[4][2] = {{-1, -1}, {0, -1}, {0, 0}, {-1, 0}};
    int64_t stride = S3 * 3;
    int64_t nint = 0, skipped = 0;
    int64_t* qp = (int64_t*)malloc(32 * K);    /* pids per interior edge */
    int64_t* qrow = (int64_t*)malloc(8 * K);   /* edge row per interior edge */
    for (int64_t k = 0; k < K; k++) {
      int64_t key = r->edge_key[k], vid = key / 3;
      int a = (int)(key % 3), b = (a + 1) % 3, c = (a + 2) % 3;
      int64_t vc[3];
      vcoords(g, vid, vc);
      int fwd = r->v_in[k] == vid;
      int ok = 1;
      int64_t cid[4];
      for (int j = 0; j < 4; j++) {
        int rj = fwd ? j : 3 - j;
        int64_t cc[3] = {vc[0], vc[1], vc[2]};
        cc[b] += RING[rj][0];
        cc[c] += RING[rj][1];
        for (int t = 0; t < 3; t++) if (cc[t] < 0 || cc[t] >= R) ok = 0;
        cid[j] = cc[0] + cc[1] * R + cc[2] * R * R;
      }
      if (!ok) { skipped++; continue; }
      for (int j = 0; j < 4; j++) {
        kv_t kk = {cid[j] * stride + key, 0};
        kv_t* hit = (kv_t*)bsearch(&kk, lookup, Ns, sizeof(kv_t), kv_cmp);
        if (!hit) FAIL(ORC_E_CONTRACT, "crossing edge without a partition in its cell");
        qp[4 * nint + j] = hit->pid;
      }
      qrow[nint] = k;
      nint++;
    }
    r->n_interior = nint;
    r->skipped = skipped;
    r->split_cases = (int8_t*)xalloc(nint);
    int64_t nfan = 0, ntri = 0;
    for (int64_t e = 0; e < nint; e++) {
      int cs = 1;
      if (opt->split == 0) {
        double pin[3], pout[3];
        vposition(g, r->v_in[qrow[e]], pin);
        vposition(g, r->v_out[qrow[e]], pout);
        int conc[4];
        for (int k = 0; k < 4; k++) {
          const double* pk = r->qef_pos + 3 * qp[4 * e + k];
          const double* da = r->qef_pos + 3 * qp[4 * e + (k + 3) % 4];
          const double* db = r->qef_pos + 3 * qp[4 * e + (k + 1) % 4];
          double u[3], v[3], w[3], x[3];
          for (int t = 0; t < 3; t++) { u[t] = da[t] - pout[t]; v[t] = db[t] - pout[t]; w[t] = pk[t] - pout[t]; }
          cross3(u, v, x);
          int plus = einsum3(w, x) < 0.0;
          for (int t = 0; t < 3; t++) { u[t] = da[t] - pin[t]; v[t] = db[t] - pin[t]; w[t] = pk[t] - pin[t]; }
          cross3(u, v, x);
          int minus = einsum3(w, x) > 0.0;
          conc[k] = plus || minus;
        }
        if (!(conc[1] || conc[3])) cs = 1;
        else if (!(conc[0] || conc[2])) cs = 2;
        else cs = 3;
      }
      r->split_cases[e] = (int8_t)cs;
      if (cs == 3) nfan++;
      ntri += cs == 3 ? 4 : 2;
    }
    int64_t V = P + nfan;
    double* verts = (double*)xalloc(24 * V);
    int64_t* kind = (int64_t*)xalloc(8 * V);
    int64_t* ref = (int64_t*)xalloc(16 * V);
    int64_t* tris = (int64_t*)xalloc(24 * ntri);
    memcpy(verts, r->qef_pos, 24 * P);
    for (int64_t p = 0; p < P; p++) { kind[p] = 0; ref[2 * p] = r->part_cell[p]; ref[2 * p + 1] = r->part_index[p]; }
    int64_t fv = P, o = 0;
    for (int64_t e = 0; e < nint; e++) {
      const int64_t* pd = qp + 4 * e;
      int cs = r->split_cases[e];
      if (cs == 1) {
        int64_t t[6] = {pd[0], pd[1], pd[2], pd[0], pd[2], pd[3]};
        memcpy(tris + 3 * o, t, 48); o += 2;
      } else if (cs == 2) {
        int64_t t[6] = {pd[0], pd[1], pd[3], pd[1], pd[2], pd[3]};
        memcpy(tris + 3 * o, t, 48); o += 2;
      } else {
        for (int j = 0; j < 4; j++) {
          tris[3 * o] = fv; tris[3 * o + 1] = pd[j]; tris[3 * o + 2] = pd[(j + 1) % 4]; o++;
        }
        memcpy(verts + 3 * fv, r->pos1d + 3 * qrow[e], 24);
        kind[fv] = 1; ref[2 * fv] = r->edge_key[qrow[e]]; ref[2 * fv + 1] = -1;
        fv++;
      }
    }
    /* drop unreferenced vertices (polygonize.py:199-209) */
    uint8_t* used = (uint8_t*)xalloc(V);
    for (int64_t i = 0; i < 3 * ntri; i++) used[tris[i]] = 1;
    int64_t nu = 0;
    for (int64_t i = 0; i < V; i++) nu += used[i];
    if (nu != V) {
      int64_t* remap = (int64_t*)malloc(8 * V);
      int64_t j = 0;
      for (int64_t i = 0; i < V; i++) {
        remap[i] = used[i] ? j : -1;
        if (used[i]) {
          memmove(verts + 3 * j, verts + 3 * i, 24);
          kind[j] = kind[i];
          ref[2 * j] = ref[2 * i]; ref[2 * j + 1] = ref[2 * i + 1];
          j++;
        }
      }
      for (int64_t i = 0; i < 3 * ntri; i++) tris[i] = remap[tris[i]];
      free(remap);
      V = nu;
    }
    free(used);
    free(qp); free(qrow);
    r->V0 = V; r->T0 = ntri; r->v0 = verts; r->t0 = tris; r->kind0 = kind; r->ref0 = ref;
  }

  /* ---- repair_nonmanifold (polygonize.py:253-374) ---- */
  if (opt->repair) {
    int rc = repair_nonmanifold(r->v0, r->V0, r->t0, r->T0, r->kind0, r->ref0, r);
    if (rc) FAIL(ORC_E_ALLOC, "repair failed");
  } else {
    r->V1 = r->V0; r->T1 = r->T0;
    r->v1 = (double*)xalloc(24 * r->V0); memcpy(r->v1, r->v0, 24 * r->V0);
    r->t1 = (int64_t*)xalloc(24 * r->T0); memcpy(r->t1, r->t0, 24 * r->T0);
    r->kind1 = (int64_t*)xalloc(8 * r->V0); memcpy(r->kind1, r->kind0, 8 * r->V0);
    r->ref1 = (int64_t*)xalloc(16 * r->V0); memcpy(r->ref1, r->ref0, 16 * r->V0);
  }

done:
#undef CROSS
  free(pts); free(lab); free(crossing); free(inst_start); free(center_lab);
  free(lo1); free(hi1); free(lookup); free(part_pos_tmp);
  free(sample_part); free(sample_edge); free(sample_pe); free(edge_normals);
  return r->error;
}

/* ------------------------------------------------------------------------ */
/* repair_nonmanifold (polygonize.py:220-374)                                */
/* ------------------------------------------------------------------------ */
typedef struct { int64_t a, b; int64_t n; int64_t* pairs; /* 2n owners */ } over_t;

static int64_t uf_find(int64_t* parent, int64_t x) {
  while (parent[x] != x) { parent[x] = parent[parent[x]]; x = parent[x]; }
  return x;
}

static int repair_nonmanifold(const double* v_in, int64_t V, const int64_t* t_in, int64_t T,
                              const int64_t* kind_in, const int64_t* ref_in, orc_result* r) {
  int64_t capV = V + 16;
  double* verts = (double*)malloc(24 * capV);
  memcpy(verts, v_in, 24 * V);
  int64_t* tris = (int64_t*)malloc(24 * (T ? T : 1));
  memcpy(tris, t_in, 24 * T);
  int64_t nV = V;
  if (T > 0) {
    for (int pass = 0; pass < 4; pass++) {
      /* _edge_sort_key (polygonize.py:220-230) */
      int64_t M = 3 * T;
      ks_t* ks = (ks_t*)malloc(sizeof(ks_t) * M);
      int64_t *elo = (int64_t*)malloc(8 * M), *ehi = (int64_t*)malloc(8 * M);
      uint8_t* dir = (uint8_t*)malloc(M);
      for (int64_t t = 0; t < T; t++)
        for (int j = 0; j < 3; j++) {
          int64_t s = 3 * t + j;
          int64_t e0 = tris[3 * t + j], e1 = tris[3 * t + (j + 1) % 3];
          elo[s] = e0 < e1 ? e0 : e1;
          ehi[s] = e0 < e1 ? e1 : e0;
          dir[s] = e0 < e1;
          ks[s].key = elo[s] * (nV + 1) + ehi[s];
          ks[s].slot = s;
        }
      qsort(ks, M, sizeof(ks_t), ks_cmp);
      /* over-populated edges -> sheet pairs */
      int64_t nover = 0, capo = 8;
      over_t* over = (over_t*)malloc(sizeof(over_t) * capo);
      for (int64_t i = 0; i < M;) {
        int64_t j = i;
        while (j < M && ks[j].key == ks[i].key) j++;
        int64_t gn = j - i;
        if (gn > 2) {
          const ks_t* gs = ks + i;
          int64_t a = elo[gs[0].slot], b = ehi[gs[0].slot];
          double axis[3];
          for (int c = 0; c < 3; c++) axis[c] = verts[3 * b + c] - verts[3 * a + c];
          double an = sqrt(dot3_fma(axis, axis));
          if (an == 0.0) an = 1.0;
          for (int c = 0; c < 3; c++) axis[c] /= an;
          double(*rel)[3] = (double(*)[3])malloc(24 * gn);
          for (int64_t u = 0; u < gn; u++) {
            int64_t t = gs[u].slot / 3;
            int64_t other = -1;
            for (int c = 0; c < 3 && other < 0; c++)
              if (tris[3 * t + c] != a && tris[3 * t + c] != b) other = tris[3 * t + c];
            double rr[3];
            for (int c = 0; c < 3; c++) rr[c] = verts[3 * other + c] - verts[3 * a + c];
            double pr = dot3_fma(rr, axis);
            for (int c = 0; c < 3; c++) rel[u][c] = rr[c] - axis[c] * pr;
          }
          double refv[3] = {rel[0][0], rel[0][1], rel[0][2]};
          double rn = sqrt(dot3_fma(refv, refv));
          if (rn == 0.0) rn = 1.0;
          for (int c = 0; c < 3; c++) refv[c] /= rn;
          double perp[3];
          cross3(axis, refv, perp);
          th_t* th = (th_t*)malloc(sizeof(th_t) * gn);
          for (int64_t u = 0; u < gn; u++) {
            th[u].th = atan2(dot3_fma(rel[u], perp), dot3_fma(rel[u], refv));
            th[u].idx = u;
          }
          qsort(th, gn, sizeof(th_t), th_cmp);
          /* _pair_fan_triangles (polygonize.py:233-250) */
          int64_t np_ = gn / 2;
          int64_t* pr = (int64_t*)malloc(16 * np_);
          int done_pairs = 0;
          int nstarts = (gn % 2 == 0) ? 2 : 1;
          for (int st = 0; st < nstarts && !done_pairs; st++) {
            int ok = 1;
            for (int64_t i2 = 0; i2 < np_; i2++) {
              int64_t x = th[(st + 2 * i2) % gn].idx, y = th[(st + 2 * i2 + 1) % gn].idx;
              pr[2 * i2] = x; pr[2 * i2 + 1] = y;
              if (dir[gs[x].slot] == dir[gs[y].slot]) ok = 0;
            }
            if (ok) done_pairs = 1;
          }
          if (!done_pairs)
            for (int64_t i2 = 0; i2 < np_; i2++) { pr[2 * i2] = th[2 * i2].idx; pr[2 * i2 + 1] = th[2 * i2 + 1].idx; }
          if (nover == capo) { capo *= 2; over = (over_t*)realloc(over, sizeof(over_t) * capo); }
          over[nover].a = a; over[nover].b = b; over[nover].n = np_;
          over[nover].pairs = (int64_t*)malloc(16 * (np_ ? np_ : 1));
          for (int64_t i2 = 0; i2 < np_; i2++) {
            over[nover].pairs[2 * i2] = gs[pr[2 * i2]].slot / 3;
            over[nover].pairs[2 * i2 + 1] = gs[pr[2 * i2 + 1]].slot / 3;
          }
          nover++;
          free(pr); free(th); free(rel);
        }
        i = j;
      }
      /* per-vertex fan components (polygonize.py:308-358) */
      int64_t* deg = (int64_t*)xalloc(8 * (nV + 1));
      for (int64_t i = 0; i < 3 * T; i++) deg[tris[i] + 1]++;
      for (int64_t v = 0; v < nV; v++) deg[v + 1] += deg[v];
      int64_t* inc = (int64_t*)malloc(8 * 3 * T);
      int64_t* fillp = (int64_t*)malloc(8 * (nV + 1));
      memcpy(fillp, deg, 8 * (nV + 1));
      for (int64_t i = 0; i < 3 * T; i++) inc[fillp[tris[i]]++] = i / 3; /* ascending triangle ids */
      free(fillp);
      int64_t nnew = 0, capn = 16;
      int64_t* newrows = (int64_t*)malloc(24 * capn); /* (t, old, new) */
      int64_t nappend = 0;
      int64_t next_vid = nV;
      int64_t* vapp = (int64_t*)malloc(8 * capn);
      for (int64_t vid = 0; vid < nV; vid++) {
        int64_t d0 = deg[vid], d1 = deg[vid + 1];
        int64_t nt = d1 - d0;
        if (nt <= 1) continue;
        const int64_t* tl = inc + d0; /* sorted unique (a vertex appears once per triangle) */
        int64_t* parent = (int64_t*)malloc(8 * nt);
        for (int64_t i = 0; i < nt; i++) parent[i] = i;
        /* edge_map in insertion order */
        int64_t* eo = (int64_t*)malloc(8 * 2 * nt);  /* other vertex per entry */
        int64_t* et = (int64_t*)malloc(8 * 2 * nt);  /* local triangle index */
        int64_t ne = 0;
        for (int64_t i = 0; i < nt; i++) {
          int64_t t = tl[i];
          for (int c = 0; c < 3; c++) {
            int64_t v = tris[3 * t + c];
            if (v == vid) continue;
            eo[ne] = v; et[ne] = i; ne++;
          }
        }
        uint8_t* seen = (uint8_t*)xalloc(ne);
        for (int64_t i = 0; i < ne; i++) {
          if (seen[i]) continue;
          int64_t members[64];
          int64_t nm = 0;
          for (int64_t j = i; j < ne; j++)
            if (eo[j] == eo[i]) { seen[j] = 1; if (nm < 64) members[nm++] = et[j]; }
          int64_t ea = vid < eo[i] ? vid : eo[i], eb = vid < eo[i] ? eo[i] : vid;
          int64_t oi = -1;
          for (int64_t u = 0; u < nover; u++) if (over[u].a == ea && over[u].b == eb) oi = u;
          if (nm == 2 && oi < 0) {
            int64_t ra = uf_find(parent, members[0]), rb = uf_find(parent, members[1]);
            if (ra != rb) parent[ra] = rb;
          } else if (oi >= 0) {
            for (int64_t u = 0; u < over[oi].n; u++) {
              int64_t pa = over[oi].pairs[2 * u], pb = over[oi].pairs[2 * u + 1];
              int64_t la = -1, lb = -1;
              for (int64_t x = 0; x < nt; x++) { if (tl[x] == pa) la = x; if (tl[x] == pb) lb = x; }
              if (la >= 0 && lb >= 0) {
                int64_t ra = uf_find(parent, la), rb = uf_find(parent, lb);
                if (ra != rb) parent[ra] = rb;
              }
            }
          }
        }
        /* components ordered by min triangle: the first local index of each root */
        int64_t* root = (int64_t*)malloc(8 * nt);
        for (int64_t i = 0; i < nt; i++) root[i] = uf_find(parent, i);
        int64_t* comp_of_root = (int64_t*)malloc(8 * nt);
        for (int64_t i = 0; i < nt; i++) comp_of_root[i] = -1;
        int64_t ncomp = 0;
        int64_t* comp = (int64_t*)malloc(8 * nt);
        for (int64_t i = 0; i < nt; i++) {
          if (comp_of_root[root[i]] < 0) comp_of_root[root[i]] = ncomp++;
          comp[i] = comp_of_root[root[i]];
        }
        if (ncomp > 1) {
          for (int64_t cidx = 1; cidx < ncomp; cidx++) {
            if (nappend + 1 >= capn || nnew + nt >= capn) {
              while (nappend + 1 >= capn || nnew + nt >= capn) capn *= 2;
              newrows = (int64_t*)realloc(newrows, 24 * capn);
              vapp = (int64_t*)realloc(vapp, 8 * capn);
            }
            vapp[nappend++] = vid;
            for (int64_t i = 0; i < nt; i++)
              if (comp[i] == cidx) {
                newrows[3 * nnew] = tl[i]; newrows[3 * nnew + 1] = vid; newrows[3 * nnew + 2] = next_vid; nnew++;
              }
            next_vid++;
          }
        }
        free(root); free(comp_of_root); free(comp); free(seen); free(eo); free(et); free(parent);
      }
      free(inc); free(deg);
      for (int64_t u = 0; u < nover; u++) free(over[u].pairs);
      free(over);
      free(ks); free(elo); free(ehi); free(dir);
      if (nnew == 0) { free(newrows); free(vapp); break; }
      for (int64_t i = 0; i < nnew; i++) {
        int64_t t = newrows[3 * i], old = newrows[3 * i + 1], nw = newrows[3 * i + 2];
        for (int c = 0; c < 3; c++) if (tris[3 * t + c] == old) tris[3 * t + c] = nw;
      }
      if (nV + nappend > capV) {
        capV = (nV + nappend) * 2;
        verts = (double*)realloc(verts, 24 * capV);
      }
      for (int64_t i = 0; i < nappend; i++) memcpy(verts + 3 * (nV + i), verts + 3 * vapp[i], 24);
      nV += nappend;
      free(newrows); free(vapp);
    }
  }
  r->V1 = nV; r->T1 = T;
  r->v1 = verts; r->t1 = tris;
  r->kind1 = (int64_t*)xalloc(8 * nV);
  r->ref1 = (int64_t*)xalloc(16 * nV);
  memcpy(r->kind1, kind_in, 8 * V);
  memcpy(r->ref1, ref_in, 16 * V);
  for (int64_t i = V; i < nV; i++) { r->kind1[i] = 2; r->ref1[2 * i] = -1; r->ref1[2 * i + 1] = -1; }
  return 0;
}

void orc_free(orc_result* r) {
  void* ptrs[] = {r->labels, r->raw, r->edge_key, r->v_in, r->v_out, r->face_key, r->face_ncross, r->cells,
                  r->inst_face_row, r->inst_edges, r->t1d, r->pos1d, r->pos2, r->pos3, r->status, r->mid_label,
                  r->part_cell, r->part_index, r->cyc_off, r->cyc_edges, r->cyc_insts, r->normals, r->qef_pos,
                  r->qef_resid, r->qef_rank, r->split_cases, r->v0, r->t0, r->kind0, r->ref0, r->v1, r->t1,
                  r->kind1, r->ref1};
  for (size_t i = 0; i < sizeof ptrs / sizeof ptrs[0]; i++) free(ptrs[i]);
  memset(r, 0, sizeof *r);
}
