/*
 * odc_oracle.h -- CPU oracle for the ODC extraction path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_2409_13418_b200/) includes, links or calls this code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may use it, and only as the checker / the CPU baseline.
 *
 * It is a plain-C, single-threaded, lock-step restatement of
 * occmesh.pipeline.contour (/root/reference/pkg/src/occmesh/pipeline.py:154-240)
 * and everything below it.  Every field query goes through one batched
 * evaluation per logical batch, exactly like the reference's EvalCounter
 * (pipeline.py:30-57), so batch/eval counts are reproduced and an external
 * field (numpy MlpField, or the GPU evaluator for the shared-field oracle)
 * can be plugged in through a callback.
 *
 * Pinning: tests/test_oracle_golden.py checks this oracle against golden
 * vectors produced by the unmodified reference (tests/golden/make_golden.py).
 */
#ifndef ODC_ORACLE_H
#define ODC_ORACLE_H
#include <stdint.h>

/* Field program opcodes (postfix; see paper_2409_13418_b200/fields.py for the
 * lowering rules and fields.py:64-242 of the reference for semantics). */
enum {
  ORC_OP_END = 0,
  ORC_OP_SPHERE_SD = 1,  /* p[0..2] centre, p[3] radius                       */
  ORC_OP_BOX_SD = 2,     /* p[0..2] centre, p[3..5] half, p[6] has_rot, p[7..15] R */
  ORC_OP_TORUS_SD = 3,   /* p[0..2] centre, p[3] major, p[4] minor             */
  ORC_OP_PLANE_SD = 4,   /* p[0..2] point, p[3..5] unit normal                 */
  ORC_OP_SD2RAW = 5,     /* raw = (sd < 0) ? 1 : 0                             */
  ORC_OP_RAW_MAX = 6,    /* union of raws                                      */
  ORC_OP_RAW_MIN = 7,    /* intersection                                       */
  ORC_OP_RAW_DIFF = 8,   /* min(a, 1 - b)                                      */
  ORC_OP_RAW_COMPL = 9,  /* 1 - a                                              */
  ORC_OP_SD_MIN = 10,    /* union of distances                                 */
  ORC_OP_SD_MAX = 11,    /* intersection                                       */
  ORC_OP_SD_DIFF = 12,   /* max(a, -b)                                         */
  ORC_OP_SD_NEG = 13,    /* -a                                                 */
  ORC_OP_XFORM_BEGIN = 14, /* p[0..2] translation, p[6] has_rot, p[7..15] R     */
  ORC_OP_XFORM_END = 15,
  ORC_OP_SMOOTH = 16,    /* p[0] sharpness: raw = 1/(1+exp(clip(k*sd,+-500)))   */
};

typedef struct {
  int32_t op;
  int32_t pad;
  double p[16];
} orc_node;

/* Eval categories, in the order the reference first records them. */
enum {
  ORC_CAT_LABELS = 0,
  ORC_CAT_SEARCH_1D = 1,
  ORC_CAT_PROBE_FACE_CENTER = 2,
  ORC_CAT_PROBE_FACE_MIDPOINT = 3,
  ORC_CAT_SEARCH_2D = 4,
  ORC_CAT_FD_GRADIENT = 5,
  ORC_N_CAT = 6
};

/* External field: fill raw[n] for pts[n*3] (raw values; label = raw > iso). */
typedef void (*orc_raw_cb)(const double* pts, int64_t n, double* raw, int32_t category, void* user);

typedef struct {
  int32_t one_d;    /* 0 binary-search, 1 midpoint, 2 linear-interp       */
  int32_t normals;  /* 0 two-d-points, 1 fd-gradient                      */
  int32_t split;    /* 0 ic, 1 mdc                                        */
  int32_t repair;   /* bool                                               */
  int32_t iters_1d;
  int32_t s1_lin, s1_bin;
  int32_t s2_lin, s2_bin;
  int32_t continuous; /* field.continuous                                 */
  double s1_range, s2_range;
  double qef_truncation, fd_step_factor;
  double iso_level;
  /* numpy's bundled LAPACK dsyevd (Fortran ABI, 64-bit ints), required: the
     QEF eigensolve is numpy.linalg.eigh (dualize.py:358) itself. */
  void* dsyevd;
} orc_options;

typedef struct {
  int64_t S, R;
  double h[3];
  /* labels / raw (raw only when continuous) */
  uint8_t* labels;
  double* raw;
  int64_t boundary_inside;
  /* active sets (grid.py:129-296) */
  int64_t K;
  int64_t *edge_key, *v_in, *v_out;
  int64_t F;
  int64_t *face_key, *face_ncross;
  int64_t C;
  int64_t* cells;
  int64_t F4;
  /* pairings (dualize.py:51-94) */
  int64_t Q;
  int64_t *inst_face_row, *inst_edges; /* (Q), (Q,2) */
  /* 1D points (search.py:71-94) */
  double *t1d, *pos1d; /* (K), (K,3) */
  /* 2D points (search.py:194-322) */
  double *pos2, *pos3; /* (Q,2), (Q,3) */
  uint8_t *status, *mid_label;
  /* partitions (dualize.py:194-238) */
  int64_t P, Ns;
  int64_t *part_cell, *part_index, *cyc_off, *cyc_edges, *cyc_insts; /* cyc_off (P+1) */
  /* plane samples + QEF (dualize.py:299-444) */
  double* normals;       /* (Ns,3) */
  int64_t n_fallback;
  double *qef_pos, *qef_resid; /* (P,3), (P) */
  int64_t* qef_rank;
  /* polygonize (polygonize.py:110-217) */
  int64_t n_interior, skipped;
  int8_t* split_cases; /* (n_interior) */
  int64_t V0, T0;
  double* v0; int64_t *t0, *kind0, *ref0;
  /* repair (polygonize.py:253-374) */
  int64_t V1, T1;
  double* v1; int64_t *t1, *kind1, *ref1;
  /* eval accounting (pipeline.py:30-57) */
  int64_t eval_batches[ORC_N_CAT], eval_evals[ORC_N_CAT];
  int32_t cat_order[ORC_N_CAT]; /* first-record order, -1 terminated */
  int32_t error;                /* 0 ok, 1 AssertionError, 2 InternalContractError, 3 ConfigurationError, 4 ValueError, 5 alloc */
  char errmsg[256];
} orc_result;

#ifdef __cplusplus
extern "C" {
#endif
int orc_contour(const orc_node* prog, int32_t n_nodes, orc_raw_cb cb, void* user,
                const double lo[3], const double hi[3], int64_t R,
                const orc_options* opt, orc_result* out);
void orc_free(orc_result* r);
/* Batched raw evaluation of an analytic program (oracle-side field). */
int orc_eval_raw(const orc_node* prog, int32_t n_nodes, const double* pts, int64_t n, double* raw);
/* Exhaustive single-cell partition helper (dualize.py:266-296 semantics with
 * the global instance order): returns number of cycles. */
int orc_version(void);
#ifdef __cplusplus
}
#endif
#endif
