"""CPU oracle for the ODC extraction path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) import this package, and only as the checker / the CPU
baseline.  The product package never imports it.

``contour_oracle`` runs the plain-C lock-step restatement of
occmesh.pipeline.contour (/root/reference/pkg/src/occmesh/pipeline.py:154-240)
in odc_oracle.c and returns every intermediate as numpy arrays.  Analytic
fields are lowered to the same postfix program the device uses; any other
field is evaluated through a Python callback (numpy MlpField below, or the
GPU evaluator for the shared-field oracle).

Pinned against the unmodified reference by tests/test_oracle_golden.py
(golden vectors from tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libodc_oracle.so"

CATEGORIES = ("labels", "search_1d", "probe_face_center", "probe_face_midpoint", "search_2d", "fd_gradient")
STATUS_NAMES = {0: "exact", 1: "midpoint-fallback", 2: "clamped", 3: "range-exhausted"}
ERRORS = {1: AssertionError, 2: RuntimeError, 3: ValueError, 4: ValueError, 5: MemoryError}


def build():
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)


class _Node(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("pad", ctypes.c_int32), ("p", ctypes.c_double * 16)]


class _Options(ctypes.Structure):
    _fields_ = [
        ("one_d", ctypes.c_int32), ("normals", ctypes.c_int32), ("split", ctypes.c_int32),
        ("repair", ctypes.c_int32), ("iters_1d", ctypes.c_int32),
        ("s1_lin", ctypes.c_int32), ("s1_bin", ctypes.c_int32),
        ("s2_lin", ctypes.c_int32), ("s2_bin", ctypes.c_int32),
        ("continuous", ctypes.c_int32),
        ("s1_range", ctypes.c_double), ("s2_range", ctypes.c_double),
        ("qef_truncation", ctypes.c_double), ("fd_step_factor", ctypes.c_double),
        ("iso_level", ctypes.c_double),
        ("dsyevd", ctypes.c_void_p),
    ]


_P = ctypes.POINTER
_i64p = _P(ctypes.c_int64)
_f64p = _P(ctypes.c_double)
_u8p = _P(ctypes.c_uint8)


class _Result(ctypes.Structure):
    _fields_ = [
        ("S", ctypes.c_int64), ("R", ctypes.c_int64), ("h", ctypes.c_double * 3),
        ("labels", _u8p), ("raw", _f64p), ("boundary_inside", ctypes.c_int64),
        ("K", ctypes.c_int64), ("edge_key", _i64p), ("v_in", _i64p), ("v_out", _i64p),
        ("F", ctypes.c_int64), ("face_key", _i64p), ("face_ncross", _i64p),
        ("C", ctypes.c_int64), ("cells", _i64p), ("F4", ctypes.c_int64),
        ("Q", ctypes.c_int64), ("inst_face_row", _i64p), ("inst_edges", _i64p),
        ("t1d", _f64p), ("pos1d", _f64p),
        ("pos2", _f64p), ("pos3", _f64p), ("status", _u8p), ("mid_label", _u8p),
        ("P", ctypes.c_int64), ("Ns", ctypes.c_int64),
        ("part_cell", _i64p), ("part_index", _i64p), ("cyc_off", _i64p), ("cyc_edges", _i64p), ("cyc_insts", _i64p),
        ("normals", _f64p), ("n_fallback", ctypes.c_int64),
        ("qef_pos", _f64p), ("qef_resid", _f64p), ("qef_rank", _i64p),
        ("n_interior", ctypes.c_int64), ("skipped", ctypes.c_int64), ("split_cases", _P(ctypes.c_int8)),
        ("V0", ctypes.c_int64), ("T0", ctypes.c_int64),
        ("v0", _f64p), ("t0", _i64p), ("kind0", _i64p), ("ref0", _i64p),
        ("V1", ctypes.c_int64), ("T1", ctypes.c_int64),
        ("v1", _f64p), ("t1", _i64p), ("kind1", _i64p), ("ref1", _i64p),
        ("eval_batches", ctypes.c_int64 * 6), ("eval_evals", ctypes.c_int64 * 6),
        ("cat_order", ctypes.c_int32 * 6),
        ("error", ctypes.c_int32), ("errmsg", ctypes.c_char * 256),
    ]


_CB = ctypes.CFUNCTYPE(None, _f64p, ctypes.c_int64, _f64p, ctypes.c_int32, ctypes.c_void_p)
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.orc_contour.argtypes = [
            _P(_Node), ctypes.c_int32, _CB, ctypes.c_void_p,
            _f64p, _f64p, ctypes.c_int64, _P(_Options), _P(_Result),
        ]
        L.orc_contour.restype = ctypes.c_int
        L.orc_free.argtypes = [_P(_Result)]
        L.orc_eval_raw.argtypes = [_P(_Node), ctypes.c_int32, _f64p, ctypes.c_int64, _f64p]
        _lib = L
    return _lib


def _arr(ptr, n, dtype, shape=None):
    if n == 0 or not ptr:
        out = np.zeros(0, dtype=dtype)
    else:
        out = np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)
    if shape is not None:
        out = out.reshape(shape)
    return out


def _program(field):
    from paper_2409_13418_b200.fields import lower_program

    prog = lower_program(field)
    nodes = (_Node * max(1, len(prog)))()
    for i, n in enumerate(prog):
        nodes[i].op = int(n["op"])
        for j in range(16):
            nodes[i].p[j] = float(n["p"][j])
    return nodes, len(prog)


def eval_raw_program(field, points):
    """Analytic program evaluated by the oracle interpreter (fields.py semantics)."""
    nodes, n = _program(field)
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    out = np.empty(len(pts))
    lib().orc_eval_raw(nodes, n, pts.ctypes.data_as(_f64p), len(pts), out.ctypes.data_as(_f64p))
    return out


def _opts(options, continuous, iso):
    o = _Options()
    one_d = {"binary-search": 0, "midpoint": 1, "linear-interp": 2}
    nrm = {"two-d-points": 0, "fd-gradient": 1}
    spl = {"ic": 0, "mdc": 1}
    if options is None:
        o.one_d, o.normals, o.split, o.repair = 0, 0, 0, 1
        o.iters_1d, o.s1_lin, o.s1_bin, o.s1_range = 15, 4, 11, 0.8
        o.s2_lin, o.s2_bin, o.s2_range = 3, 12, math.sqrt(2.0) / 2.0
        o.qef_truncation, o.fd_step_factor = 0.1, 0.01
    else:
        o.one_d = one_d.get(options.one_d, -1)
        o.normals = nrm.get(options.normals, -1)
        o.split = spl.get(options.split, -1)
        o.repair = int(bool(options.repair))
        b = options.budget
        o.iters_1d = b.iters_1d
        o.s1_lin, o.s1_bin, o.s1_range = b.step1.n_linear, b.step1.n_binary, b.step1.max_range_factor
        o.s2_lin, o.s2_bin, o.s2_range = b.step2.n_linear, b.step2.n_binary, b.step2.max_range_factor
        o.qef_truncation, o.fd_step_factor = options.qef_truncation, options.fd_step_factor
    o.continuous = int(bool(continuous))
    o.iso_level = float(iso)
    return o


def numpy_dsyevd():
    """Address of the LAPACK dsyevd that numpy.linalg.eigh uses (scipy-openblas)."""
    import glob

    libs = glob.glob(str(Path(np.__file__).resolve().parent.parent / "numpy.libs" / "libscipy_openblas64_*.so"))
    if not libs:
        return None
    L = ctypes.CDLL(libs[0])
    for name in ("scipy_dsyevd_64_", "dsyevd_64_", "dsyevd_"):
        try:
            return ctypes.cast(getattr(L, name), ctypes.c_void_p).value
        except AttributeError:
            continue
    return None


def contour_oracle(field, lo, hi, resolution, options=None, raw_fn=None, continuous=None):
    """Run the C oracle.  ``raw_fn(points (N,3) f64, category:str) -> (N,) f64``
    evaluates non-analytic fields (MLP / shared GPU field)."""
    from paper_2409_13418_b200.fields import field_continuous, is_mlp

    L = lib()
    if continuous is None:
        continuous = field_continuous(field)
    iso = float(getattr(field, "iso_level", 0.5))
    cb = None
    if raw_fn is None and is_mlp(field):
        raw_fn = lambda pts, cat: mlp_raw_numpy(field, pts)  # noqa: E731
    if raw_fn is not None:
        nodes, n = (_Node * 1)(), 0

        def _cb(p, n_, out, cat, user):
            pts = np.ctypeslib.as_array(p, shape=(n_, 3))
            vals = np.asarray(raw_fn(pts, CATEGORIES[cat]), dtype=np.float64)
            np.ctypeslib.as_array(out, shape=(n_,))[:] = vals

        cb = _CB(_cb)
    else:
        nodes, n = _program(field)
        cb = _CB()
    lo = (ctypes.c_double * 3)(*[float(v) for v in lo])
    hi = (ctypes.c_double * 3)(*[float(v) for v in hi])
    res = _Result()
    o = _opts(options, continuous, iso)
    o.dsyevd = numpy_dsyevd()  # the QEF eigensolve is numpy's own LAPACK (dualize.py:358)
    if not o.dsyevd:
        raise RuntimeError("numpy's LAPACK dsyevd not found")
    rc = L.orc_contour(nodes, n, cb, None, lo, hi, int(resolution), ctypes.byref(o), ctypes.byref(res))
    try:
        if rc:
            raise ERRORS.get(rc, RuntimeError)(res.errmsg.decode())
        return _collect(res)
    finally:
        L.orc_free(ctypes.byref(res))


def _collect(r):
    S = r.S
    K, F, C, Q, P, Ns = r.K, r.F, r.C, r.Q, r.P, r.Ns
    d = dict(
        S=S, R=r.R, h=np.array(list(r.h)),
        labels=_arr(r.labels, S**3, np.uint8),
        raw=_arr(r.raw, S**3 if r.raw else 0, np.float64),
        boundary_inside=r.boundary_inside,
        edge_key=_arr(r.edge_key, K, np.int64), v_in=_arr(r.v_in, K, np.int64), v_out=_arr(r.v_out, K, np.int64),
        face_key=_arr(r.face_key, F, np.int64), face_n_crossing=_arr(r.face_ncross, F, np.int64),
        cells=_arr(r.cells, C, np.int64), n_probes=r.F4,
        instance_face_row=_arr(r.inst_face_row, Q if K else 0, np.int64),
        instance_edges=_arr(r.inst_edges, 2 * Q if K else 0, np.int64, (-1, 2)),
        t1d=_arr(r.t1d, K, np.float64), pos1d=_arr(r.pos1d, 3 * K, np.float64, (-1, 3)),
        pos2=_arr(r.pos2, 2 * Q if r.pos2 else 0, np.float64, (-1, 2)),
        pos3=_arr(r.pos3, 3 * Q if r.pos3 else 0, np.float64, (-1, 3)),
        status=_arr(r.status, Q if r.status else 0, np.uint8),
        mid_label=_arr(r.mid_label, Q if r.mid_label else 0, np.uint8),
        part_cell=_arr(r.part_cell, P, np.int64), part_index=_arr(r.part_index, P, np.int64),
        cyc_off=_arr(r.cyc_off, P + 1 if P else 0, np.int64),
        cyc_edges=_arr(r.cyc_edges, Ns, np.int64), cyc_insts=_arr(r.cyc_insts, Ns, np.int64),
        normals=_arr(r.normals, 3 * Ns, np.float64, (-1, 3)), n_fallback=r.n_fallback,
        qef_pos=_arr(r.qef_pos, 3 * P, np.float64, (-1, 3)), qef_rank=_arr(r.qef_rank, P, np.int64),
        qef_resid=_arr(r.qef_resid, P, np.float64),
        split_cases=_arr(r.split_cases, r.n_interior, np.int8).astype(np.int64), skipped=r.skipped,
        raw_vertices=_arr(r.v0, 3 * r.V0, np.float64, (-1, 3)), raw_triangles=_arr(r.t0, 3 * r.T0, np.int64, (-1, 3)),
        raw_kind=_arr(r.kind0, r.V0, np.int64), raw_ref=_arr(r.ref0, 2 * r.V0, np.int64, (-1, 2)),
        vertices=_arr(r.v1, 3 * r.V1, np.float64, (-1, 3)), triangles=_arr(r.t1, 3 * r.T1, np.int64, (-1, 3)),
        kind=_arr(r.kind1, r.V1, np.int64), ref=_arr(r.ref1, 2 * r.V1, np.int64, (-1, 2)),
    )
    counts = {}
    for c in list(r.cat_order):
        if c < 0:
            break
        counts[CATEGORIES[c]] = {"batches": int(r.eval_batches[c]), "evals": int(r.eval_evals[c])}
    counts["total_evals"] = sum(v["evals"] for k, v in counts.items() if k != "total_evals")
    d["eval_counts"] = counts
    return d


# ---------------------------------------------------------------------------
# numpy MlpField evaluation (CPU baseline / label-agreement statistics)
# ---------------------------------------------------------------------------
def mlp_encode_numpy(field, pts):
    x = (np.asarray(pts, dtype=np.float64) - 0.5)
    feats = [x]
    for k in range(field.n_freq):
        arg = (math.pi * (2.0**k)) * x
        feats.append(np.sin(arg))
        feats.append(np.cos(arg))
    return np.concatenate(feats, axis=1).astype(np.float32)


def mlp_logit_numpy(field, pts, chunk=1 << 16):
    pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    out = np.empty(len(pts))
    for s in range(0, len(pts), chunk):
        p = pts[s:s + chunk]
        h = mlp_encode_numpy(field, p)
        for w, b in zip(field.weights, field.biases):
            h = np.maximum(h @ w + b, 0.0, dtype=np.float32)
        mlp = (h @ field.w_head.astype(np.float32)).astype(np.float64) + field.b_head
        d = np.linalg.norm(p - field.prior_center, axis=1)
        out[s:s + chunk] = field.amplitude * mlp - field.prior_scale * (d - field.prior_radius)
    return out


def mlp_dot_bf16_numpy(field, pts, chunk=1 << 15):
    """The head dot product h_7 . w_head as the device evaluator computes it
    in exact arithmetic where it rounds: fp32 encoding x = (float)(p - 0.5)
    and sin/cos(pi 2^k x) rounded to fp32, every layer input rounded to bf16
    (RNE), products exact, sums in fp64 then rounded to fp32 (the tensor
    core accumulates in fp32 in its own order), bias + ReLU, and the head in
    fp32 activations (not bf16).  The device differs from this only by its
    fp32 accumulation order and sincospif's last ulp (a bf16 rounding of an
    activation may then fall the other way): tests/test_gpu_mlp.py bounds
    the difference.  Test infrastructure only."""
    from paper_2409_13418_b200.fields import bf16_round

    pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    out = np.empty(len(pts), dtype=np.float32)
    W = [np.asarray(w, dtype=np.float64) for w in field.weights]
    B = [np.asarray(b, dtype=np.float32) for b in field.biases]
    wh = np.asarray(field.w_head, dtype=np.float64)
    for s0 in range(0, len(pts), chunk):
        x = (pts[s0:s0 + chunk] - 0.5).astype(np.float32)
        feats = [x]
        for k in range(field.n_freq):
            arg = np.pi * (x.astype(np.float64) * (2.0**k))
            feats.append(np.sin(arg).astype(np.float32))
            feats.append(np.cos(arg).astype(np.float32))
        h = bf16_round(np.concatenate(feats, axis=1)).astype(np.float64)
        for i in range(len(W)):
            acc = (h @ W[i]).astype(np.float32) + B[i]
            acc = np.maximum(acc, np.float32(0))
            h = (bf16_round(acc) if i + 1 < len(W) else acc).astype(np.float64)
        out[s0:s0 + chunk] = (h @ wh).astype(np.float32)
    return out


def mlp_raw_numpy(field, pts):
    z = mlp_logit_numpy(field, pts)
    return 1.0 / (1.0 + np.exp(-np.clip(z, -500.0, 500.0)))
