"""CPU restatement of the generalized winding number of MeshWindingField --
TEST INFRASTRUCTURE ONLY (the product evaluates it in csrc/odc_winding.cu).

Follows _winding_batch (/root/reference/pkg/src/occmesh/fields.py:281-357):
per (point, triangle) the Van Oosterom-Strackee solid angle
2 atan2(a.(b x c), |a||b||c| + (a.b)|c| + (b.c)|a| + (c.a)|b|), summed over
the triangles (numpy's pairwise sum of a contiguous row) and divided by
4 pi; a query within 1e-12 of a triangle's plane and inside it (barycentric
slack 1e-12) is nudged by k * 1e-9 * scale / sqrt(3) along (1, 1, 1) on
attempt k, at most 8 attempts.  Pinned to the reference's own values
(tests/golden/winding_golden.npz, made by make_winding_golden.py).
"""

from __future__ import annotations

import math

import numpy as np


def _ein(a, b):  # numpy's 3-term einsum order: (x0 y0 + x2 y2) + x1 y1
    return (a[..., 0] * b[..., 0] + a[..., 2] * b[..., 2]) + a[..., 1] * b[..., 1]


def _norm(a):
    return np.sqrt((a[..., 0] * a[..., 0] + a[..., 1] * a[..., 1]) + a[..., 2] * a[..., 2])


def _cross(a, b):
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)


def winding(vertices, triangles, points, chunk=512):
    V = np.asarray(vertices, dtype=np.float64)
    T = np.asarray(triangles, dtype=np.int64)
    P = np.array(points, dtype=np.float64).reshape(-1, 3)
    A, B, C = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    eab, eac = B - A, C - A
    n = _cross(eab, eac)
    ln = _norm(n)
    ok = ln > 0
    nh = np.zeros_like(n)
    nh[ok] = n[ok] / ln[ok, None]
    d00, d01, d11 = _ein(eab, eab), _ein(eab, eac), _ein(eac, eac)
    db = d00 * d11 - d01 * d01
    db = np.where(np.abs(db) < 1e-300, 1.0, db)
    scale = float(np.max(V.max(axis=0) - V.min(axis=0))) or 1.0
    nudge = 1e-9 * scale * np.ones(3) / math.sqrt(3.0)
    out = np.empty(len(P))
    for s in range(0, len(P), chunk):
        p = P[s:s + chunk].copy()
        for attempt in range(8):
            a = A[None] - p[:, None]
            b = B[None] - p[:, None]
            c = C[None] - p[:, None]
            la, lb, lc = _norm(a), _norm(b), _norm(c)
            num = _ein(a, _cross(b, c))
            den = ((la * lb * lc + _ein(a, b) * lc) + _ein(b, c) * la) + _ein(c, a) * lb
            near = (np.abs(_ein(a, nh[None])) <= 1e-12) & ok[None]
            bad = np.zeros(len(p), dtype=bool)
            if near.any():
                pi, ti = np.nonzero(near)
                ap = p[pi] - A[ti]
                d20, d21 = _ein(ap, eab[ti]), _ein(ap, eac[ti])
                v = (d11[ti] * d20 - d01[ti] * d21) / db[ti]
                w = (d00[ti] * d21 - d01[ti] * d20) / db[ti]
                hit = (v >= -1e-12) & (w >= -1e-12) & (v + w <= 1 + 1e-12)
                bad[pi[hit]] = True
            if bad.any():
                p[bad] += nudge * (attempt + 1)
                continue
            out[s:s + chunk] = (2.0 * np.arctan2(num, den)).sum(axis=1) / (4.0 * math.pi)
            break
        else:
            raise ValueError("could not perturb queries off the surface")
    return out
