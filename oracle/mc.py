"""CPU restatement of the marching-cubes baseline -- TEST INFRASTRUCTURE ONLY.

occmesh.baseline.marching_cubes (/root/reference/pkg/src/occmesh/
baseline.py:48-127) on top of the C oracle's stage outputs (labels, raw grid
values, crossing edges with their inside ends, partition cycles as edge
keys): one vertex per crossing edge (midpoint, or the inverse lerp of the raw
values in "continuous" mode), each cycle fanned from its first edge and
flipped when the fan normal (sum of the fan's cross products) points against
the summed edge directions (numpy's 1-D ``@`` is an fma chain), unused edge
vertices dropped.  Pinned to the reference's own outputs
(tests/golden/mc_golden.*, made by make_mc_golden.py).  Only tests/ may use
this module.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

from . import contour_oracle


def _fma(a, b, c):
    return float(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def marching_cubes_oracle(field, lo, hi, R, mode="binary", raw_fn=None):
    """(vertices, triangles, info) of the reference's marching_cubes."""
    if mode not in ("binary", "continuous"):
        raise ValueError(mode)
    d = contour_oracle(field, lo, hi, R, raw_fn=raw_fn)
    S = d["S"]
    h = d["h"]
    lo = np.asarray(lo, dtype=np.float64)
    info = {"boundary_inside_vertices": int(d["boundary_inside"]), "n_crossing_edges": len(d["edge_key"]),
            "n_crossing_cells": len(d["cells"])}
    K = len(d["edge_key"])
    if K == 0:
        return np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64), info

    def pos(v):
        c = np.stack([v % S, (v // S) % S, v // (S * S)], axis=1).astype(np.float64)
        return lo + c * h

    p_in, p_out = pos(d["v_in"]), pos(d["v_out"])
    if mode == "binary":
        t = np.full(K, 0.5)
    else:
        raw = d["raw"]
        if len(raw) == 0:
            raise ValueError("continuous marching cubes requires a field with raw values")
        iso = float(getattr(field, "iso_level", 0.5))
        a, b = raw[d["v_in"]] - iso, raw[d["v_out"]] - iso
        den = a - b
        with np.errstate(divide="ignore", invalid="ignore"):
            t = np.clip(a / np.where(np.abs(den) < 1e-300, 1.0, den), 0.0, 1.0)
    verts = p_in + t[:, None] * (p_out - p_in)
    dirs = p_out - p_in
    row_of = {int(k): i for i, k in enumerate(d["edge_key"])}
    tris = []
    off = d["cyc_off"]
    for pid in range(len(off) - 1):
        rows = [row_of[int(k)] for k in d["cyc_edges"][off[pid]:off[pid + 1]]]
        if len(rows) < 3:
            continue
        fan = [(rows[0], rows[j], rows[j + 1]) for j in range(1, len(rows) - 1)]
        n = np.zeros(3)
        for a, b, c in fan:
            n = n + np.cross(verts[b] - verts[a], verts[c] - verts[a])
        o = dirs[rows[0]].copy()
        for r in rows[1:]:
            o = o + dirs[r]
        dot = _fma(n[2], o[2], _fma(n[1], o[1], n[0] * o[0]))
        if dot < 0:
            fan = [(a, c, b) for a, b, c in fan]
        tris.extend(fan)
    t = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    used = np.zeros(K, dtype=bool)
    used[t.reshape(-1)] = True
    remap = -np.ones(K, dtype=np.int64)
    remap[used] = np.arange(int(used.sum()))
    info["open_boundary"] = bool((~used).any()) and info["boundary_inside_vertices"] > 0
    return verts[used], remap[t], info
