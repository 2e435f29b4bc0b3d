"""CPU restatement of the reference's mesh checks -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's reference leg may use
this module, and only as the checker; the product computes these checks on
the GPU (libodc, csrc/odc_validate.cu).  Pinned against the reference's own
outputs on golden and synthetic meshes (tests/golden/checks.json, made by
tests/golden/make_checks_golden.py).

* validate_manifold -- /root/reference/pkg/src/occmesh/mesh.py:91-150:
  edge multiplicities over undirected edges (>2 non-manifold, ==1 boundary),
  per-vertex union of incident triangles through shared neighbour vertices
  (more than one component = pinched), unused vertices = isolated; an empty
  triangle list is reported manifold with empty lists.
* count_self_intersections -- mesh.py:395-487 with _tri_tri_cross
  (:300-349) and _coplanar_overlap_area (:368-392): unit-box normalisation,
  uniform-hash broad phase (cell = 1.0001 x the largest triangle box side),
  vertex-sharing / degenerate / box rejects, exact interval test in numpy
  fp64 (same expression order), coplanar pairs by clipped overlap area.
* mesh_distance -- MeshDistanceIndex.query (mesh.py:202-270) by brute force:
  Ericson's closest point (_closest_point_on_triangles, mesh.py:153-199) to
  every triangle and the minimum distance; on exact ties the winner is the
  first of the 8 nearest centroids attaining it (the reference's KD-tree
  pass; equal centroid distances by index), else the smallest index.
"""

from __future__ import annotations

from collections import defaultdict

import numpy as np


def validate_manifold(vertices, triangles):
    """(manifold, nonmanifold_edges, pinched, boundary, isolated) as plain
    Python values, following mesh.py:91-150."""
    t = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
    nv = len(vertices)
    if len(t) == 0:
        return True, [], [], 0, []
    mult = defaultdict(int)
    for a, b, c in t.tolist():
        for u, w in ((a, b), (b, c), (c, a)):
            mult[(u, w) if u < w else (w, u)] += 1
    nonmanifold = sorted(e for e, k in mult.items() if k > 2)
    boundary = sum(1 for k in mult.values() if k == 1)

    fans = defaultdict(list)
    for ti, tri in enumerate(t.tolist()):
        for x in tri:
            fans[x].append(ti)
    pinched = []
    for vid in sorted(fans):
        tl = sorted(set(fans[vid]))
        if len(tl) <= 1:
            continue
        parent = list(range(len(tl)))

        def root(i):
            while parent[i] != i:
                parent[i] = parent[parent[i]]
                i = parent[i]
            return i

        seen = {}
        for i, ti in enumerate(tl):
            for x in t[ti].tolist():
                if x == vid:
                    continue
                if x in seen:
                    ra, rb = root(seen[x]), root(i)
                    if ra != rb:
                        parent[ra] = rb
                else:
                    seen[x] = i
        if len({root(i) for i in range(len(tl))}) > 1:
            pinched.append(vid)
    used = np.zeros(nv, dtype=bool)
    used[t.reshape(-1)] = True
    isolated = np.nonzero(~used)[0].tolist()
    return (not nonmanifold and not pinched), [list(e) for e in nonmanifold], pinched, boundary, isolated


def _cross(a, b):
    return np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1],
                     a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
                     a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], axis=1)


def _dot(a, b):  # numpy's 3-term einsum('ij,ij->i') order: (p0 + p2) + p1
    return (a[:, 0] * b[:, 0] + a[:, 2] * b[:, 2]) + a[:, 1] * b[:, 1]


def _norm(a):  # np.linalg.norm(axis=1) order: (x0^2 + x1^2) + x2^2
    return np.sqrt((a[:, 0] * a[:, 0] + a[:, 1] * a[:, 1]) + a[:, 2] * a[:, 2])


def _pair_test(P, Q, tol):
    """(crossing, coplanar) per pair, arrays of (n, 3, 3) corners."""
    n1 = _cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0])
    n2 = _cross(Q[:, 1] - Q[:, 0], Q[:, 2] - Q[:, 0])
    dq = np.stack([_dot(Q[:, k] - P[:, 0], n1) for k in range(3)], axis=1)
    dp = np.stack([_dot(P[:, k] - Q[:, 0], n2) for k in range(3)], axis=1)
    tq = tol * np.maximum(_norm(n1), 1e-300)[:, None]
    tp = tol * np.maximum(_norm(n2), 1e-300)[:, None]
    sep = (dq > tq).all(1) | (dq < -tq).all(1) | (dp > tp).all(1) | (dp < -tp).all(1)
    cop = (np.abs(dq) <= tq).all(1) & (np.abs(dp) <= tp).all(1)
    d = _cross(n1, n2)
    ax = np.argmax(np.abs(d), axis=1)

    def span(T, dist, tl):
        pr = T[np.arange(len(T)), :, ax]
        sg = np.where(dist > tl, 1, -1)
        lo = np.full(len(T), np.inf)
        hi = np.full(len(T), -np.inf)
        for i in range(3):
            j = (i + 1) % 3
            m = sg[:, i] * sg[:, j] < 0
            df = dist[:, i] - dist[:, j]
            with np.errstate(divide="ignore", invalid="ignore"):
                tt = pr[:, i] + (pr[:, j] - pr[:, i]) * (dist[:, i] / np.where(np.abs(df) < 1e-300, 1.0, df))
            lo = np.where(m, np.minimum(lo, tt), lo)
            hi = np.where(m, np.maximum(hi, tt), hi)
        return lo, hi

    with np.errstate(invalid="ignore"):
        l1, h1 = span(Q, dq, tq)
        l2, h2 = span(P, dp, tp)
        ov = np.minimum(h1, h2) - np.maximum(l1, l2)
        crossing = ~sep & ~cop & (ov > tol) & np.isfinite(ov)
    return crossing, cop & ~sep


def _clip_left(poly, a, b):
    out = []
    for i in range(len(poly)):
        c, n = poly[i], poly[(i + 1) % len(poly)]
        sc = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])
        sn = (b[0] - a[0]) * (n[1] - a[1]) - (b[1] - a[1]) * (n[0] - a[0])
        if sc >= 0:
            out.append(c)
        if sc * sn < 0:
            tt = sc / (sc - sn)
            out.append((c[0] + tt * (n[0] - c[0]), c[1] + tt * (n[1] - c[1])))
    return out


def _coplanar_area(P, Q):
    p = [np.float64(x) for x in P.reshape(-1)]
    u = [p[3] - p[0], p[4] - p[1], p[5] - p[2]]
    w = [p[6] - p[0], p[7] - p[1], p[8] - p[2]]
    n = [u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]]
    ax = int(np.argmax(np.abs(n)))
    k0, k1 = [k for k in range(3) if k != ax]
    A = [(P[i, k0], P[i, k1]) for i in range(3)]
    B = [(Q[i, k0], Q[i, k1]) for i in range(3)]
    if n[ax] < 0:
        A = A[::-1]
    nb = (B[1][0] - B[0][0]) * (B[2][1] - B[0][1]) - (B[1][1] - B[0][1]) * (B[2][0] - B[0][0])
    if nb < 0:
        B = B[::-1]
    poly = B
    for i in range(3):
        poly = _clip_left(poly, A[i], A[(i + 1) % 3])
        if len(poly) < 3:
            return 0.0
    area = 0.0
    for i in range(1, len(poly) - 1):
        area += 0.5 * abs((poly[i][0] - poly[0][0]) * (poly[i + 1][1] - poly[0][1])
                          - (poly[i + 1][0] - poly[0][0]) * (poly[i][1] - poly[0][1]))
    return area


def count_self_intersections(vertices, triangles, tolerance=1e-12):
    """Sorted list of intersecting (a, b) triangle pairs, a < b."""
    V = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
    T = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
    nt = len(T)
    if nt < 2:
        return []
    lo = V.min(axis=0)
    ext = float((V.max(axis=0) - lo).max()) or 1.0
    C = ((V - lo) / ext)[T]
    degen = 0.5 * _norm(_cross(C[:, 1] - C[:, 0], C[:, 2] - C[:, 0])) < 1e-20
    blo, bhi = C.min(axis=1), C.max(axis=1)
    cell = max(float((bhi - blo).max()) * 1.0001, 1e-9)
    ns = int(1.0 / cell) + 3
    ilo = np.floor(blo / cell).astype(np.int64)
    ihi = np.floor(bhi / cell).astype(np.int64)
    cells = {}
    for c in range(8):
        ix = ihi[:, 0] if c & 4 else ilo[:, 0]
        iy = ihi[:, 1] if c & 2 else ilo[:, 1]
        iz = ihi[:, 2] if c & 1 else ilo[:, 2]
        for tri, key in enumerate(((ix * ns + iy) * ns + iz).tolist()):
            cells.setdefault(key, set()).add(tri)
    cand = set()
    for members in cells.values():
        m = sorted(members)
        for i in range(len(m)):
            for j in range(i + 1, len(m)):
                cand.add((m[i], m[j]))
    if not cand:
        return []
    pa, pb = np.array(sorted(cand), dtype=np.int64).T
    share = (T[pa][:, :, None] == T[pb][:, None, :]).any(axis=(1, 2))
    keep = ~share & ~degen[pa] & ~degen[pb]
    keep &= ((blo[pa] <= bhi[pb] + tolerance) & (blo[pb] <= bhi[pa] + tolerance)).all(axis=1)
    pa, pb = pa[keep], pb[keep]
    if len(pa) == 0:
        return []
    crossing, cop = _pair_test(C[pa], C[pb], tolerance)
    hits = [(int(a), int(b)) for a, b in zip(pa[crossing], pb[crossing])]
    for i in np.nonzero(cop)[0]:
        if _coplanar_area(C[pa[i]], C[pb[i]]) > tolerance:
            hits.append((int(pa[i]), int(pb[i])))
    return sorted(hits)


def _closest(p, a, b, c):
    """Ericson's region walk, vectorised, first matching region wins."""
    ab, ac = b - a, c - a
    ap, bp, cp = p - a, p - b, p - c
    d1, d2 = _dot(ab, ap), _dot(ac, ap)
    d3, d4 = _dot(ab, bp), _dot(ac, bp)
    d5, d6 = _dot(ab, cp), _dot(ac, cp)
    vc = d1 * d4 - d3 * d2
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4

    def safe(x):
        return np.where(np.abs(x) < 1e-300, 1.0, x)

    with np.errstate(divide="ignore", invalid="ignore"):
        e43, e56 = d4 - d3, d5 - d6
        den = safe((va + vb) + vc)
        choices = [
            ((d1 <= 0) & (d2 <= 0), a),
            ((d3 >= 0) & (d4 <= d3), b),
            ((vc <= 0) & (d1 >= 0) & (d3 <= 0), a + ab * np.clip(d1 / safe(d1 - d3), 0, 1)[:, None]),
            ((d6 >= 0) & (d5 <= d6), c),
            ((vb <= 0) & (d2 >= 0) & (d6 <= 0), a + ac * np.clip(d2 / safe(d2 - d6), 0, 1)[:, None]),
            ((va <= 0) & (e43 >= 0) & (e56 >= 0), b + (c - b) * np.clip(e43 / safe(e43 + e56), 0, 1)[:, None]),
        ]
        out = a + ab * (vb / den)[:, None] + ac * (vc / den)[:, None]
    for m, val in reversed(choices):
        out = np.where(m[:, None], val, out)
    return out


def mesh_distance(vertices, triangles, points, chunk=256):
    """(distance, triangle, closest point) per query point, exact."""
    V = np.asarray(vertices, dtype=np.float64)
    T = np.asarray(triangles, dtype=np.int64)
    P = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    A, B, C = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    nt = len(T)
    dist = np.empty(len(P))
    tri = np.empty(len(P), dtype=np.int64)
    cpo = np.empty((len(P), 3))
    for s in range(0, len(P), chunk):
        q = P[s:s + chunk]
        qq = np.repeat(q, nt, axis=0)
        cp = _closest(qq, np.tile(A, (len(q), 1)), np.tile(B, (len(q), 1)), np.tile(C, (len(q), 1)))
        d = _norm(cp - qq).reshape(len(q), nt)
        k = np.argmin(d, axis=1)  # first minimum = smallest index on ties
        cen = (((A + B) + C) / 3.0)
        for r in range(len(q)):
            e = cen - q[r]
            d2 = (e[:, 0] * e[:, 0] + e[:, 1] * e[:, 1]) + e[:, 2] * e[:, 2]
            near = np.argsort(d2, kind="stable")[: min(8, nt)]
            hit = near[d[r, near] == d[r, k[r]]]
            if len(hit):
                k[r] = hit[0]
        dist[s:s + chunk] = d[np.arange(len(q)), k]
        tri[s:s + chunk] = k
        cpo[s:s + chunk] = cp.reshape(len(q), nt, 3)[np.arange(len(q)), k]
    return dist, tri, cpo
