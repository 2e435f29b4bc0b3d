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
