"""Golden vectors for repair_nonmanifold (polygonize.py:253-374) on synthetic
meshes whose vertex fans exceed 64 triangles (the device's local-array fan
size; larger fans take the global-scratch path).  Generated from the
UNMODIFIED reference in the build container:

    python tests/golden/make_repair_golden.py
"""

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from occmesh.mesh import TriangleMesh  # noqa: E402
from occmesh.polygonize import repair_nonmanifold  # noqa: E402


def disk(apex, normal_axis, m, r, z, flip):
    """Fan of m triangles around vertex 0 (the apex) over a ring of m
    vertices in a plane; returns (ring vertices, triangles in ring ids)."""
    ang = 2 * np.pi * np.arange(m) / m
    ring = np.zeros((m, 3))
    a, b = [(1, 2), (0, 2), (0, 1)][normal_axis]
    ring[:, a], ring[:, b] = r * np.cos(ang), r * np.sin(ang)
    ring[:, normal_axis] = z
    ring += apex
    tris = [(0, 1 + j, 1 + (j + 1) % m) for j in range(m)]
    if flip:
        tris = [(t[0], t[2], t[1]) for t in tris]
    return ring, tris


def bowtie(m1=50, m2=47):
    """Two disks sharing an apex: the apex fan has m1 + m2 triangles in two
    components (one duplicate vertex)."""
    apex = np.array([0.5, 0.5, 0.5])
    r1, t1 = disk(apex, 2, m1, 0.2, 0.1, False)
    r2, t2 = disk(apex, 2, m2, 0.2, -0.1, True)
    verts = np.concatenate([apex[None], r1, r2])
    tris = [t for t in t1] + [(0, a + m1 if a else 0, b + m1 if b else 0) for _, a, b in t2]
    return verts, np.array(tris, dtype=np.int64)


def book(pages=4, m=20, seed=0):
    """``pages`` fans around vertex a = 0, each containing the spine edge
    (0, 1): the spine edge has ``pages`` triangles (sheet pairing by dihedral
    angle) and vertex 0 has pages * m triangles; pages alternate traversal
    direction so both pairing branches are exercised."""
    rng = np.random.default_rng(seed)
    a = np.array([0.5, 0.5, 0.3])
    b = np.array([0.5, 0.5, 0.7])
    verts = [a, b]
    tris = []
    for k in range(pages):
        th = 2 * np.pi * k / pages + rng.uniform(-0.2, 0.2)
        d = np.array([np.cos(th), np.sin(th), 0.0])
        ids = [1]
        for j in range(1, m + 1):
            phi = np.pi * j / (m + 1)
            p = a + 0.4 * (np.cos(phi) * np.array([0, 0, 1.0]) + np.sin(phi) * d)
            verts.append(p)
            ids.append(len(verts) - 1)
        for j in range(m):
            t = (0, ids[j], ids[j + 1])
            tris.append(t if (k % 2 == 0) else (t[0], t[2], t[1]))
    return np.array(verts), np.array(tris, dtype=np.int64)


def main():
    cases = {"bowtie_97": bowtie(), "book_4x20": book(4, 20), "book_6x13": book(6, 13, seed=1),
             "bowtie_small": bowtie(5, 6)}
    out = {}
    for name, (v, t) in cases.items():
        n = len(v)
        mesh = TriangleMesh(v, t, provenance_kind=np.zeros(n, np.int64),
                            provenance_ref=np.stack([np.arange(n), np.zeros(n, np.int64)], 1))
        r = repair_nonmanifold(mesh)
        out[f"{name}__in_vertices"] = v
        out[f"{name}__in_triangles"] = t
        out[f"{name}__vertices"] = r.vertices
        out[f"{name}__triangles"] = r.triangles
        out[f"{name}__kind"] = r.provenance_kind
        out[f"{name}__ref"] = r.provenance_ref
        print(name, "V", n, "->", len(r.vertices), "T", len(t), "max fan",
              np.bincount(t.ravel()).max())
    np.savez_compressed(HERE / "repair_golden.npz", **out)


if __name__ == "__main__":
    main()
