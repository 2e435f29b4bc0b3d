"""Golden outputs of the reference's mesh checks: occmesh.mesh.validate_manifold
(mesh.py:91-150) and count_self_intersections (mesh.py:395-487), run here on
the golden meshes (raw and repaired) and on small synthetic meshes that hit
every branch (pinched vertices, boundary and isolated vertices, crossing and
coplanar-overlapping triangle pairs, degenerate triangles).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_checks_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
from occmesh.mesh import TriangleMesh, count_self_intersections, icosphere, validate_manifold  # noqa: E402


def synthetic():
    out = {}
    # two tetrahedra-like cones sharing an apex -> pinched apex
    v = np.array([[0, 0, 0], [1, 0, 1], [0, 1, 1], [-1, -1, 1], [1, 0, -1], [0, 1, -1], [-1, -1, -1.0]])
    t = np.array([[0, 1, 2], [0, 2, 3], [0, 3, 1], [1, 3, 2], [0, 5, 4], [0, 6, 5], [0, 4, 6], [4, 5, 6]])
    out["double_cone"] = (v, t)
    # open strip + two isolated vertices
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0], [2, 0, 0], [5, 5, 5], [6, 6, 6.0]])
    t = np.array([[0, 1, 2], [1, 3, 2], [1, 4, 3]])
    out["open_strip"] = (v, t)
    # fin: three triangles on one edge (non-manifold edge) + a crossing pair
    v = np.array([[0, 0, 0], [1, 0, 0], [0.5, 1, 0], [0.5, -1, 0.2], [0.5, 0.3, 1],
                  [0.2, 0.2, -0.5], [0.8, 0.3, 0.5], [0.3, 0.6, 0.5]])
    t = np.array([[0, 1, 2], [0, 1, 3], [1, 0, 4], [5, 6, 7]])
    out["fin_cross"] = (v, t)
    # coplanar overlapping triangles (no shared vertex) + a degenerate one
    v = np.array([[0, 0, 0], [2, 0, 0], [0, 2, 0], [0.5, 0.5, 0], [2.5, 0.5, 0], [0.5, 2.5, 0],
                  [3, 3, 3], [3, 3, 3.0 + 1e-15], [3, 3, 3.0 + 2e-15]])
    t = np.array([[0, 1, 2], [3, 4, 5], [6, 7, 8]])
    out["coplanar"] = (v, t)
    ico = icosphere(subdivisions=2)
    out["icosphere"] = (ico.vertices, ico.triangles)
    # icosphere pushed through itself: one cap reflected inward
    v = ico.vertices.copy()
    cap = v[:, 2] > 0.6
    v[cap, 2] = 1.2 - v[cap, 2] - 0.9
    out["dented"] = (v, ico.triangles.copy())
    return out


def main():
    meshes = {k: v for k, v in synthetic().items()}
    np.savez_compressed(HERE / "checks_meshes.npz",
                        **{f"{k}_v": v for k, (v, t) in meshes.items()},
                        **{f"{k}_t": t for k, (v, t) in meshes.items()})
    for name in ("sphere_32", "torus_64", "mlp_amp4_32", "mlp_amp1_32", "thin_shell_64"):
        d = np.load(HERE / f"{name}.npz")
        meshes[name] = (d["vertices"], d["triangles"])
        meshes[name + "_raw"] = (d["raw_vertices"], d["raw_triangles"])
    out = {}
    for name, (v, t) in meshes.items():
        m = TriangleMesh(v, t)
        r = validate_manifold(m)
        n, pairs = count_self_intersections(m, return_pairs=True)
        out[name] = {
            "manifold": bool(r.manifold), "nonmanifold_edges": [list(e) for e in r.nonmanifold_edges],
            "pinched_vertices": list(map(int, r.pinched_vertices)), "boundary_edges": int(r.boundary_edges),
            "isolated_vertices": list(map(int, r.isolated_vertices)),
            "si_count": int(n), "si_pairs": [list(map(int, p)) for p in pairs],
        }
        print(name, out[name]["manifold"], len(out[name]["nonmanifold_edges"]), out[name]["boundary_edges"],
              len(out[name]["pinched_vertices"]), len(out[name]["isolated_vertices"]), n)
    (HERE / "checks.json").write_text(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
