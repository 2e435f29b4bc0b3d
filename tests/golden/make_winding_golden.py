"""Golden winding numbers and a mesh-field extraction from the reference:
occmesh.fields._winding_batch (fields.py:281-357) on an icosphere and on a
torus-like open/closed mix, and occmesh.pipeline.contour on a
MeshWindingField at a small resolution.

    python tests/golden/make_winding_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
from occmesh import GridSpec  # noqa: E402
from occmesh.fields import MeshWindingField, _winding_batch  # noqa: E402
from occmesh.mesh import icosphere  # noqa: E402
from occmesh.pipeline import contour  # noqa: E402


def main():
    ico = icosphere(center=(0.5, 0.5, 0.5), radius=0.3, subdivisions=3)
    rng = np.random.default_rng(4)
    pts = np.concatenate([rng.random((600, 3)), ico.vertices[:40],  # on-surface queries (perturbed)
                          0.5 + 0.3 * rng.normal(size=(200, 3)) / np.sqrt(3)])
    w_ico = _winding_batch(ico.vertices, ico.triangles, pts, on_surface="perturb")
    # an open mesh: the icosphere minus its upper cap
    keep = ico.vertices[ico.triangles][:, :, 2].max(axis=1) < 0.7
    open_t = ico.triangles[keep]
    w_open = _winding_batch(ico.vertices, open_t, pts[:600], on_surface="perturb")
    R = 24
    res = contour(MeshWindingField(ico.vertices, ico.triangles), GridSpec((0, 0, 0), (1, 1, 1), R))
    np.savez_compressed(HERE / "winding_golden.npz", ico_v=ico.vertices, ico_t=ico.triangles, open_t=open_t,
                        points=pts, w_ico=w_ico, w_open=w_open, mesh_v=res.mesh.vertices, mesh_t=res.mesh.triangles,
                        raw_v=res.raw_mesh.vertices, raw_t=res.raw_mesh.triangles, R=R)
    print(len(pts), res.mesh.n_vertices, res.mesh.n_triangles, res.stats["eval_counts"]["total_evals"])


if __name__ == "__main__":
    main()
